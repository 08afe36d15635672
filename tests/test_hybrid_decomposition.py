"""Pin of the hybrid dense-core decomposition (NEXT-3) on the CPU, independent of
the CUDA path: the identity the hybrid path computes — route G (Alg. 2) with
the core wedges skipped, plus the butterflies of the core subgraph G[C] counted in full, plus the
mixed core pairs' terms (balanced a_c a_r + d_c d_r, unbalanced a_c d_r + a_r d_c to the pair and
its two ends; (a_c, d_c) or (d_c, a_c) to a non-core middle; (a_r, d_r) or (d_r, a_r) to a core
middle, by the middle's wedge class) — is evaluated here in plain Python, role by role, and must
equal the oracle's brute force over 4-tuples (global and every per-vertex count) for random
graphs and random core sizes, including cores that are empty on one side or cover a side.
The priority order is the oracle's (Def. Vertex Priority); the core of each
side is its top-priority prefix, as on the GPU."""
import itertools

import numpy as np
import pytest

import oracle as O
from synth import graphs as G


def f(a, d):
    """Lemma 2 and the unbalanced count a*d (reading R3)."""
    return a * (a - 1) // 2 + d * (d - 1) // 2, a * d


def decomposed(g, nc_u, nc_v):
    n_u, n_v = g.n_u, g.n_v
    n = n_u + n_v
    pos = O.priority_order(g).astype(np.int64)  # 0 = highest priority, global ids
    u, v, s = g.edges()
    adj = [dict() for _ in range(n)]
    for a, b, sg in zip(u.tolist(), v.tolist(), s.tolist()):
        adj[a][n_u + b] = 1 if sg else -1
        adj[n_u + b][a] = 1 if sg else -1
    # core = the top-priority prefix of each side (side-local ranks < nc)
    core = np.zeros(n, bool)
    for lo, hi, k in ((0, n_u, nc_u), (n_u, n, nc_v)):
        ids = sorted(range(lo, hi), key=lambda x: pos[x])
        core[ids[:k]] = True
    B = np.zeros(n, dtype=object)
    N = np.zeros(n, dtype=object)
    gB = gN = 0
    for x in range(n):  # route G start x; middles / ends of lower priority
        a_r, d_r, a_c, d_c = {}, {}, {}, {}
        mids = {}
        for m, sx in adj[x].items():
            if pos[m] <= pos[x]:
                continue
            for w, sw in adj[m].items():
                if pos[w] <= pos[x]:
                    continue
                cw = core[x] and core[m] and core[w]  # a core wedge: the engine skips it
                agree = sx == sw
                tgt = (a_c if agree else d_c) if cw else (a_r if agree else d_r)
                tgt[w] = tgt.get(w, 0) + 1
                mids.setdefault(w, []).append((m, agree, cw))
        for w in mids:
            ar, dr, ac, dc = a_r.get(w, 0), d_r.get(w, 0), a_c.get(w, 0), d_c.get(w, 0)
            # the engine: f of the partial (non-core-middle) counts, 4-role scatter from them
            eb, en = f(ar, dr)
            cb, cn = (ac * ar + dc * dr, ac * dr + ar * dc) if core[x] and core[w] else (0, 0)
            gB += eb + cb
            gN += en + cn
            for z in (x, w):
                B[z] += eb + cb
                N[z] += en + cn
            for m, agree, cw in mids[w]:
                if cw:  # core middle: only its mixed butterflies (other middle non-core)
                    B[m] += ar if agree else dr
                    N[m] += dr if agree else ar
                else:  # non-core middle: engine share from (a_r, d_r) plus the correction
                    B[m] += (ar - 1 if agree else dr - 1) + (ac if agree else dc)
                    N[m] += (dr if agree else ar) + (dc if agree else ac)
    # the dense core: every butterfly of G[C], all four roles (order-free, brute force here)
    cu = [x for x in range(n_u) if core[x]]
    cv = [y for y in range(n_u, n) if core[y]]
    for x, w in itertools.combinations(cu, 2):
        for y, z in itertools.combinations(cv, 2):
            e = [adj[x].get(y), adj[x].get(z), adj[w].get(y), adj[w].get(z)]
            if None in e:
                continue
            bal = e[0] * e[1] * e[2] * e[3] == 1
            gB += bal
            gN += not bal
            for t in (x, w, y, z):
                B[t] += bal
                N[t] += not bal
    return gB, gN, B, N


@pytest.mark.parametrize("seed", range(16))
def test_hybrid_identity_equals_brute_force(seed):
    rng = np.random.default_rng(900 + seed)
    n_u, n_v = int(rng.integers(4, 14)), int(rng.integers(4, 14))
    g = G.random_bipartite(n_u, n_v, float(rng.uniform(0.3, 0.9)), float(rng.uniform(0.0, 1.0)), seed=seed)
    br = O.brute(g)
    want_b = np.concatenate([br["bal_u"], br["bal_v"]]).astype(object)
    want_n = np.concatenate([br["unb_u"], br["unb_v"]]).astype(object)
    for nc_u, nc_v in [(0, 0), (int(rng.integers(1, n_u + 1)), int(rng.integers(1, n_v + 1))), (n_u, n_v),
                       (n_u, 0), (2, n_v)]:
        gB, gN, B, N = decomposed(g, nc_u, nc_v)
        assert (gB, gN) == (br["B"], br["N"]), (nc_u, nc_v)
        assert list(B) == list(want_b) and list(N) == list(want_n), (nc_u, nc_v)


def test_hybrid_identity_planted_core():
    """A small core-periphery graph (the hybrid workload's shape) with its planted core."""
    g = G.core_periphery(14, 12, 30, 2.2, 6.0, 6.0, 6, 5, 0.7, 0.6, 3)
    br = O.brute(g)
    gB, gN, B, N = decomposed(g, 6, 5)
    assert (gB, gN) == (br["B"], br["N"])
    assert list(B) == list(np.concatenate([br["bal_u"], br["bal_v"]]).astype(object))
    assert list(N) == list(np.concatenate([br["unb_u"], br["unb_v"]]).astype(object))
