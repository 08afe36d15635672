"""Pins of the CPU oracle to things other than itself (paper worked example, SPEC literal
examples, closed forms, textbook matrix identities, invariants, brute force).

A plausible mistake anywhere in oracle/bbf_oracle.c — a dropped C(d,2) term, a wrong sign
comparison, a missing w != u exclusion, a wrong priority tie-break, a lost start vertex in
the parallel split — fails at least one test here.  CPU only."""
import itertools
import os

import numpy as np
import pytest

import oracle as O
from synth import graphs as G

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def comb2(x):
    x = np.asarray(x, dtype=np.int64)  # entries are common-neighbour counts (< 2^31)
    return x * (x - 1) // 2


def gram(M):
    """M M^T exactly: float64 BLAS is exact for integer entries while sums stay < 2^53."""
    Mf = M.astype(np.float64)
    return np.rint(Mf @ Mf.T).astype(np.int64)


def matrix_identity(g):
    """Independent count from the textbook identity: with A the 0/1 adjacency,
    S the +1/-1/0 signed adjacency, T = A A^T, P = S S^T (numpy int64 matmul), a same-side
    pair has a = (T+P)/2 agreeing and d = (T-P)/2 disagreeing common neighbours, and
    B = sum_{u<w} C(a,2)+C(d,2), N = sum_{u<w} a*d."""
    S = g.dense_sign().astype(np.int64)
    A = (S != 0).astype(np.int64)
    T, P = gram(A), gram(S)
    iu = np.triu_indices(g.n_u, 1)
    t, p = T[iu], P[iu]
    assert np.all((t + p) % 2 == 0)
    a, d = (t + p) // 2, (t - p) // 2
    return int(np.sum(comb2(a) + comb2(d))), int(np.sum(a * d)), T


def load_fig1():
    rows = []
    for line in open(os.path.join(GOLDEN, "fig1_butterflies.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        s = list(map(int, f[2:6]))
        edges = [(0, 0, s[0]), (1, 0, s[1]), (0, 1, s[2]), (1, 1, s[3])]  # (u, v, sign)
        rows.append((f[0], f[1], edges, int(f[6]), int(f[7])))
    return rows


def load_spec():
    rows = []
    for line in open(os.path.join(GOLDEN, "spec_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, sizes, edges, want, cite = [x.strip() for x in line.split("|")]
        n_u, n_v = map(int, sizes.split())
        e = [tuple(map(int, t.split(":"))) for t in edges.split(",") if t]
        b, n = map(int, want.split())
        rows.append((name, n_u, n_v, e, b, n, cite))
    return rows


def graph_of(n_u, n_v, edges):
    if not edges:
        return G.from_edges(n_u, n_v, [], [], [])
    u, v, s = zip(*edges)
    return G.from_edges(n_u, n_v, u, v, s)


# ----------------------------------------------------------------------------- worked examples

@pytest.mark.parametrize("panel", load_fig1(), ids=lambda r: r[0])
def test_fig1_six_signed_butterflies(panel):
    name, caption, edges, want_b, want_n = panel
    g = graph_of(2, 2, edges)
    negatives = sum(1 for e in edges if e[2] == 0)
    assert (negatives % 2 == 0) == (want_b == 1)  # caption consistent with Def. Balanced
    br = O.brute(g)
    assert (br["B"], br["N"]) == (want_b, want_n)
    rg = O.route_g(g)
    assert (rg["B"], rg["N"]) == (want_b, want_n)
    bal, unb = O.route_s(g)
    assert list(bal) == [want_b] * 4 and list(unb) == [want_n] * 4


@pytest.mark.parametrize("ex", load_spec(), ids=lambda r: r[0])
def test_spec_literal_examples(ex):
    name, n_u, n_v, edges, want_b, want_n, cite = ex
    g = graph_of(n_u, n_v, edges)
    assert (O.brute(g)["B"], O.brute(g)["N"]) == (want_b, want_n), cite
    rg = O.route_g(g)
    assert (rg["B"], rg["N"]) == (want_b, want_n), cite
    bal, unb = O.route_s(g)
    assert int(bal.sum()) == 4 * want_b and int(unb.sum()) == 4 * want_n, cite


def test_priority_example_spec68():
    """degrees by global id {1:3, 2:3, 3:2} -> priority order 2 > 1 > 3
    (Def. Vertex Priority: degree, then larger id)."""
    # U = {0,1,2,3}, V = {4,5,6} in global ids; deg(1)=deg(2)=3, deg(3)=2, deg(0)=0
    g = graph_of(4, 3, [(1, 0, 1), (1, 1, 1), (1, 2, 1), (2, 0, 1), (2, 1, 1), (2, 2, 0),
                        (3, 0, 1), (3, 1, 0)])
    pos = O.priority_order(g)
    assert pos[2] < pos[1] < pos[3]
    # full order: deg 3 = {1,2,4,5} by id desc, then deg 2 = {3,6} by id desc, then 0
    assert list(np.argsort(pos)) == [5, 4, 2, 1, 6, 3, 0]


def test_priority_all_equal_degree_is_id_order():
    g = G.complete(3, 3)  # every degree 3 -> pure id tie-break
    pos = O.priority_order(g)
    assert list(np.argsort(pos)) == [5, 4, 3, 2, 1, 0]


# ----------------------------------------------------------------------------- closed forms

@pytest.mark.parametrize("m,n", [(2, 2), (3, 3), (4, 5), (6, 3), (1, 7), (7, 1)])
def test_complete_bipartite_closed_form(m, n):
    g = G.complete(m, n)
    c = lambda k: k * (k - 1) // 2
    br = O.brute(g, pairs=True)
    assert br["B"] == c(m) * c(n) and br["N"] == 0
    assert O.route_g(g)["B"] == c(m) * c(n)
    assert np.all(br["bal_u"] == (m - 1) * c(n)) and np.all(br["bal_v"] == (n - 1) * c(m))
    bal, unb = O.route_s(g)
    assert np.all(bal[:m] == (m - 1) * c(n)) and np.all(bal[m:] == (n - 1) * c(m))
    assert np.all(unb == 0)
    z, y, b, nn = O.pairs(g, 0)
    assert len(z) == (c(m) if c(n) else 0) and np.all(b == c(n))


def test_complete_bipartite_rank_one_signs_closed_form():
    """sign(u,v) = alpha_u * beta_v is switching-equivalent to all-positive:
    N = 0 and B = C(m,2) C(n,2)."""
    alpha = [1, -1, 1, -1]
    beta = [1, 1, -1, 1, -1]
    g = G.complete(4, 5, sign_fn=lambda u, v: 1 if alpha[u] * beta[v] > 0 else 0)
    for r in (O.brute(g), O.route_g(g)):
        assert (r["B"], r["N"]) == (6 * 10, 0)


# ----------------------------------------------------------------------------- SPEC corpus

def corpus(n_graphs=1000):
    rng = np.random.default_rng(600)
    p_edges = [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
    p_pos = [0.0, 0.25, 0.5, 0.75, 1.0]
    for i in range(n_graphs):
        n_u, n_v = int(rng.integers(1, 13)), int(rng.integers(1, 13))
        yield G.random_bipartite(n_u, n_v, p_edges[i % 9], p_pos[(i // 9) % 5], seed=i)


def test_corpus_brute_vs_routes_vs_matrix_identity():
    """oracle equivalence on a 1,000-graph corpus (|U|,|V| <= 12): brute force
    (definition) == Alg. 2 == vBBFC == Lemma-2 pairs == T/P matrix identity, per vertex too."""
    for g in corpus():
        br = O.brute(g, pairs=True)
        rg = O.route_g(g, threads=2)
        assert (rg["B"], rg["N"]) == (br["B"], br["N"]), g.name
        mb, mn, T = matrix_identity(g)
        assert (mb, mn) == (br["B"], br["N"]), g.name
        bal, unb = O.route_s(g, threads=2)
        assert np.array_equal(bal[:g.n_u], br["bal_u"]) and np.array_equal(unb[:g.n_u], br["unb_u"])
        assert np.array_equal(bal[g.n_u:], br["bal_v"]) and np.array_equal(unb[g.n_u:], br["unb_v"])
        # SPEC.md:313 / SURVEY P8: sum over all vertices = 4B; each side = 2B
        assert int(bal.sum()) == 4 * br["B"] and int(bal[:g.n_u].sum()) == 2 * br["B"]
        # per-pair Lemma 2 vs brute per-pair
        z, y, b, _ = O.pairs(g, 0)
        pm = np.zeros((g.n_u, g.n_u), np.uint64)
        pm[z, y] = b
        assert np.array_equal(pm, br["pairs_u"]), g.name
        # Lemma 2 decomposition summed: B + N = sum_{u<w} C(T_uw, 2)
        iu = np.triu_indices(g.n_u, 1)
        assert br["B"] + br["N"] == int(np.sum(comb2(T[iu])))


def test_route_g_wedge_count_matches_priority_definition():
    """W_G counts the wedges (u,v,w) with p(v)<p(u) and p(w)<p(u) (Alg. 2 lines 9-10):
    recount it with a plain Python loop over the oracle's priority positions."""
    for g in list(corpus(60)):
        pos = O.priority_order(g)  # 0 = highest priority
        u, v, s = g.edges()
        adj = {x: [] for x in range(g.n_u + g.n_v)}
        for a, b in zip(u, v):
            adj[int(a)].append(int(b) + g.n_u)
            adj[int(b) + g.n_u].append(int(a))
        W = 0
        for x in adj:
            for m in adj[x]:
                if pos[m] > pos[x]:
                    W += sum(1 for w in adj[m] if pos[w] > pos[x])
        assert O.route_g(g)["W_G"] == W


# ----------------------------------------------------------------------------- invariants

def switch(g, gid):
    u, v, s = g.edges()
    s = s.copy()
    if gid < g.n_u:
        s[u == gid] ^= 1
    else:
        s[v == gid - g.n_u] ^= 1
    return G.from_edges(g.n_u, g.n_v, u, v, s)


def negate(g):
    u, v, s = g.edges()
    return G.from_edges(g.n_u, g.n_v, u, v, s ^ 1)


@pytest.mark.parametrize("seed", range(6))
def test_switching_and_negation_invariance(seed):
    """SPEC.md:311-312 / SURVEY P5: a butterfly has 0 or 2 edges at any vertex, so flipping all
    signs at a vertex (or everywhere) keeps B, N, per-vertex and per-pair counts."""
    g = G.random_bipartite(30, 25, 0.3, 0.6, seed=100 + seed)
    base = O.route_g(g)
    bal, unb = O.route_s(g)
    pz = O.pairs(g, 0)
    rng = np.random.default_rng(seed)
    h = g
    for gid in rng.integers(0, g.n_u + g.n_v, size=5):
        h = switch(h, int(gid))
    for k in (h, negate(g)):
        r = O.route_g(k)
        assert (r["B"], r["N"]) == (base["B"], base["N"])
        b2, n2 = O.route_s(k)
        assert np.array_equal(b2, bal) and np.array_equal(n2, unb)
        q = O.pairs(k, 0)
        assert sorted(zip(*[a.tolist() for a in q])) == sorted(zip(*[a.tolist() for a in pz]))


def test_all_positive_and_rank_one_config2():
    """config 2 signs are per movie (sigma = beta_v), so N = 0 everywhere and
    B equals the unsigned count sum_{u<w} C(T_uw,2); all-positive graphs likewise."""
    g = G.config2()
    r = O.route_g(g)
    assert r["N"] == 0
    S = g.dense_sign().astype(np.int64)
    T = gram((S != 0).astype(np.int64))
    iu = np.triu_indices(g.n_u, 1)
    assert r["B"] == int(np.sum(comb2(T[iu])))
    bal, unb = O.route_s(g)
    assert not unb.any() and int(bal.sum()) == 4 * r["B"]


def test_config1_matrix_identity_and_routes():
    g = G.config1()
    mb, mn, _ = matrix_identity(g)
    br = O.brute(g)
    rg = O.route_g(g)
    assert (br["B"], br["N"]) == (mb, mn) == (rg["B"], rg["N"])
    bal, unb = O.route_s(g)
    assert np.array_equal(bal[:g.n_u], br["bal_u"]) and np.array_equal(unb[g.n_u:], br["unb_v"])
    # SURVEY P11 (statistical sanity, generator): balanced fraction ~ (1 + (2p-1)^4) / 2
    frac = mb / (mb + mn)
    assert abs(frac - (1 + 0.4 ** 4) / 2) < 0.05


@pytest.mark.parametrize("threads", [1, 2, 3, 4, 8])
def test_route_g_schedule_independent(threads):
    """identical counts for worker counts {1,2,3,4,8}."""
    g = G.random_bipartite(120, 90, 0.15, 0.5, seed=77)
    ref = O.route_g(g, threads=1)
    got = O.route_g(g, threads=threads)
    assert (got["B"], got["N"], got["W_G"]) == (ref["B"], ref["N"], ref["W_G"])


def test_route_g_start_partition_additive():
    """Any partition of the start vertices sums to the whole (PAPER.md:953 'each vertex u ...
    can be processed independently') — the property the multi-GPU split relies on."""
    g = G.random_bipartite(80, 70, 0.2, 0.7, seed=5)
    full = O.route_g(g)
    rng = np.random.default_rng(1)
    lab = rng.integers(0, 3, size=g.n_u + g.n_v)
    parts = [O.route_g(g, starts=np.nonzero(lab == k)[0]) for k in range(3)]
    for key in ("B", "N", "W_G"):
        assert sum(p[key] for p in parts) == full[key]


def test_topk_pairs_against_brute_pair_matrix():
    g = G.random_bipartite(40, 30, 0.35, 0.6, seed=9)
    br = O.brute(g, pairs=True)
    pm = br["pairs_u"]
    cand = [(int(pm[a, b]), a, b) for a in range(g.n_u) for b in range(a + 1, g.n_u) if pm[a, b] > 0]
    cand.sort(key=lambda t: (-t[0], t[1], t[2]))
    got = O.topk_pairs(g, 25, side=0)
    assert [(a, b, s) for a, b, s, _ in got] == [(a, b, s) for s, a, b in cand[:25]]


# ----------------------------------------------------------------------------- errors / edges

def test_errors_duplicate_range_sign():
    g = G.from_edges(2, 2, [0, 1], [0, 1], [1, 1])
    dup = G.SignedBipartite(2, 2, np.array([0, 2, 2], np.uint64), np.array([0, 0], np.uint32),
                            np.array([1, 0], np.uint8))
    with pytest.raises(O.OracleError) as e:
        O.route_g(dup)
    assert e.value.name == "EDUP"  # SPEC.md:60 (0,0,+),(0,0,-) -> DuplicateEdge
    bad = G.SignedBipartite(2, 2, g.row_ptr, np.array([0, 2], np.uint32), g.sign)
    with pytest.raises(O.OracleError) as e:
        O.brute(bad)
    assert e.value.name == "ERANGE"
    badsign = G.SignedBipartite(2, 2, g.row_ptr, g.col, np.array([1, 2], np.uint8))
    with pytest.raises(O.OracleError) as e:
        O.route_s(badsign)
    assert e.value.name == "EINVAL"


def test_isolated_vertices_zero():
    g = G.from_edges(5, 4, [0, 0, 1, 1], [0, 1, 0, 1], [1, 1, 1, 0])
    bal, unb = O.route_s(g)
    assert list(bal) == [0, 0, 0, 0, 0, 0, 0, 0, 0] and list(unb) == [1, 1, 0, 0, 0, 1, 1, 0, 0]


@pytest.mark.parametrize("seed", range(4))
def test_bb_base_alg1_against_brute_and_fig1(seed):
    """Alg. 1 BB-Base (explicit balance check of every pair in H(w)) equals the brute-force
    4-cycle classification (Def. Balanced butterfly) on random tiny graphs, visits exactly the
    priority-eligible wedges of Alg. 2, and counts each panel of Fig. 1 as the paper labels it."""
    rng = np.random.default_rng(900 + seed)
    for i in range(60):
        g = G.random_bipartite(int(rng.integers(1, 10)), int(rng.integers(1, 10)),
                               float(rng.uniform(0.1, 0.9)), float(rng.uniform(0.0, 1.0)),
                               seed=1000 * seed + i)
        b, r = O.bb_base(g, threads=1 + i % 3), O.brute(g)
        assert (b["B"], b["N"]) == (r["B"], r["N"])
        assert b["W_G"] == O.route_g(g)["W_G"]
    # one butterfly, every sign pattern: balanced iff an even number of negative edges
    for signs in itertools.product([0, 1], repeat=4):
        g = G.from_edges(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], list(signs))
        b = O.bb_base(g)
        neg = 4 - sum(signs)
        assert (b["B"], b["N"]) == ((1, 0) if neg % 2 == 0 else (0, 1))


def test_bb_base_vs_bucket_regime_desk_scale():
    """The paper's speedup regime: on a Senate-shaped graph (few dense
    left vertices, many right ones; 10 x 1000, density 0.5) BB-Bucket's counting loop is
    faster than BB-Base's (the paper reports > 100x on Senate/House; the bar here is only
    'not slower', measured single-threaded) and both give the same counts."""
    g = G.random_bipartite(10, 1000, 0.5, 0.5, seed=7)
    b = min((O.bb_base(g, threads=1) for _ in range(3)), key=lambda r: r["count_s"])
    r = min((O.route_g(g, threads=1) for _ in range(3)), key=lambda r: r["count_s"])
    assert (b["B"], b["N"], b["W_G"]) == (r["B"], r["N"], r["W_G"])
    assert b["count_s"] > r["count_s"]


# ----------------------------------------------------------------------------- 4-role scatter

def test_route_g_pv_corpus_against_brute_force():
    """oracle_route_g_pv (Alg. 2 + the 4-role scatter) equals the brute-force
    4-tuple classification per vertex of both sides, on the SPEC-style corpus.
    A swapped middle share ((a, d-1) for (a-1, d)), a missing end share or a start share sent to
    the wrong vertex changes some vertex of some graph here."""
    for g in corpus(1000):
        br = O.brute(g)
        pv = O.route_g_pv(g, threads=1 + g.n_u % 3)
        assert (pv["B"], pv["N"]) == (br["B"], br["N"]), g.name
        for k in ("bal_u", "unb_u", "bal_v", "unb_v"):
            assert np.array_equal(pv[k], br[k]), (g.name, k)
        assert pv["W_G"] == O.route_g(g)["W_G"]


@pytest.mark.parametrize("m,n", [(2, 2), (3, 5), (9, 4), (1, 6)])
def test_route_g_pv_complete_closed_form(m, n):
    """K_{m,n}, all positive: every U vertex is in (m-1) C(n,2) butterflies, every V
    vertex in (n-1) C(m,2), all balanced."""
    g = G.complete(m, n)
    c = lambda k: k * (k - 1) // 2
    pv = O.route_g_pv(g)
    assert np.all(pv["bal_u"] == (m - 1) * c(n)) and np.all(pv["bal_v"] == (n - 1) * c(m))
    assert not pv["unb_u"].any() and not pv["unb_v"].any()


@pytest.mark.parametrize("seed", range(3))
def test_route_g_pv_against_vbbfc_medium(seed):
    """On graphs too large for brute force, the route-G per-vertex arrays equal the definition
    path vBBFC vertex by vertex, and each side sums to 2B."""
    g = G.random_bipartite(300, 200, 0.04 + 0.03 * seed, 0.3 + 0.3 * seed, seed=4242 + seed)
    pv = O.route_g_pv(g, threads=4)
    bal, unb = O.route_s(g, threads=4)
    assert np.array_equal(np.concatenate([pv["bal_u"], pv["bal_v"]]), bal)
    assert np.array_equal(np.concatenate([pv["unb_u"], pv["unb_v"]]), unb)
    assert int(pv["bal_u"].sum()) == 2 * pv["B"] == int(pv["bal_v"].sum())
    assert int(pv["unb_v"].sum()) == 2 * pv["N"]


def test_route_g_pv_switching_invariant_and_powerlaw():
    """A skewed Chung-Lu graph (hub starts with many ends): route-G per-vertex == vBBFC, and
    switching the signs at a hub leaves every per-vertex count unchanged."""
    key, rng = G.chung_lu(3000, 800, 20000, 2.0, 400.0, 400.0, seed=31)
    s = rng.random(key.size) < 0.6
    g = G._from_sorted_keys(3000, 800, key, s, "cl")
    pv = O.route_g_pv(g, threads=3)
    bal, unb = O.route_s(g, threads=8)
    assert np.array_equal(np.concatenate([pv["bal_u"], pv["bal_v"]]), bal)
    assert np.array_equal(np.concatenate([pv["unb_u"], pv["unb_v"]]), unb)
    hub = int(np.argmax(np.diff(g.row_ptr.astype(np.int64))))
    h = switch(g, hub)
    q = O.route_g_pv(h, threads=2)
    for k in ("bal_u", "unb_u", "bal_v", "unb_v"):
        assert np.array_equal(q[k], pv[k])


def test_route_g_pv_start_partition_additive():
    """Per-vertex counts of disjoint start sets sum to the whole (the property the
    reference arm's start slices and the multi-GPU split rely on)."""
    g = G.random_bipartite(90, 60, 0.25, 0.6, seed=12)
    full = O.route_g_pv(g)
    lab = np.random.default_rng(2).integers(0, 4, size=g.n_u + g.n_v)
    parts = [O.route_g_pv(g, starts=np.nonzero(lab == k)[0], threads=2) for k in range(4)]
    with O.Prepared(g) as h:  # the prepared-graph form used by bench.py's reference arm
        parts2 = [h.route_g_pv(starts=np.nonzero(lab == k)[0], threads=3) for k in range(4)]
    for p, q in zip(parts, parts2):
        assert (p["B"], p["N"], p["W_G"]) == (q["B"], q["N"], q["W_G"])
        assert np.array_equal(p["bal_v"], q["bal_v"]) and np.array_equal(p["unb_u"], q["unb_u"])
    for key in ("B", "N", "W_G"):
        assert sum(p[key] for p in parts) == full[key]
    for key in ("bal_u", "unb_u", "bal_v", "unb_v"):
        assert np.array_equal(sum(p[key] for p in parts), full[key])


# ----------------------------------------------------------------------------- per-edge counts

def test_edge_counts_corpus_against_brute_force():
    """oracle_edge (the definition, edge by edge) equals brute force (every
    butterfly adds one to each of its 4 edges) on the corpus; per-edge sums are 4B / 4N, and the
    edges at a vertex sum to twice its per-vertex count (each butterfly containing z has exactly
    two edges at z)."""
    for g in corpus(400):
        bb, bn = O.edge_brute(g)
        eb, en = O.edge_counts(g, threads=1 + g.n_v % 3)
        assert np.array_equal(bb, eb) and np.array_equal(bn, en), g.name
        br = O.brute(g)
        assert int(eb.sum()) == 4 * br["B"] and int(en.sum()) == 4 * br["N"]
        u = np.repeat(np.arange(g.n_u), np.diff(g.row_ptr.astype(np.int64)))
        assert np.array_equal(np.bincount(u, weights=eb.astype(np.float64), minlength=g.n_u).astype(np.int64),
                              2 * br["bal_u"].astype(np.int64))
        assert np.array_equal(np.bincount(g.col.astype(np.int64), weights=en.astype(np.float64),
                                          minlength=g.n_v).astype(np.int64), 2 * br["unb_v"].astype(np.int64))


@pytest.mark.parametrize("m,n", [(2, 2), (4, 5), (7, 3)])
def test_edge_counts_complete_closed_form(m, n):
    """K_{m,n} all positive: every edge lies in (m-1)(n-1) butterflies, all balanced."""
    eb, en = O.edge_counts(G.complete(m, n))
    assert np.all(eb == (m - 1) * (n - 1)) and not en.any()


def test_edge_counts_medium_switching_invariant():
    """On a graph beyond brute force: switching a vertex's signs leaves every edge count unchanged
    (a butterfly has 0 or 2 edges at the vertex), and the vertex relation holds."""
    g = G.random_bipartite(150, 120, 0.08, 0.6, seed=77)
    eb, en = O.edge_counts(g, threads=4)
    h = switch(g, 7)
    hb, hn = O.edge_counts(h, threads=4)
    assert np.array_equal(eb, hb) and np.array_equal(en, hn)
    pv = O.route_g_pv(g)
    u = np.repeat(np.arange(g.n_u), np.diff(g.row_ptr.astype(np.int64)))
    assert np.array_equal(np.bincount(u, weights=en.astype(np.float64), minlength=g.n_u).astype(np.int64),
                          2 * pv["unb_u"].astype(np.int64))
