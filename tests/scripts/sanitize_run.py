"""Small end-to-end driver for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
family of libbbf.so on tiny graphs, each result checked against the oracle.
  compute-sanitizer --tool memcheck --error-exitcode 9 python tests/scripts/sanitize_run.py
Covers: build (hashed and shared-memory histograms), plan, the T1 / T2 / T3 tiers (T2_MAX lowered so
hubs take the hub kernel), a hub with a large end side, both counter encodings, top-k pairs and vertices,
the positive-only mask, the dense FP4 (one and two accumulators), int8 pair and 1-CTA kernels, the
FP4-only operand build followed by the int8 kernels on demand, and the sampling estimator."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import oracle as O  # noqa: E402  (test infrastructure: this script is a checker)
from synth import graphs as G  # noqa: E402


def hub_graph(n_v=2000, deg_u0=2000, fan=2, seed=7):
    """U vertex 0 adjacent to every V vertex; n_v * 150 / fan other U vertices with `fan` random
    V neighbours each: the hub (highest priority) has ~150K ends behind 2,000 middles."""
    rng = np.random.default_rng(seed)
    n_other = n_v * 150 // fan
    n_u = 1 + n_other
    us = [np.zeros(deg_u0, np.int64)]
    vs = [np.arange(deg_u0) % n_v]
    for k in range(fan):
        us.append(np.arange(1, n_u))
        vs.append((np.arange(1, n_u) * (k + 1) * 7919 + rng.integers(0, n_v, n_u - 1)) % n_v)
    u = np.concatenate(us)
    v = np.concatenate(vs)
    key = np.unique(u * n_v + v)
    s = rng.random(key.size) < 0.5
    return G.from_edges(n_u, n_v, (key // n_v).tolist(), (key % n_v).tolist(), s.astype(np.uint8).tolist())


def check_sparse(B, g, name, flags=0):
    with B.Graph.from_synth(g, flags=flags) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
    rg = O.route_g(g, threads=os.cpu_count() or 8)
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], rg["N"], rg["W_G"]), name
    bal, unb = O.route_s(g, threads=os.cpu_count() or 8)
    assert np.array_equal(bu, bal[:g.n_u]) and np.array_equal(nu, unb[:g.n_u]), name
    assert np.array_equal(bv, bal[g.n_u:]) and np.array_equal(nv, unb[g.n_u:]), name
    print("ok", name, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="skip the multi-window hub graph (racecheck)")
    a = ap.parse_args()
    import torch
    assert torch.cuda.is_available()
    from paper_2308_07932_b200 import bbf as B

    check_sparse(B, G.config1(), "config1")
    check_sparse(B, G.config2(), "config2")
    check_sparse(B, G.random_bipartite(300, 700, 0.3, 0.5, seed=1), "random 300x700 (T2)")
    os.environ["BBF_T2_MAX"] = "512"
    check_sparse(B, G.random_bipartite(300, 700, 0.3, 0.5, seed=1), "random 300x700 (T3)", B.BBF_FORCE_SPARSE)
    if not a.quick:
        check_sparse(B, hub_graph(), "hub graph (T3, 150K ends)", B.BBF_FORCE_SPARSE)
    os.environ["BBF_NO_COMPACT"] = "1"
    check_sparse(B, G.random_bipartite(200, 500, 0.3, 0.5, seed=2), "general counter encoding", B.BBF_FORCE_SPARSE)
    del os.environ["BBF_NO_COMPACT"]
    del os.environ["BBF_T2_MAX"]

    g = G.config2()
    th = os.cpu_count() or 8
    with B.Graph.from_synth(g) as h:
        assert h.count_pairs_topk(20, side=0) == O.topk_pairs(g, 20, side=0, threads=th)
        assert h.topk_vertices(10, side=1, metric=B.BBF_METRIC_BALANCED) == O.topk_vertices(g, 10, 1, "balanced", threads=th)
    print("ok top-k pairs / vertices", flush=True)
    gp = G.random_bipartite(250, 400, 0.3, 0.5, seed=3)
    with B.Graph.from_synth(gp, flags=B.BBF_POSITIVE_ONLY) as h:
        c = h.count_global()
    rg = O.route_g(O.positive_subgraph(gp), threads=th)
    assert (c["balanced"], c["unbalanced"]) == (rg["B"], rg["N"])
    print("ok positive-only", flush=True)

    gd = G.random_bipartite(517, 391, 0.4, 0.6, seed=11)
    bal, unb = O.route_s(gd, threads=os.cpu_count() or 8)
    for env in (None, "BBF_DENSE_F4_TP", "BBF_DENSE_I8", "BBF_DENSE_1CTA"):
        if env:
            os.environ[env] = "1"
        with B.Graph.from_synth(gd, flags=B.BBF_FORCE_DENSE) as h:
            tot, bu, nu, bv, nv = h.count_per_vertex()
        if env:
            del os.environ[env]
        assert np.array_equal(bu, bal[:gd.n_u]) and np.array_equal(nv, unb[gd.n_u:]), env
        print("ok dense", env or "fp4 (one accumulator)", flush=True)
    with B.Graph.from_synth(gd, flags=B.BBF_FORCE_DENSE) as h:
        h.count_per_vertex()
        os.environ["BBF_DENSE_I8"] = "1"
        tot, bu, nu, bv, nv = h.count_per_vertex()
        del os.environ["BBF_DENSE_I8"]
    assert np.array_equal(bu, bal[:gd.n_u]) and np.array_equal(nv, unb[gd.n_u:])
    print("ok dense fp4-only operands then int8", flush=True)

    ge = G.config2()
    est = B.estimate_global(ge.n_u, ge.n_v, ge.row_ptr, ge.col, ge.sign, rho=0.5, trials=4, seed=1)
    ref = O.estimate(ge, 0.5, 4, seed=1, threads=th)
    assert [int(x) for x in est["sampled_B"]] == ref["sampled_B"], (est, ref)
    assert [int(x) for x in est["sampled_N"]] == ref["sampled_N"]
    print("ok estimator", flush=True)
    torch.cuda.synchronize()
    print("SANITIZE_RUN_DONE")


if __name__ == "__main__":
    main()
