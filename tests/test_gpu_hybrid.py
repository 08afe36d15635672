"""GPU parity of the NEXT-3 hybrid path (hybrid.cu): dense core on the tensor
cores + sparse remainder on the wedge engine + the mixed core pairs merged per pair before f.
Every count must equal the oracle's (Alg. 2 + 4-role scatter, vBBFC) element by element, for
forced core sizes (BBF_HYBRID_CORE=nu,nv) from the degenerate 2 x 2 to cores covering the
whole graph, and for the automatic dispatch on the hybrid workload."""
import os

import numpy as np
import pytest

import oracle as O
from synth import graphs as G

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def bbf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_07932_b200 import build
    build.build()
    from paper_2308_07932_b200 import bbf as B
    return B


def run(B, g, core=None, monkeypatch=None, flags=0):
    if core is not None:
        monkeypatch.setenv("BBF_HYBRID_CORE", f"{core[0]},{core[1]}")
    try:
        with B.Graph.from_synth(g, flags=flags) as h:
            c = h.count_global()
            tot, bu, nu, bv, nv = h.count_per_vertex()
            du = np.diff(g.row_ptr.astype(np.int64))
            dv = np.bincount(g.col, minlength=g.n_v)
            if core is not None and (du >= 2).sum() >= 2 and (dv >= 2).sum() >= 2:
                assert h.hybrid_core() != (0, 0)
    finally:
        if core is not None:
            monkeypatch.delenv("BBF_HYBRID_CORE")
    return c, tot, bu, nu, bv, nv


def check(B, g, want, core, monkeypatch):
    c, tot, bu, nu, bv, nv = run(B, g, core, monkeypatch)
    tag = f"{g.name} core={core}"
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (want["B"], want["N"], want["W_G"]), tag
    assert (tot["balanced"], tot["unbalanced"]) == (want["B"], want["N"]), tag
    assert np.array_equal(bu, want["bal_u"]) and np.array_equal(nu, want["unb_u"]), tag
    assert np.array_equal(bv, want["bal_v"]) and np.array_equal(nv, want["unb_v"]), tag


def small_cp(seed):
    rng = np.random.default_rng(7000 + seed)
    n_u, n_v = int(rng.integers(300, 3000)), int(rng.integers(200, 2000))
    m = int(rng.integers(2000, 20000))
    cu, cv = int(rng.integers(2, 300)), int(rng.integers(2, 300))
    return G.core_periphery(n_u, n_v, m, float(rng.uniform(2.0, 2.6)), n_v / 4.0, n_u / 4.0, min(cu, n_u),
                            min(cv, n_v), float(rng.uniform(0.05, 0.6)), float(rng.uniform(0.0, 1.0)), seed)


@pytest.mark.parametrize("seed", range(12))
def test_hybrid_small_forced_cores(bbf, monkeypatch, seed):
    """Core-periphery and uniform random graphs, several forced core sizes per graph (2 x 2,
    asymmetric, about the planted core, larger than a side): full per-vertex arrays and global
    counts equal the oracle's."""
    g = small_cp(seed) if seed % 4 else G.random_bipartite(int(40 + 37 * seed), int(30 + 29 * seed), 0.2, 0.6, seed)
    rg = O.route_g_pv(g, threads=THREADS)
    bal, unb = O.route_s(g, threads=THREADS)  # vBBFC: the definition path, checks the oracle's scatter too
    assert np.array_equal(bal[:g.n_u], rg["bal_u"]) and np.array_equal(unb[g.n_u:], rg["unb_v"])
    rng = np.random.default_rng(seed)
    cores = [(2, 2), (int(rng.integers(2, 64)), int(rng.integers(2, 64))), (256, 256), (100000, 100000),
             (int(rng.integers(2, 1200)), 2)]
    for core in cores:
        check(bbf, g, rg, core, monkeypatch)
    for hook in ("BBF_HYBRID_BITS", "BBF_HYBRID_GEMM"):  # the bitmap / library-GEMM forms
        monkeypatch.setenv(hook, "1")
        check(bbf, g, rg, cores[1], monkeypatch)
        monkeypatch.delenv(hook)


def test_hybrid_complete_bipartite(bbf, monkeypatch):
    """K_{m,n} with a core of part of each side: every pair is mixed or inside the core."""
    for m, n, core in [(40, 30, (10, 7)), (300, 200, (256, 64)), (50, 600, (3, 512))]:
        g = G.complete(m, n)
        check(bbf, g, O.route_g_pv(g, threads=THREADS), core, monkeypatch)


def test_hybrid_tiers_and_encodings(bbf, monkeypatch):
    """A medium core-periphery graph whose remainder uses all three engine tiers: forced cores of
    1,024 / 2,048, with the T2 tier off (hub kernel only), with the wide counter encoding, and
    with the mixed pairs on the bitmap kernel, and with the library-GEMM form instead of the
    fused FP4 cross-term kernel."""
    g = G.core_periphery(60_000, 20_000, 400_000, 2.1, 4000.0, 4000.0, 2048, 2048, 0.15, 0.7, 61)
    rg = O.route_g_pv(g, threads=THREADS)
    for core in [(1024, 1024), (2048, 2048), (2048, 512)]:
        check(bbf, g, rg, core, monkeypatch)
    for env in ("BBF_T2_MAX=0", "BBF_NO_COMPACT=1", "BBF_NO_PACKED_END=1", "BBF_HYBRID_BITS=1", "BBF_HYBRID_GEMM=1"):
        k, v = env.split("=")
        monkeypatch.setenv(k, v)
        check(bbf, g, rg, (2048, 2048), monkeypatch)
        monkeypatch.delenv(k)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("form", ["fused", "BBF_HYBRID_GEMM", "BBF_HYBRID_BITS"])
def test_hybrid_fake_world_shards_sum(bbf, monkeypatch, world, form):
    """Rank shards of the hybrid count (engine items, dense tiles, mixed middles y mod N) sum to
    the single-GPU result."""
    g = G.core_periphery(30_000, 10_000, 200_000, 2.2, 2000.0, 2000.0, 1024, 1024, 0.2, 0.6, 62)
    rg = O.route_g_pv(g, threads=THREADS)
    monkeypatch.setenv("BBF_HYBRID_CORE", "1024,1024")
    if form != "fused":
        monkeypatch.setenv(form, "1")
    acc = None
    for r in range(world):
        monkeypatch.setenv("BBF_FAKE_WORLD", f"{r}/{world}")
        with bbf.Graph.from_synth(g) as h:
            part = h.count_per_vertex()
        vals = [part[0]["balanced"], part[0]["unbalanced"]] + [a.astype(object) for a in part[1:]]
        acc = vals if acc is None else [x + y for x, y in zip(acc, vals)]
    monkeypatch.delenv("BBF_FAKE_WORLD")
    monkeypatch.delenv("BBF_HYBRID_CORE")
    if form != "fused":
        monkeypatch.delenv(form)
    assert (acc[0], acc[1]) == (rg["B"], rg["N"])
    for a, b in zip(acc[2:], (rg["bal_u"], rg["unb_u"], rg["bal_v"], rg["unb_v"])):
        assert np.array_equal(a.astype(np.uint64), b)


def test_hybrid_workload_full_size(bbf):
    """The hybrid workload (config 3 + an 8,192 x 8,192 core at density 0.1, ~16.5M edges):
    the automatic dispatch takes the hybrid path, and the global counts and both sides' entire
    per-vertex arrays equal the oracle's Alg. 2 + 4-role scatter."""
    g = G.config_hybrid()
    rg = O.route_g_pv(g, threads=THREADS)
    with bbf.Graph.from_synth(g) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
        core = h.hybrid_core()
    assert core[0] >= 1024 and core[1] >= 1024, core  # the dispatch found the planted core
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], rg["N"], rg["W_G"])
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"])
    assert np.array_equal(bu, rg["bal_u"]) and np.array_equal(nu, rg["unb_u"])
    assert np.array_equal(bv, rg["bal_v"]) and np.array_equal(nv, rg["unb_v"])


def test_hybrid_second_workload_auto(bbf):
    """Another closed core at a different size, density and sign mix (a 4,096 x 3,072 community at
    density 0.35 in a 400K x 150K periphery, signs p = 0.5): the automatic dispatch takes a core
    and the full per-vertex arrays equal the oracle's."""
    g = G.core_periphery(400_000, 150_000, 2_000_000, 2.3, 600.0, 600.0, 4096, 3072, 0.35, 0.5, 63,
                         core_random=True)
    rg = O.route_g_pv(g, threads=THREADS)
    with bbf.Graph.from_synth(g) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
        core = h.hybrid_core()
    assert core != (0, 0)
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], rg["N"], rg["W_G"])
    assert np.array_equal(bu, rg["bal_u"]) and np.array_equal(nu, rg["unb_u"])
    assert np.array_equal(bv, rg["bal_v"]) and np.array_equal(nv, rg["unb_v"])


def test_hybrid_dense_core_beyond_packed_accumulator(bbf, monkeypatch):
    """A core whose inside degrees exceed 2,047 (a 3,072 x 3,072 community at p = 0.8): the dense
    core runs on the two-accumulator FP4 kernel and the mixed pairs on the library-GEMM form (the
    fused kernel's packed accumulator would not be exact); counts equal the oracle's."""
    g = G.core_periphery(60_000, 30_000, 300_000, 2.2, 1500.0, 1500.0, 3072, 3072, 0.8, 0.6, 64, core_random=True)
    rg = O.route_g_pv(g, threads=THREADS)
    check(bbf, g, rg, (3072, 3072), monkeypatch)
    with bbf.Graph.from_synth(g) as h:  # the automatic dispatch on the same graph
        tot, bu, nu, bv, nv = h.count_per_vertex()
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"])
    assert np.array_equal(bu, rg["bal_u"]) and np.array_equal(nv, rg["unb_v"])


def test_hybrid_single_rank_nccl_communicator(bbf, monkeypatch):
    """The hybrid path under a real one-rank NCCL communicator (the per-vertex all-reduce over the
    degree >= 2 row prefixes, the status max-reduce): counts equal the oracle's."""
    g = G.core_periphery(30_000, 10_000, 200_000, 2.2, 2000.0, 2000.0, 1024, 1024, 0.2, 0.6, 62)
    rg = O.route_g_pv(g, threads=THREADS)
    monkeypatch.setenv("BBF_HYBRID_CORE", "1024,1024")
    comm = bbf.Comm(bbf.nccl_unique_id(), 1, 0, 0)
    try:
        with bbf.Graph.from_synth(g, comm=comm) as h:
            tot, bu, nu, bv, nv = h.count_per_vertex()
            assert h.hybrid_core() == (1024, 1024)
    finally:
        comm.free()
        monkeypatch.delenv("BBF_HYBRID_CORE")
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"])
    assert np.array_equal(bu, rg["bal_u"]) and np.array_equal(nu, rg["unb_u"])
    assert np.array_equal(bv, rg["bal_v"]) and np.array_equal(nv, rg["unb_v"])
