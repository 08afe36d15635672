"""GPU parity: libbbf.so (through the C ABI) vs the CPU oracle, element by element, on the same
seeded inputs.  Integer results must be bit-exact."""
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


def gpu_all(B, g, flags=0):
    with B.Graph.from_synth(g) as h:
        glob = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex(flags=flags)
    return glob, tot, bu, nu, bv, nv


def check_full(B, g, flags=0):
    glob, tot, bu, nu, bv, nv = gpu_all(B, g, flags)
    rg = O.route_g(g, threads=THREADS)
    assert (glob["balanced"], glob["unbalanced"]) == (rg["B"], rg["N"]), g.name
    assert glob["wedges_G"] == rg["W_G"], g.name
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"])
    bal, unb = O.route_s(g, threads=THREADS)
    assert np.array_equal(bu, bal[:g.n_u]), g.name
    assert np.array_equal(nu, unb[:g.n_u]), g.name
    assert np.array_equal(bv, bal[g.n_u:]), g.name
    assert np.array_equal(nv, unb[g.n_u:]), g.name


def test_config1_global_and_per_vertex(bbf):
    g = G.config1()
    check_full(bbf, g)
    br = O.brute(g)
    with bbf.Graph.from_synth(g) as h:
        c = h.count_global()
    assert (c["balanced"], c["unbalanced"]) == (br["B"], br["N"])


def test_config2_per_vertex_and_topk(bbf):
    g = G.config2()
    check_full(bbf, g)
    with bbf.Graph.from_synth(g) as h:
        for side in (0, 1):
            got = h.count_pairs_topk(100, side=side)
            want = O.topk_pairs(g, 100, side=side, threads=THREADS)
            assert got == want, side
        assert h.count_per_vertex()[0]["unbalanced"] == 0  # signs per movie: N = 0


def test_spec_corpus_subset(bbf):
    rng = np.random.default_rng(600)
    pe = [0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
    pp = [0.0, 0.25, 0.5, 0.75, 1.0]
    for i in range(300):
        n_u, n_v = int(rng.integers(1, 13)), int(rng.integers(1, 13))
        g = G.random_bipartite(n_u, n_v, pe[i % 9], pp[(i // 9) % 5], seed=i)
        check_full(bbf, g)


@pytest.mark.parametrize("m,n", [(2, 2), (3, 3), (40, 30), (300, 200), (700, 600)])
def test_complete_bipartite_closed_form(bbf, m, n):
    g = G.complete(m, n)
    c = lambda k: k * (k - 1) // 2
    glob, tot, bu, nu, bv, nv = gpu_all(bbf, g)
    assert glob["balanced"] == c(m) * c(n) and glob["unbalanced"] == 0
    assert np.all(bu == (m - 1) * c(n)) and np.all(bv == (n - 1) * c(m))
    assert not nu.any() and not nv.any()


def test_edge_cases(bbf):
    # empty graph, isolated vertices, a single butterfly, a star
    for g, want in [
        (G.from_edges(1, 1, [], [], []), (0, 0)),
        (G.from_edges(5, 4, [0, 0, 1, 1], [0, 1, 0, 1], [1, 1, 1, 0]), (0, 1)),
        (G.from_edges(1, 6, [0] * 6, list(range(6)), [1, 0, 1, 1, 0, 1]), (0, 0)),
        (G.from_edges(3, 3, [0, 0, 1, 1], [0, 1, 0, 1], [0, 0, 0, 0]), (1, 0)),
    ]:
        check_full(bbf, g)
        with bbf.Graph.from_synth(g) as h:
            c = h.count_global()
        assert (c["balanced"], c["unbalanced"]) == want


def test_errors(bbf):
    dup = G.SignedBipartite(2, 2, np.array([0, 2, 2], np.uint64), np.array([0, 0], np.uint32),
                            np.array([1, 0], np.uint8))
    with pytest.raises(bbf.BBFError) as e:
        bbf.Graph.from_synth(dup)
    assert e.value.name == "BBF_EDUP"
    rng_bad = G.SignedBipartite(2, 2, np.array([0, 1, 2], np.uint64), np.array([0, 2], np.uint32),
                                np.array([1, 1], np.uint8))
    with pytest.raises(bbf.BBFError) as e:
        bbf.Graph.from_synth(rng_bad)
    assert e.value.name == "BBF_ERANGE"
    sgn_bad = G.SignedBipartite(2, 2, np.array([0, 1, 2], np.uint64), np.array([0, 1], np.uint32),
                                np.array([1, 3], np.uint8))
    with pytest.raises(bbf.BBFError) as e:
        bbf.Graph.from_synth(sgn_bad)
    assert e.value.name == "BBF_EINVAL"
    mono_bad = G.SignedBipartite(2, 2, np.array([0, 2, 1], np.uint64), np.array([0, 1], np.uint32),
                                 np.array([1, 1], np.uint8))
    with pytest.raises(bbf.BBFError) as e:
        bbf.Graph.from_synth(mono_bad)
    assert e.value.name == "BBF_ERANGE"
    with bbf.Graph.from_synth(G.config1()) as h:
        with pytest.raises(bbf.BBFError):
            h.count_pairs_topk(0)


def zoned_graph(seed=11):
    """Degrees spanning every counter zone (deg > 65535 down to 2) on the U side, enough
    degree-2/3 ends to need several 48K-word windows, and hub starts split into units."""
    rng = np.random.default_rng(seed)
    n_v = 80_000
    degs = [70_000] * 2 + [300] * 40 + [40] * 1500 + [6] * 20_000 + [2] * 450_000 + [3] * 60_000 + [1] * 5000
    n_u = len(degs)
    w = 1.0 / np.arange(1, n_v + 1) ** 0.6
    cdf = np.cumsum(w) / w.sum()
    degs = np.array(degs)
    big = np.nonzero(degs >= 1000)[0]
    us = [np.full(degs[b], b) for b in big]
    vs = [rng.choice(n_v, size=degs[b], replace=False) for b in big]
    small = np.nonzero(degs < 1000)[0]
    su = np.repeat(small, degs[small])
    sv = np.searchsorted(cdf, rng.random(su.size), side="right").clip(0, n_v - 1)
    key = np.unique(su.astype(np.int64) * n_v + sv)  # duplicates dropped: degrees <= target
    us.append(key // n_v)
    vs.append(key % n_v)
    u = np.concatenate(us)
    v = np.concatenate(vs)
    s = (rng.random(u.size) < 0.6).astype(np.uint8)
    return G.from_edges(n_u, n_v, u, v, s, name="zoned")


def test_zoned_windows_global_and_sampled_vertices(bbf):
    g = zoned_graph()
    rg = O.route_g(g, threads=THREADS)
    with bbf.Graph.from_synth(g) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], rg["N"], rg["W_G"])
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"])
    # per-vertex: sum identities at any size + sampled vBBFC vertices
    assert int(bu.sum()) == 2 * rg["B"] and int(bv.sum()) == 2 * rg["B"]
    assert int(nu.sum()) == 2 * rg["N"] and int(nv.sum()) == 2 * rg["N"]
    rng = np.random.default_rng(0)
    su = np.unique(np.concatenate([np.arange(0, 50), rng.integers(0, g.n_u, 400)]))
    sv = np.unique(rng.integers(0, g.n_v, 60))
    bal, unb = O.route_s(g, verts=np.concatenate([su, g.n_u + sv]), threads=THREADS)
    assert np.array_equal(bu[su], bal[:su.size]) and np.array_equal(nu[su], unb[:su.size])
    assert np.array_equal(bv[sv], bal[su.size:]) and np.array_equal(nv[sv], unb[su.size:])


def test_config3_full_size(bbf):
    g = G.config3()
    rg = O.route_g(g, threads=THREADS)
    with bbf.Graph.from_synth(g) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
        c2 = h.count_global()
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], rg["N"], rg["W_G"])
    assert c2["balanced"] == c["balanced"] and c2["unbalanced"] == c["unbalanced"]  # deterministic
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"])
    assert int(bu.sum()) == 2 * rg["B"] and int(bv.sum()) == 2 * rg["B"]
    assert int(nu.sum()) == 2 * rg["N"] and int(nv.sum()) == 2 * rg["N"]
    rng = np.random.default_rng(3)
    deg_u = np.diff(g.row_ptr.astype(np.int64))
    top = np.argsort(-deg_u)[:20]
    su = np.unique(np.concatenate([top, rng.integers(0, g.n_u, 300)]))
    sv = np.unique(rng.integers(0, g.n_v, 200))
    bal, unb = O.route_s(g, verts=np.concatenate([su, g.n_u + sv]), threads=THREADS)
    assert np.array_equal(bu[su], bal[:su.size]) and np.array_equal(nu[su], unb[:su.size])
    assert np.array_equal(bv[sv], bal[su.size:]) and np.array_equal(nv[sv], unb[su.size:])


# ----------------------------------------------------------------------------- dense int8 path
def dense_all(B, g):
    """Counts through the dense path (BBF_FORCE_DENSE at load)."""
    with B.Graph.from_synth(g, flags=B.BBF_FORCE_DENSE) as h:
        glob = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
        st = h.stats()
    # the tcgen05 kernel ran (not the sparse engine); it has no algorithmic ops below 2 rows
    assert st["algo_ops"] > 0 or max(g.n_u, g.n_v) < 2
    assert st["algo_bytes"] == 0
    return glob, tot, bu, nu, bv, nv


def check_dense(B, g):
    glob, tot, bu, nu, bv, nv = dense_all(B, g)
    rg = O.route_g(g, threads=THREADS)
    assert (glob["balanced"], glob["unbalanced"]) == (rg["B"], rg["N"]), g.name
    assert glob["wedges_G"] == rg["W_G"]
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"]), g.name
    bal, unb = O.route_s(g, threads=THREADS)
    assert np.array_equal(bu, bal[:g.n_u]) and np.array_equal(nu, unb[:g.n_u]), g.name
    assert np.array_equal(bv, bal[g.n_u:]) and np.array_equal(nv, unb[g.n_u:]), g.name


def test_dense_config1_and_edge_cases(bbf):
    check_dense(bbf, G.config1())
    for g in [G.from_edges(1, 1, [], [], []),
              G.from_edges(5, 4, [0, 0, 1, 1], [0, 1, 0, 1], [1, 1, 1, 0]),
              G.from_edges(3, 3, [0, 0, 1, 1], [0, 1, 0, 1], [0, 0, 0, 0]),
              G.from_edges(1, 6, [0] * 6, list(range(6)), [1, 0, 1, 1, 0, 1])]:
        check_dense(bbf, g)


@pytest.mark.parametrize("n_u,n_v,pe,pp,seed", [
    (300, 700, 0.3, 0.5, 1),     # several 128/256 tiles on both sides, ragged tails
    (517, 263, 0.5, 0.7, 2),
    (1000, 129, 0.2, 0.9, 3),    # K just above one 128-byte block
    (257, 1500, 0.1, 0.3, 4),
])
def test_dense_random_multi_tile(bbf, n_u, n_v, pe, pp, seed):
    check_dense(bbf, G.random_bipartite(n_u, n_v, pe, pp, seed=seed))


@pytest.mark.parametrize("m,n", [(2, 2), (130, 70), (700, 600)])
def test_dense_complete_bipartite_closed_form(bbf, m, n):
    c = lambda k: k * (k - 1) // 2
    glob, tot, bu, nu, bv, nv = dense_all(bbf, G.complete(m, n))
    assert glob["balanced"] == c(m) * c(n) and glob["unbalanced"] == 0
    assert np.all(bu == (m - 1) * c(n)) and np.all(bv == (n - 1) * c(m))
    assert not nu.any() and not nv.any()


def test_dense_config2_per_vertex(bbf):
    check_dense(bbf, G.config2())


def test_dense_equals_sparse_config4_full_size(bbf):
    """configs[3] at full size: dense (tcgen05) and sparse engines agree element by element on
    both sides' per-vertex arrays; global B/N/W_G equal the oracle's Alg. 2 count; sampled
    vertices equal vBBFC computed one by one."""
    g = G.config4()
    rg = O.route_g(g, threads=THREADS)
    res = {}
    for name, fl in (("dense", bbf.BBF_FORCE_DENSE), ("sparse", bbf.BBF_FORCE_SPARSE)):
        with bbf.Graph.from_synth(g, flags=fl) as h:
            c = h.count_global()
            res[name] = (c,) + tuple(h.count_per_vertex()[1:])
            assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], rg["N"], rg["W_G"]), name
    for a, b in zip(res["dense"][1:], res["sparse"][1:]):
        assert np.array_equal(a, b)
    _, bu, nu, bv, nv = res["dense"]
    assert int(bu.sum()) == 2 * rg["B"] and int(nv.sum()) == 2 * rg["N"]
    rng = np.random.default_rng(4)
    su = np.unique(rng.integers(0, g.n_u, 40))
    sv = np.unique(rng.integers(0, g.n_v, 40))
    bal, unb = O.route_s(g, verts=np.concatenate([su, g.n_u + sv]), threads=THREADS)
    assert np.array_equal(bu[su], bal[:su.size]) and np.array_equal(nu[su], unb[:su.size])
    assert np.array_equal(bv[sv], bal[su.size:]) and np.array_equal(nv[sv], unb[su.size:])


def test_counter_encodings_agree(bbf, monkeypatch):
    """The hub kernel's two counter-address encodings (compact, and the general one used when
    a side has more than 2^20 counter words) give identical per-vertex arrays."""
    g = G.config3()
    with bbf.Graph.from_synth(g) as h:
        ref = h.count_per_vertex()
    monkeypatch.setenv("BBF_NO_COMPACT", "1")
    with bbf.Graph.from_synth(g) as h:
        got = h.count_per_vertex()
    assert got[0]["balanced"] == ref[0]["balanced"] and got[0]["unbalanced"] == ref[0]["unbalanced"]
    for a, b in zip(got[1:], ref[1:]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("m,n", [(300, 2040), (2047, 96)])
def test_dense_fp4_packed_accumulator_near_limit(bbf, monkeypatch, m, n):
    """The FP4 dense kernels at degrees just under the packed-accumulator limit (|Q| = |T + 2048 P|
    up to ~2^22): all-positive K_{m,n} per-vertex closed forms, and a random-sign graph of the same
    degrees bit-identical to the int8 tensor path (BBF_DENSE_I8) and to the two-accumulator FP4
    kernel (BBF_DENSE_F4_TP)."""
    c2 = lambda k: k * (k - 1) // 2
    with bbf.Graph.from_synth(G.complete(m, n), flags=bbf.BBF_FORCE_DENSE) as h:
        tot, bu, nu, bv, nv = h.count_per_vertex()
    assert tot["balanced"] == c2(m) * c2(n) and tot["unbalanced"] == 0
    assert (bu == (m - 1) * c2(n)).all() and (bv == (n - 1) * c2(m)).all()
    assert (nu == 0).all() and (nv == 0).all()
    g = G.random_bipartite(m, n, 0.97, 0.5, seed=m + n)
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_DENSE) as h:
        ref = h.count_per_vertex()
    for env in ("BBF_DENSE_I8", "BBF_DENSE_F4_TP"):
        monkeypatch.setenv(env, "1")
        with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_DENSE) as h:
            got = h.count_per_vertex()
        monkeypatch.delenv(env)
        assert got[0]["balanced"] == ref[0]["balanced"] and got[0]["unbalanced"] == ref[0]["unbalanced"]
        for x, y in zip(got[1:], ref[1:]):
            assert np.array_equal(x, y)


def test_dense_fp4_only_operands_then_int8(bbf, monkeypatch):
    """A graph loaded FP4-only (packed operands built by the row kernel and the nibble transpose,
    no u8 copies) counted first on the FP4 kernels, then on the same handle with the int8 pair
    kernel and the 1-CTA int8 kernel (u8 operands built on demand): identical per-vertex arrays,
    equal to the oracle's vBBFC."""
    g = G.random_bipartite(517, 391, 0.4, 0.6, seed=11)   # ragged on both sides
    bal, unb = O.route_s(g, threads=THREADS)
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_DENSE) as h:
        runs = [h.count_per_vertex()]
        for env in ("BBF_DENSE_I8", "BBF_DENSE_1CTA"):
            monkeypatch.setenv(env, "1")
            runs.append(h.count_per_vertex())
            monkeypatch.delenv(env)
        runs.append(h.count_per_vertex())
    for tot, bu, nu, bv, nv in runs:
        assert np.array_equal(bu, bal[:g.n_u]) and np.array_equal(nu, unb[:g.n_u])
        assert np.array_equal(bv, bal[g.n_u:]) and np.array_equal(nv, unb[g.n_u:])


def test_upload_and_async_outputs(bbf):
    """Pipelined loading (bbf_upload_csr / bbf_graph_load_upload, the next graph's copy in flight
    while the current one counts) and BBF_OUTPUT_ASYNC host outputs give the same counts as the
    synchronous calls, on config 3 (sparse) and a dense-path graph; outputs complete after
    bbf_device_sync."""
    import torch
    for g, fl in ((G.config3(), 0), (G.random_bipartite(600, 500, 0.2, 0.6, seed=5), bbf.BBF_FORCE_DENSE)):
        with bbf.Graph.from_synth(g, flags=fl) as h:
            ref = h.count_per_vertex()
        pin = [torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).pin_memory()
               for a in (g.row_ptr, g.col.view(np.int32), g.sign)]
        outs = [tuple(torch.zeros(k, dtype=torch.int64).pin_memory() for k in (g.n_u, g.n_u, g.n_v, g.n_v))
                for _ in range(2)]
        up = bbf.Upload(g.n_u, g.n_v, *pin)
        tots = []
        for k in range(2):
            h = bbf.Graph.from_upload(up, flags=fl)
            if k == 0:
                up = bbf.Upload(g.n_u, g.n_v, *pin)  # in flight during the first count
            tots.append(h.count_per_vertex(out=outs[k], flags=bbf.BBF_OUTPUT_ASYNC)[0])
            h.free()
        bbf.device_sync(0)
        for k in range(2):
            assert tots[k]["balanced"] == ref[0]["balanced"] and tots[k]["unbalanced"] == ref[0]["unbalanced"]
            for a, b in zip(outs[k], ref[1:]):
                assert np.array_equal(a.numpy().view(np.uint64), b)


def test_end_role_packing_agrees(bbf, monkeypatch):
    """End-role counts of "safe" ends go through one packed 64-bit RED (plan.cu k_rsafe); the
    unpacked path (BBF_NO_PACKED_END) gives identical per-vertex arrays on config 3."""
    g = G.config3()
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_SPARSE) as h:
        ref = h.count_per_vertex()
    monkeypatch.setenv("BBF_NO_PACKED_END", "1")
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_SPARSE) as h:
        got = h.count_per_vertex()
    assert got[0]["balanced"] == ref[0]["balanced"] and got[0]["unbalanced"] == ref[0]["unbalanced"]
    for a, b in zip(got[1:], ref[1:]):
        assert np.array_equal(a, b)


def test_kmn_per_vertex_beyond_2_32(bbf):
    """All-positive K_{120,9000} on the sparse path: per-U-vertex counts (m-1)C(n,2) = 4.8e9 and
    per-V-vertex (n-1)C(m,2) exceed 2^32, and the low-priority U ends have ~1e6 incoming wedges
    at degree 9,000, so the end-role packing must fall back to 64-bit REDs for them (closed
    forms, SV §8(c) P2)."""
    m, n = 120, 9000
    g = G.complete(m, n)
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_SPARSE) as h:
        tot, bu, nu, bv, nv = h.count_per_vertex()
    c2 = lambda k: k * (k - 1) // 2
    assert tot["balanced"] == c2(m) * c2(n) and tot["unbalanced"] == 0
    assert (bu == (m - 1) * c2(n)).all() and (nu == 0).all()
    assert (bv == (n - 1) * c2(m)).all() and (nv == 0).all()
    assert (m - 1) * c2(n) > 2**32


@pytest.mark.parametrize("path", ["sparse", "dense"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_fake_world_shards_sum_to_full_count(bbf, monkeypatch, path, world):
    """Multi-GPU decomposition on one GPU (SURVEY §4 "fake world"): each rank's shard of the
    work (hub units / light starts / dense tiles, item i -> rank i mod N) is counted alone,
    without the NCCL all-reduce, and the shards' global and per-vertex counts sum to the
    single-GPU result element by element."""
    g = G.config2() if path == "sparse" else G.random_bipartite(700, 600, 0.2, 0.6, seed=9)
    fl = bbf.BBF_FORCE_SPARSE if path == "sparse" else bbf.BBF_FORCE_DENSE
    with bbf.Graph.from_synth(g, flags=fl) as h:
        full = h.count_per_vertex()
    acc = None
    for r in range(world):
        monkeypatch.setenv("BBF_FAKE_WORLD", f"{r}/{world}")
        with bbf.Graph.from_synth(g, flags=fl) as h:
            part = h.count_per_vertex()
        vals = [part[0]["balanced"], part[0]["unbalanced"]] + [a.astype(object) for a in part[1:]]
        acc = vals if acc is None else [x + y for x, y in zip(acc, vals)]
    monkeypatch.delenv("BBF_FAKE_WORLD")
    assert acc[0] == full[0]["balanced"] and acc[1] == full[0]["unbalanced"]
    for a, b in zip(acc[2:], full[1:]):
        assert np.array_equal(a.astype(np.uint64), b)


# ----------------------------------------------------------------------------- NEXT-1 SBESPAR
@pytest.mark.parametrize("name,rho,trials", [("config1", 0.5, 6), ("config2", 0.7, 3), ("config3", 0.6, 2),
                                             ("corpus", 1.0, 2)])
def test_estimator_samples_match_oracle(bbf, name, rho, trials):
    """bbf_estimate_global draws the same edge samples as the oracle (same documented
    counter-based generator) and counts each sample exactly: per-trial sampled B and N are
    bit-exact and the estimates equal B * rho^-4."""
    g = {"config1": G.config1, "config2": G.config2, "config3": G.config3,
         "corpus": lambda: G.random_bipartite(12, 11, 0.5, 0.5, seed=4)}[name]()
    got = bbf.estimate_global(g.n_u, g.n_v, g.row_ptr, g.col, g.sign, rho, trials, seed=123)
    for t in range(trials):
        r = O.route_g(O.sparsify(g, rho, 123, t), threads=THREADS)
        assert (int(got["sampled_B"][t]), int(got["sampled_N"][t])) == (r["B"], r["N"]), (name, t)
        # the estimate is the one floating-point step: equal up to rounding (a few ulps)
        assert abs(got["estimates"][t] - r["B"] / rho ** 4) <= 1e-12 * max(1.0, r["B"] / rho ** 4)


# ----------------------------------------------------------------------------- NEXT-2 analytics
@pytest.mark.parametrize("name", ["config2", "random", "config1"])
def test_positive_only_analytics(bbf, name):
    """BBF_POSITIVE_ONLY at load: every count describes the positive subgraph (case study,
    PAPER.md:15-27): per-vertex arrays = vBBFC on the oracle's positive subgraph, N = 0, top-k
    pairs and top-k vertices (by balanced count and by positive degree) = the oracle rankings."""
    g = {"config2": G.config2, "config1": G.config1,
         "random": lambda: G.random_bipartite(300, 200, 0.1, 0.5, seed=8)}[name]()
    p = O.positive_subgraph(g)
    with bbf.Graph.from_synth(g, flags=bbf.BBF_POSITIVE_ONLY) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
        pairs = h.count_pairs_topk(50, side=0)
        tv_b = h.topk_vertices(20, side=0, metric=bbf.BBF_METRIC_BALANCED)
        tv_d = h.topk_vertices(20, side=1, metric=bbf.BBF_METRIC_DEGREE)
    rg = O.route_g(p, threads=THREADS)
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], 0, rg["W_G"])
    bal, unb = O.route_s(p, threads=THREADS)
    assert np.array_equal(bu, bal[:g.n_u]) and np.array_equal(bv, bal[g.n_u:])
    assert not nu.any() and not nv.any()
    assert pairs == O.topk_pairs(p, 50, side=0, threads=THREADS)
    assert tv_b == O.topk_vertices(p, 20, 0, "balanced", threads=THREADS)
    assert tv_d == O.topk_vertices(p, 20, 1, "degree")


def test_topk_vertices_signed_graph(bbf):
    g = G.config2()
    with bbf.Graph.from_synth(g) as h:
        got = h.topk_vertices(100, side=1, metric=bbf.BBF_METRIC_BALANCED)
        got_all = h.topk_vertices(10 ** 6, side=0, metric=bbf.BBF_METRIC_DEGREE)
    assert got == O.topk_vertices(g, 100, 1, "balanced", threads=THREADS)
    assert got_all == O.topk_vertices(g, 10 ** 6, 0, "degree")


@pytest.mark.parametrize("env", [{"BBF_T3_BSZ": "2"}, {"BBF_T3_BSZ": "32"}, {"BBF_T3_BSZ": "0"},
                                 {"BBF_DENSE_DIV": "1000000"}, {"BBF_DENSE_DIV": "1"}])
def test_schedule_independence(bbf, monkeypatch, env):
    """Counts do not depend on the hub kernel's schedule (record batch size, dense-window
    threshold) — the GPU analogue of SPEC.md:359's determinism across worker counts."""
    g = G.config2()
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_SPARSE) as h:
        ref = h.count_per_vertex()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_SPARSE) as h:
        got = h.count_per_vertex()
    assert (got[0]["balanced"], got[0]["unbalanced"]) == (ref[0]["balanced"], ref[0]["unbalanced"])
    for a, b in zip(got[1:], ref[1:]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cap", ["120", "400", "3000"])
def test_topk_threshold_search(bbf, monkeypatch, cap):
    """Top-k pairs when the candidate buffer is smaller than the number of pairs: the threshold
    search (raise tau from a sample, lower on too few, exact buffer on ties) still returns the
    oracle's ranking."""
    g = G.config2()
    want = O.topk_pairs(g, 100, side=1, threads=THREADS)
    monkeypatch.setenv("BBF_TOPK_CAP", cap)
    with bbf.Graph.from_synth(g) as h:
        assert h.count_pairs_topk(100, side=1) == want
        assert h.count_pairs_topk(7, side=0) == O.topk_pairs(g, 7, side=0, threads=THREADS)


def _sweep_graph(seed):
    """Seeded shapes for the randomized sweep: uniform random bipartite graphs of mixed aspect
    ratio, density and sign balance, and small Chung-Lu power-law graphs (hubs on both sides)."""
    rng = np.random.default_rng(1000 + seed)
    if seed % 3 == 2:
        n_u, n_v = int(rng.integers(200, 3000)), int(rng.integers(100, 2000))
        m = int(min(n_u * n_v // 3, rng.integers(2000, 30000)))
        keys, r2 = G.chung_lu(n_u, n_v, m, float(rng.uniform(2.1, 2.8)), n_v / 3.0, n_u / 3.0, seed=seed)
        s = (r2.random(keys.size) < rng.uniform(0.0, 1.0)).astype(np.uint8)
        return G.from_edges(n_u, n_v, (keys // n_v).tolist(), (keys % n_v).tolist(), s.tolist())
    n_u, n_v = int(rng.integers(1, 500)), int(rng.integers(1, 500))
    return G.random_bipartite(n_u, n_v, float(rng.uniform(0.005, 0.5)), float(rng.uniform(0.0, 1.0)),
                              seed=seed)


# BBF_SWEEP_SEEDS="a:b" widens the sweep (e.g. 40:400 for an extended run on the GPU box)
_SWEEP = range(*map(int, os.environ.get("BBF_SWEEP_SEEDS", "0:40").split(":")))


@pytest.mark.parametrize("seed", _SWEEP)
def test_random_sweep_tiers_dense_topk(bbf, monkeypatch, seed):
    """Randomized sweep: per-vertex counts of the default tiering, of T3-only (T2 disabled, every
    start above the warp tier goes through the hub kernel), of the hybrid path with a random
    forced core and of the dense path equal the oracle's vBBFC element by element; global B/N/W_G equal Alg. 2; top-k pairs of both sides
    equal the oracle's."""
    g = _sweep_graph(seed)
    rg = O.route_g(g, threads=THREADS)
    bal, unb = O.route_s(g, threads=THREADS)
    rng = np.random.default_rng(5000 + seed)
    core = f"{int(rng.integers(2, max(3, g.n_u)))},{int(rng.integers(2, max(3, g.n_v)))}"
    runs = [("default", {}, 0), ("t3-only", {"BBF_T2_MAX": "0"}, bbf.BBF_FORCE_SPARSE),
            ("hybrid", {"BBF_HYBRID_CORE": core}, 0)]  # a random forced dense core
    if max(g.n_u, g.n_v) <= 65536:
        runs.append(("dense", {}, bbf.BBF_FORCE_DENSE))
    for name, env, fl in runs:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with bbf.Graph.from_synth(g, flags=fl) as h:
            c = h.count_global()
            tot, bu, nu, bv, nv = h.count_per_vertex()
            if name == "default":
                for side in (0, 1):
                    assert h.count_pairs_topk(10, side=side) == O.topk_pairs(g, 10, side=side, threads=THREADS)
        for k in env:
            monkeypatch.delenv(k)
        assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], rg["N"], rg["W_G"]), name
        assert np.array_equal(bu, bal[:g.n_u]) and np.array_equal(nu, unb[:g.n_u]), name
        assert np.array_equal(bv, bal[g.n_u:]) and np.array_equal(nv, unb[g.n_u:]), name


@pytest.mark.parametrize("name", ["config1", "config2", "skewed", "sweep5", "sweep11", "chung_lu"])
def test_bb_base_gpu_equals_oracle_alg1(bbf, name):
    """bbf_count_global_base (Alg. 1 BB-Base on the GPU: explicit pair checks per H(w)) equals the
    oracle's Alg. 1 and Alg. 2 counts and the bucketed GPU count."""
    g = {"config1": G.config1, "config2": G.config2,
         "skewed": lambda: G.random_bipartite(10, 1000, 0.5, 0.5, seed=7),
         "sweep5": lambda: _sweep_graph(5), "sweep11": lambda: _sweep_graph(11),
         "chung_lu": lambda: _sweep_graph(2)}[name]()
    ob = O.bb_base(g, threads=THREADS)
    with bbf.Graph.from_synth(g) as h:
        base = h.count_global_base()
        buck = h.count_global()
    assert (base["balanced"], base["unbalanced"]) == (ob["B"], ob["N"])
    assert (buck["balanced"], buck["unbalanced"]) == (ob["B"], ob["N"])
    assert base["wedges_G"] == ob["W_G"]


def test_bb_base_gpu_table_limit_error(bbf):
    """A start with more distinct ends than BB-Base's 8,192-slot table: BBF_EINVAL, not a wrong
    count (u0 adjacent to all 200 V vertices; 12,000 other U vertices of degree 2, so every V
    vertex has degree 121 < 200 and u0 is the top-priority start with 12,000 distinct ends)."""
    n_v, n_e = 200, 12000
    us, vs = [0] * n_v, list(range(n_v))
    for i in range(n_e):
        a = i % n_v
        b = (a + 1 + (i // n_v) % (n_v - 1)) % n_v
        us += [1 + i, 1 + i]
        vs += [a, b]
    g = G.from_edges(1 + n_e, n_v, us, vs, [1] * len(us))
    with bbf.Graph.from_synth(g) as h:
        with pytest.raises(bbf.BBFError) as e:
            h.count_global_base()
        assert e.value.name == "BBF_EINVAL"
        assert h.count_global()["balanced"] == O.route_g(g)["B"]


@pytest.mark.parametrize("world", [2, 5])
def test_bb_base_fake_world_shards_sum(bbf, monkeypatch, world):
    """BB-Base's start sharding (start x on rank x mod N): the shards' counts, each counted alone
    without the all-reduce, sum to the single-GPU count."""
    g = _sweep_graph(8)
    with bbf.Graph.from_synth(g) as h:
        full = h.count_global_base()
    tb = tn = 0
    for r in range(world):
        monkeypatch.setenv("BBF_FAKE_WORLD", f"{r}/{world}")
        with bbf.Graph.from_synth(g) as h:
            part = h.count_global_base()
        tb += part["balanced"]
        tn += part["unbalanced"]
    monkeypatch.delenv("BBF_FAKE_WORLD")
    assert (tb, tn) == (full["balanced"], full["unbalanced"])
    assert full["balanced"] == O.route_g(g)["B"]


def test_dense_mixed_fp4_int8_sides(bbf):
    """Dense path where one side's rows exceed the FP4 exactness bound (U rows of degree 9,000 >
    8,192: int8 kernel on the u8 operands) and the other side's do not (V rows of degree 120: FP4
    kernel): the load builds u8 operands with FP4 copies for the eligible side only.  Random signs
    vs the oracle's vBBFC on sampled vertices, and K_{120,9000} closed forms beyond 2^32."""
    m, n = 120, 9000
    c2 = lambda k: k * (k - 1) // 2
    with bbf.Graph.from_synth(G.complete(m, n), flags=bbf.BBF_FORCE_DENSE) as h:
        tot, bu, nu, bv, nv = h.count_per_vertex()
    assert tot["balanced"] == c2(m) * c2(n) and tot["unbalanced"] == 0
    assert (bu == (m - 1) * c2(n)).all() and (bv == (n - 1) * c2(m)).all()
    assert (m - 1) * c2(n) > 2**32
    g = G.random_bipartite(m, n, 0.95, 0.5, seed=21)
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_DENSE) as h:
        tot, bu, nu, bv, nv = h.count_per_vertex()
    rg = O.route_g(g, threads=THREADS)
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"])
    sv = np.arange(0, n, 450)
    bal, unb = O.route_s(g, verts=np.concatenate([np.arange(m), m + sv]), threads=THREADS)
    assert np.array_equal(bu, bal[:m]) and np.array_equal(nu, unb[:m])
    assert np.array_equal(bv[sv], bal[m:]) and np.array_equal(nv[sv], unb[m:])


def test_dense_wide_v_side_global_wedge_pass(bbf):
    """A dense-path candidate whose V side (60,000) is beyond the shared-memory column
    histograms (49,152): V degrees and the load-time W_G take the hashed / global-atomic kernels;
    counts and W_G equal the oracle's, per-vertex arrays equal vBBFC on sampled vertices."""
    g = G.random_bipartite(300, 60000, 0.02, 0.5, seed=31)
    rg = O.route_g(g, threads=THREADS)
    with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_DENSE) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (rg["B"], rg["N"], rg["W_G"])
    sv = np.arange(0, g.n_v, 997)
    bal, unb = O.route_s(g, verts=np.concatenate([np.arange(g.n_u), g.n_u + sv]), threads=THREADS)
    assert np.array_equal(bu, bal[:g.n_u]) and np.array_equal(nu, unb[:g.n_u])
    assert np.array_equal(bv[sv], bal[g.n_u:]) and np.array_equal(nv[sv], unb[g.n_u:])
