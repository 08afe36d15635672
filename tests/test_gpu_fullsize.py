"""Full-size GPU parity: the ENTIRE per-vertex arrays (both sides) of BASELINE configs 3, 4 and 5
and of the zoned graph against the oracle's Alg. 2 + 4-role scatter (oracle_route_g_pv), plus
global B, N and W_G, plus the expected-counts file bench.py asserts against
(tests/golden/expected_counts.json, written by tests/scripts/write_expected.py from oracle/ only).

Also the multi-GPU decomposition on hub graphs: BBF_FAKE_WORLD=r/N counts rank r's shard of the
work items alone (hub units of k_t3, k_t2 starts, k_t1 starts) on one GPU; the shards must sum to
the oracle's arrays element by element, and every shard must hold part of the work."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
from synth import graphs as G

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 8
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "expected_counts.json")
_cache = {}


@pytest.fixture(scope="module")
def bbf():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_07932_b200 import build
    build.build()
    from paper_2308_07932_b200 import bbf as B
    return B


def graph(name):
    if name not in _cache:
        if name == "zoned":
            from test_gpu_parity import zoned_graph
            g = zoned_graph()
        else:
            g = G.make_config(int(name[-1]))
        _cache[name] = (g, O.route_g_pv(g, threads=THREADS))
    return _cache[name]


def pv_sha256(bu, nu, bv, nv):
    h = hashlib.sha256()
    for a in (bu, nu, bv, nv):
        h.update(np.ascontiguousarray(a, dtype="<u8").tobytes())
    return h.hexdigest()


def assert_equal_arrays(got, want, tag):
    for k, a in zip(("bal_u", "unb_u", "bal_v", "unb_v"), got):
        b = want[k]
        if not np.array_equal(a, b):
            bad = np.nonzero(a != b)[0]
            raise AssertionError(f"{tag} {k}: {bad.size} vertices differ, first {bad[:5].tolist()} "
                                 f"got {a[bad[:5]].tolist()} want {b[bad[:5]].tolist()}")


@pytest.mark.parametrize("name,flags", [("config3", "default"), ("config4", "default"),
                                        ("config4", "sparse"), ("config5", "default"),
                                        ("zoned", "sparse")])
def test_full_per_vertex_vs_oracle(bbf, name, flags):
    g, want = graph(name)
    fl = {"default": 0, "sparse": bbf.BBF_FORCE_SPARSE}[flags]
    with bbf.Graph.from_synth(g, flags=fl) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
        st = h.stats()
    if name == "config4" and flags == "default":
        assert st["algo_ops"] > 0  # the dispatch sent it to the tensor-core path
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (want["B"], want["N"], want["W_G"])
    assert (tot["balanced"], tot["unbalanced"]) == (want["B"], want["N"])
    assert_equal_arrays((bu, nu, bv, nv), want, name)
    if name.startswith("config"):
        exp = json.load(open(GOLDEN))[name]
        assert exp["graph_sha256"] == g.sha256()
        assert (exp["B"], exp["N"], exp["W_G"]) == (want["B"], want["N"], want["W_G"])
        assert exp["pv_sha256"] == pv_sha256(bu, nu, bv, nv)


@pytest.mark.parametrize("name", ["config3", "zoned"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_fake_world_shards_on_hub_graphs(bbf, monkeypatch, name, world):
    """The sharded work items of every tier (k_t3 hub units, k_t2 and k_t1 starts; item i on rank
    i mod N) counted rank by rank: shards sum to the oracle's global and per-vertex counts, and
    no shard is empty or the whole."""
    g, want = graph(name)
    acc = None
    parts = []
    for r in range(world):
        monkeypatch.setenv("BBF_FAKE_WORLD", f"{r}/{world}")
        with bbf.Graph.from_synth(g, flags=bbf.BBF_FORCE_SPARSE) as h:
            part = h.count_per_vertex()
        parts.append(part[0]["balanced"])
        vals = [part[0]["balanced"], part[0]["unbalanced"]] + [a.astype(object) for a in part[1:]]
        acc = vals if acc is None else [x + y for x, y in zip(acc, vals)]
    monkeypatch.delenv("BBF_FAKE_WORLD")
    assert (acc[0], acc[1]) == (want["B"], want["N"])
    assert all(0 < p < want["B"] for p in parts), parts
    assert_equal_arrays([a.astype(np.uint64) for a in acc[2:]], want, f"{name} world {world}")


@pytest.mark.parametrize("world", [2, 3])
def test_fake_world_topk_shards_merge(bbf, monkeypatch, world):
    """S12 top-k: each rank's shard returns its local top-k; the merged lists (what the library's
    ncclAllGather + merge does across ranks) equal the oracle's global top-k."""
    g = G.config2()
    lists = []
    for r in range(world):
        monkeypatch.setenv("BBF_FAKE_WORLD", f"{r}/{world}")
        with bbf.Graph.from_synth(g) as h:
            lists.append(h.count_pairs_topk(100, side=0))
    monkeypatch.delenv("BBF_FAKE_WORLD")
    merged = sorted([t for lst in lists for t in lst], key=lambda t: (-t[2], t[0], t[1]))[:100]
    assert merged == O.topk_pairs(g, 100, side=0, threads=THREADS)
    assert all(len(lst) > 0 for lst in lists)


def test_single_rank_nccl_communicator(bbf):
    """The collective path with a real NCCL communicator of one rank (bbf_comm_init, the u64
    all-reduces with the status max-reduce, the top-k all-gather, the async-error polling wait):
    counts equal the oracle's."""
    g = G.config2()
    comm = bbf.Comm(bbf.nccl_unique_id(), 1, 0, 0)
    try:
        with bbf.Graph.from_synth(g, comm=comm) as h:
            c = h.count_global()
            tot, bu, nu, bv, nv = h.count_per_vertex()
            top = h.count_pairs_topk(100, side=1)
            base = h.count_global_base()
    finally:
        comm.free()
    want = O.route_g_pv(g, threads=THREADS)
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (want["B"], want["N"], want["W_G"])
    assert (base["balanced"], base["unbalanced"]) == (want["B"], want["N"])
    assert_equal_arrays((bu, nu, bv, nv), want, "comm1")
    assert top == O.topk_pairs(g, 100, side=1, threads=THREADS)


def test_estimate_rejects_malformed_input_before_sampling(bbf):
    """bbf_estimate_global validates its input CSR (S1) before the sampling kernels read it: a
    row_ptr entry beyond nnz, a column out of range and a bad sign byte return the load's codes."""
    rp = np.array([0, 5, 2], np.uint64)  # not monotone, and rp[1] > nnz
    col = np.array([0, 1], np.uint32)
    sg = np.array([1, 1], np.uint8)
    with pytest.raises(bbf.BBFError) as e:
        bbf.estimate_global(2, 2, rp, col, sg, 0.5, 2)
    assert e.value.name == "BBF_ERANGE"
    with pytest.raises(bbf.BBFError) as e:
        bbf.estimate_global(2, 2, np.array([0, 1, 2], np.uint64), np.array([0, 7], np.uint32), sg, 0.5, 2)
    assert e.value.name == "BBF_ERANGE"
    with pytest.raises(bbf.BBFError) as e:
        bbf.estimate_global(2, 2, np.array([0, 1, 2], np.uint64), col, np.array([1, 2], np.uint8), 0.5, 2)
    assert e.value.name == "BBF_EINVAL"


# ----------------------------------------------------------------------------- NEXT-4 per-edge counts
@pytest.mark.parametrize("name", ["config1", "config2", "kmn", "sweep2", "sweep7", "sweep8", "skewed", "zoned"])
def test_per_edge_counts_vs_oracle(bbf, name):
    """bbf_count_per_edge equals the oracle's per-edge definition edge by edge,
    in the caller's CSR order; totals equal Alg. 2's; each vertex's edges sum to twice its count."""
    from test_gpu_parity import _sweep_graph, zoned_graph
    g = {"config1": G.config1, "config2": G.config2, "kmn": lambda: G.complete(37, 23),
         "sweep2": lambda: _sweep_graph(2), "sweep7": lambda: _sweep_graph(7), "sweep8": lambda: _sweep_graph(8),
         "skewed": lambda: G.random_bipartite(10, 1000, 0.5, 0.5, seed=7), "zoned": zoned_graph}[name]()
    with bbf.Graph.from_synth(g) as h:
        tot, eb, en = h.count_per_edge(g.row_ptr, g.col)
        _, bu, nu, bv, nv = h.count_per_vertex()
    if name == "zoned":  # too large for the oracle's edge-by-edge definition: identities + brute-free pins
        u = np.repeat(np.arange(g.n_u), np.diff(g.row_ptr.astype(np.int64)))
        assert int(eb.astype(object).sum()) == 4 * tot["balanced"] and int(en.astype(object).sum()) == 4 * tot["unbalanced"]
        su = np.zeros(g.n_u, dtype=object)
        np.add.at(su, u, eb.astype(object))
        assert np.array_equal(su.astype(np.uint64), 2 * bu)
        return
    wb, wn = O.edge_counts(g, threads=THREADS)
    assert np.array_equal(eb, wb) and np.array_equal(en, wn)
    rg = O.route_g(g, threads=THREADS)
    assert (tot["balanced"], tot["unbalanced"]) == (rg["B"], rg["N"])


def test_per_edge_fake_world_shards(bbf, monkeypatch):
    """Per-edge counts sharded over 3 fake ranks sum to the single-GPU arrays."""
    from test_gpu_parity import _sweep_graph
    g = _sweep_graph(8)
    with bbf.Graph.from_synth(g) as h:
        _, eb, en = h.count_per_edge(g.row_ptr, g.col)
    sb = np.zeros(g.nnz, dtype=object)
    sn = np.zeros(g.nnz, dtype=object)
    for r in range(3):
        monkeypatch.setenv("BBF_FAKE_WORLD", f"{r}/3")
        with bbf.Graph.from_synth(g) as h:
            _, pb, pn = h.count_per_edge(g.row_ptr, g.col)
        sb += pb.astype(object)
        sn += pn.astype(object)
    monkeypatch.delenv("BBF_FAKE_WORLD")
    assert np.array_equal(sb.astype(np.uint64), eb) and np.array_equal(sn.astype(np.uint64), en)


def test_per_edge_rejects_foreign_csr(bbf):
    """A CSR that is not the loaded graph's edge set (other edge count, or the same count with
    other edges) is rejected with BBF_EINVAL; the graph's edges in another order are accepted."""
    g = G.config1()
    other = G.random_bipartite(200, 150, 0.05, 0.5, seed=99)
    u, v, s = g.edges()
    same_n = G.from_edges(200, 150, u, v[::-1].copy(), s, check_dup=False)  # 2,000 edges, mostly not g's
    with bbf.Graph.from_synth(g) as h:
        for bad in (other, same_n):
            with pytest.raises(bbf.BBFError) as e:
                h.count_per_edge(bad.row_ptr, bad.col)
            assert e.value.name == "BBF_EINVAL"
        _, eb, en = h.count_per_edge(g.row_ptr, g.col)
        perm = np.concatenate([np.arange(a, b)[::-1] for a, b in zip(g.row_ptr[:-1].astype(np.int64),
                                                                      g.row_ptr[1:].astype(np.int64))])
        _, pb, pn = h.count_per_edge(g.row_ptr, g.col[perm])  # rows reversed: same edges, other order
    assert np.array_equal(pb, eb[perm]) and np.array_equal(pn, en[perm])


def test_per_edge_device_pointers_and_empty(bbf):
    """Per-edge counts with device arrays (BBF_PTR_DEVICE: CUDA tensors in and out) equal the host
    call; an empty graph gives empty arrays and zero totals."""
    import torch
    g = G.config2()
    with bbf.Graph.from_synth(g) as h:
        tot, eb, en = h.count_per_edge(g.row_ptr, g.col)
        rp = torch.from_numpy(g.row_ptr.view(np.int64)).cuda()
        cl = torch.from_numpy(g.col.view(np.int32)).cuda()
        ob = torch.zeros(g.nnz, dtype=torch.int64, device="cuda")
        on = torch.zeros(g.nnz, dtype=torch.int64, device="cuda")
        tot2, _, _ = h.count_per_edge(rp, cl, out=(ob, on))
    assert (tot2["balanced"], tot2["unbalanced"]) == (tot["balanced"], tot["unbalanced"])
    assert np.array_equal(ob.cpu().numpy().view(np.uint64), eb) and np.array_equal(on.cpu().numpy().view(np.uint64), en)
    e = G.from_edges(3, 4, [], [], [])
    with bbf.Graph.from_synth(e) as h:
        tot, eb, en = h.count_per_edge(e.row_ptr, e.col)
    assert eb.size == 0 and en.size == 0 and tot["balanced"] == 0


_EDGE_SWEEP = range(*map(int, os.environ.get("BBF_EDGE_SWEEP_SEEDS", "0:12").split(":")))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", _EDGE_SWEEP)
def test_per_edge_and_shards_sweep(bbf, monkeypatch, seed):
    """Randomized sweep of the per-edge counts (all three tiers, both route-S directions) against
    the oracle's per-edge definition, and of the per-vertex counts of an N-way fake world (N = 2..8
    by seed) summed over the shards against the oracle's route-G per-vertex arrays."""
    from test_gpu_parity import _sweep_graph
    g = _sweep_graph(seed)
    with bbf.Graph.from_synth(g) as h:
        _, eb, en = h.count_per_edge(g.row_ptr, g.col)
    wb, wn = O.edge_counts(g, threads=THREADS)
    assert np.array_equal(eb, wb) and np.array_equal(en, wn)
    N = 2 + seed % 7
    acc = [np.zeros(g.n_u, dtype=object), np.zeros(g.n_u, dtype=object),
           np.zeros(g.n_v, dtype=object), np.zeros(g.n_v, dtype=object)]
    for r in range(N):
        monkeypatch.setenv("BBF_FAKE_WORLD", f"{r}/{N}")
        with bbf.Graph.from_synth(g) as h:
            _, bu, nu, bv, nv = h.count_per_vertex()
        for i, arr in enumerate((bu, nu, bv, nv)):
            acc[i] += arr.astype(object)
    monkeypatch.delenv("BBF_FAKE_WORLD")
    want = O.route_g_pv(g, threads=THREADS)
    got = [a.astype(np.uint64) for a in acc]
    assert np.array_equal(got[0], want["bal_u"]) and np.array_equal(got[1], want["unb_u"])
    assert np.array_equal(got[2], want["bal_v"]) and np.array_equal(got[3], want["unb_v"])


def _large_variant(i):
    """Large skewed stand-ins beyond the five configs (other sizes, exponents, hub weights and
    sign mixes), same recipe as config 5: Chung-Lu keys, per-V Beta sign bias."""
    spec = [(4_000_000, 1_000_000, 25_000_000, 1.8, 60_000.0, 80_000.0, (2.0, 2.0)),
            (2_000_000, 3_000_000, 30_000_000, 2.1, 150_000.0, 40_000.0, (1.0, 3.0)),
            (6_000_000, 500_000, 20_000_000, 2.4, 20_000.0, 200_000.0, (5.0, 1.0))][i]
    n_u, n_v, m, gamma, wu, wv, (ba, bb) = spec
    key, rng = G.chung_lu(n_u, n_v, m, gamma, wu, wv, 700 + i)
    b = rng.beta(ba, bb, size=n_v)
    s = rng.random(key.size) < b[key % n_v]
    return G._from_sorted_keys(n_u, n_v, key, s, f"large{i}")


@pytest.mark.gpu
@pytest.mark.skipif(not os.environ.get("BBF_FULLSIZE_EXTRA"), reason="extended run: set BBF_FULLSIZE_EXTRA=1")
@pytest.mark.parametrize("i", [0, 1, 2])
def test_full_per_vertex_large_variants(bbf, i):
    """The whole per-vertex arrays of large skewed graphs other than the configs equal the
    oracle's route-G 4-role scatter element by element (extended run, minutes of oracle time)."""
    g = _large_variant(i)
    want = O.route_g_pv(g, threads=THREADS)
    with bbf.Graph.from_synth(g) as h:
        c = h.count_global()
        tot, bu, nu, bv, nv = h.count_per_vertex()
    assert (c["balanced"], c["unbalanced"], c["wedges_G"]) == (want["B"], want["N"], want["W_G"])
    assert_equal_arrays((bu, nu, bv, nv), want, f"large{i}")
