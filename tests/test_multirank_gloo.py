"""World-size-2 tests of the N>1 path over torch.distributed gloo (one process per rank).

CPU: the bootstrap plumbing of paper_2308_07932_b200.dist (ncclUniqueId broadcast, max-over-ranks
timing, exact uint64 sums beyond 2^63) and that every rank loads libbbf.so.
GPU: each rank counts ITS OWN shard of the work with the library (BBF_FAKE_WORLD=rank/2: the
kernels skip the other rank's work items, no NCCL — one GPU is all this environment has), the
per-vertex arrays and totals are summed across the two processes over gloo, and the sum must
equal the oracle's Alg. 2 + 4-role scatter element by element; the shards' local top-k pair lists,
gathered and merged, must equal the oracle's top-k.  Config 6 (the NEXT-3 workload) runs the
hybrid dense-core path on each rank (dense tiles, engine items and mixed middles sharded)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


def _init(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _plumbing_worker(rank, world, port, q):
    dist = _init(rank, world, port)
    try:
        from paper_2308_07932_b200 import dist as D
        from paper_2308_07932_b200 import bbf
        bbf.lib()  # the library loads and resolves its symbols on every rank
        uid = bytes(np.random.default_rng(7).integers(0, 256, 128, dtype=np.uint8)) if rank == 0 else None
        got = D.broadcast_unique_id(uid, 0)
        t = D.max_over_ranks(10.0 + rank)
        big = [2**63 + 5 + rank, 2**40 * (rank + 1), 2**64 - 1 - rank if rank == 0 else 0]
        s = D.sum_over_ranks_u64(big)
        q.put((rank, got, t, [int(v) for v in s]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_plumbing():
    res = _run(_plumbing_worker, 2)
    assert all(r[1] == res[0][1] and len(r[1]) == 128 for r in res)
    assert all(r[2] == 11.0 for r in res)  # max over ranks
    want = [(2**63 + 5 + 2**63 + 6) % 2**64, 2**40 * 3, 2**64 - 1]
    assert all(r[3] == want for r in res)


def _shard_worker(rank, world, port, q, cfg):
    dist = _init(rank, world, port)
    try:
        import torch
        from paper_2308_07932_b200 import dist as D
        from paper_2308_07932_b200 import bbf
        from test_gpu_parity import _sweep_graph
        from synth import graphs as G
        torch.cuda.set_device(0)
        os.environ["BBF_FAKE_WORLD"] = f"{rank}/{world}"
        g = G.make_config(cfg) if isinstance(cfg, int) else _sweep_graph(int(cfg[5:]))
        hybrid = cfg == 6  # the NEXT-3 workload on the automatic dispatch: the hybrid dense-core path
        with bbf.Graph.from_synth(g, flags=0 if hybrid else bbf.BBF_FORCE_SPARSE) as h:
            tot, bu, nu, bv, nv = h.count_per_vertex()
            top = h.count_pairs_topk(50, side=0) if g.n_u <= 200_000 else []
            assert not hybrid or h.hybrid_core() != (0, 0)
        vals = np.concatenate([[tot["balanced"], tot["unbalanced"]], bu, nu, bv, nv]).astype(np.uint64)
        summed = D.sum_over_ranks_u64(vals)
        tops = [None] * world
        dist.all_gather_object(tops, top)
        q.put((rank, int(tot["balanced"]), summed, tops))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [3, 6, "sweep2", "sweep8"])
def test_two_rank_library_shards_sum_to_oracle(cfg):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2308_07932_b200 import build
    build.build()
    import oracle as O
    from synth import graphs as G
    from test_gpu_parity import _sweep_graph
    res = _run(_shard_worker, 2, cfg)
    g = G.make_config(cfg) if isinstance(cfg, int) else _sweep_graph(int(cfg[5:]))
    want = O.route_g_pv(g)
    n_u, n_v = g.n_u, g.n_v
    for rank, part_b, s, tops in res:
        assert 0 < part_b < want["B"]  # each rank held a real share of the work
        assert (int(s[0]), int(s[1])) == (want["B"], want["N"])
        o = 2
        for k, cnt in (("bal_u", n_u), ("unb_u", n_u), ("bal_v", n_v), ("unb_v", n_v)):
            assert np.array_equal(s[o:o + cnt], want[k]), k
            o += cnt
        if g.n_u <= 200_000:
            merged = sorted([t for lst in tops for t in lst], key=lambda t: (-t[2], t[0], t[1]))[:50]
            assert merged == O.topk_pairs(g, 50, side=0)
