"""World-size-2 CPU (gloo) tests of the N>1 path: NCCL-id broadcast plumbing, max-over-ranks
timing, the item-mod-rank sharding rule, and that per-rank partial counts of disjoint start
shards all-reduce to the exact global count (the property the multi-GPU all-reduce relies on;
each rank's partial is computed by the oracle here since there is no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_07932_b200 import dist as D
        import oracle as O
        from synth import graphs as G
        uid = bytes(np.random.default_rng(7).integers(0, 256, 128, dtype=np.uint8)) if rank == 0 else None
        got = D.broadcast_unique_id(uid, 0)
        t = D.max_over_ranks(10.0 + rank)
        g = G.random_bipartite(60, 50, 0.3, 0.65, seed=21)
        n = g.n_u + g.n_v
        # start vertices in priority order (the plan's order); item i -> rank i mod world
        order = np.argsort(O.priority_order(g), kind="stable")
        mine = [int(order[i]) for i in range(n) if D.shard_owner(i, world) == rank]
        part = O.route_g(g, starts=np.array(mine, dtype=np.uint32), threads=1)
        tot = D.sum_over_ranks_u64([part["B"], part["N"], part["W_G"]])
        q.put((rank, got, t, tot, len(mine)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_plumbing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle as O
    from synth import graphs as G
    g = G.random_bipartite(60, 50, 0.3, 0.65, seed=21)
    full = O.route_g(g)
    uid0 = res[0][1]
    assert all(r[1] == uid0 and len(r[1]) == 128 for r in res)
    assert all(r[2] == 11.0 for r in res)  # max over ranks
    assert all(tuple(r[3]) == (full["B"], full["N"], full["W_G"]) for r in res)
    assert sum(r[4] for r in res) == g.n_u + g.n_v
