"""Multi-GPU plumbing over torch.distributed (one process per GPU).

The library shards the work itself (work item i of the plan goes to rank i mod N, DESIGN.md
§Multi-GPU) and combines the counts with NCCL collectives of its own communicator; this module
only bootstraps that communicator (the 128-byte ncclUniqueId travels over the torch process
group) and provides the max-over-ranks timing reduction and an exact uint64 sum the harness uses.
Works with the nccl backend (CUDA tensors) and with gloo (CPU tensors, the CPU tests)."""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def _dev(group=None):
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_unique_id(uid: bytes | None, src: int = 0, group=None) -> bytes:
    """Rank `src` passes the id (bbf.nccl_unique_id()), every rank gets it back."""
    t = torch.zeros(128, dtype=torch.uint8, device=_dev(group))
    if dist.get_rank(group) == src:
        assert uid is not None and len(uid) == 128
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(t, src, group=group)
    return bytes(t.cpu().numpy().tobytes())


def make_comm(device: int, group=None):
    """The library's NCCL communicator for this rank (collective over the group)."""
    from . import bbf
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = bbf.nccl_unique_id() if rank == 0 else None
    uid = broadcast_unique_id(uid, 0, group)
    return bbf.Comm(uid, world, rank, device)


def max_over_ranks(x: float, group=None) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks_u64(vals, group=None) -> np.ndarray:
    """Exact uint64 sum across ranks (mod 2^64, like the library's ncclUint64 all-reduce): the
    values travel as 32-bit halves in int64 lanes, whose sums cannot overflow for < 2^31 ranks."""
    a = np.ascontiguousarray(np.asarray(vals, dtype=np.uint64))
    lo = torch.from_numpy((a & np.uint64(0xffffffff)).astype(np.int64)).to(_dev(group))
    hi = torch.from_numpy((a >> np.uint64(32)).astype(np.int64)).to(_dev(group))
    dist.all_reduce(lo, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.SUM, group=group)
    lo, hi = lo.cpu().numpy().astype(np.uint64), hi.cpu().numpy().astype(np.uint64)
    return lo + (hi << np.uint64(32))
