"""Multi-GPU plumbing over torch.distributed (one process per GPU).

The library shards the work itself (unit i of the work plan goes to rank i mod N, see
DESIGN.md §Multi-GPU) and all-reduces the counts with NCCL; this module only bootstraps the
NCCL communicator (the 128-byte ncclUniqueId travels over the torch process group) and
provides the max-over-ranks timing reduction.  Works with the nccl backend (CUDA tensors) and
with gloo (CPU tensors, used by the CPU tests)."""
from __future__ import annotations

import torch
import torch.distributed as dist


def _dev(group=None):
    backend = dist.get_backend(group)
    if backend == "nccl":
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
    """NCCL communicator of the library for this rank (collective over the group)."""
    from . import bbf
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = bbf.nccl_unique_id() if rank == 0 else None
    uid = broadcast_unique_id(uid, 0, group)
    return bbf.Comm(uid, world, rank, device)


def max_over_ranks(x: float, group=None) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks_u64(vals, group=None):
    """Exact integer sum across ranks (int64 lanes; counts < 2^63 here)."""
    t = torch.tensor([int(v) for v in vals], dtype=torch.int64, device=_dev(group))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [int(v) for v in t.cpu().tolist()]


def shard_owner(item: int, nranks: int) -> int:
    """Host mirror of the device sharding rule: work item i (T3 unit or T1 start, in plan
    order) is processed by rank i mod nranks."""
    return item % nranks
