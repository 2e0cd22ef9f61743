"""Multi-process (torchrun) plumbing for the multi-GPU count.

One process per GPU.  Every rank builds the same graph replica (no
communication), then each count runs this rank's pivot range and ONE NCCL
allreduce inside libtcb200 (tc_count_allreduce, multi.cu).  torch.distributed
is only the rendezvous: rank 0 creates the 128-byte NCCL id and the process
group carries it to the other ranks (any backend; gloo is enough).
"""
from __future__ import annotations

from . import Comm


def init_comm(device: int, group=None) -> Comm:
    """The library's NCCL communicator for this rank of the (initialised)
    torch.distributed default group."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return Comm(obj[0], world, rank, device)


def max_over_ranks(x: float, group=None) -> float:
    """Device-timed step time: the job's time is the slowest rank's (a CPU
    tensor, so any backend works)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
