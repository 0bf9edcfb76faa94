"""Multi-GPU plumbing for the residual+gradient path (one process per GPU).

The path shards without a data-path exchange: collocation points (config 2),
PDE-parameter instances mu (config 3) or points x instances (config 4) are
independent; the only exchange is the sum of the per-rank [loss, dL/ds] rows
(and the hypernetwork / meta gradients), done with one all-reduce per step over
torch.distributed (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) share of n items for `rank` (first n % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_instances(n_inst: int, world: int, rank: int) -> tuple[int, int]:
    """Instance-homogeneous sharding (configs 3/4): whole mu instances per rank."""
    return shard_range(n_inst, world, rank)


def allreduce_sum_(tensor, group=None):
    """In-place sum over ranks of a result row block (torch tensor)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def allreduce_max_(tensor, group=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.MAX, group=group)
    return tensor
