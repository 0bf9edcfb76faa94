"""Multi-GPU plumbing for the residual+gradient path (one process per GPU).

The path shards without a data-path exchange: collocation points (config 2),
PDE-parameter instances mu (config 3) or points x instances (config 4) are
independent; the only exchange is the sum of the per-rank [loss, dL/ds] rows
(and the hypernetwork / meta gradients).  On the GPU box that sum is done by
the context itself (an NCCL communicator attached with attach_nccl, one
ncclAllReduce per step on the context stream); allreduce_sum_ is the
torch.distributed form of the same sum (gloo in the CPU tests).
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


def attach_nccl(ctx, group=None):
    """Give a GpuContext an NCCL communicator over the torch.distributed ranks
    (lrnr_gpu_comm_init): rank 0 draws the ncclUniqueId, the process group
    broadcasts it, every rank joins.  From then on the context's gradient calls
    sum their results over the ranks themselves (include/lrnr_gpu.h, 'multi-GPU').
    Returns (world, rank)."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        raise RuntimeError("attach_nccl needs an initialised torch.distributed process group")
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    box = [ctx.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    ctx.comm_init(world, rank, box[0])
    return world, rank
