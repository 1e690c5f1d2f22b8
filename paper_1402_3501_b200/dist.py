"""Multi-GPU plumbing for the partitioned PLUQ: one process per GPU under torchrun.

torch.distributed is only the rendezvous here (it ships the 128-byte NCCL id from rank 0
to the others); the exchange itself is the library's own NCCL communicator
(csrc/dist.cu), created through the C ABI (ffg_dist_init), so a C++ host that never
imports torch does the same with its own id transport.
"""
from __future__ import annotations

from .ffpluq import Context, dist_partition, dist_unique_id  # noqa: F401


def share_unique_id(rank: int, make_id=dist_unique_id, group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank of the torch process group receives it."""
    import torch.distributed as tdist

    box = [make_id() if rank == 0 else None]
    tdist.broadcast_object_list(box, src=0, group=group)
    uid = box[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("dist: bad NCCL unique id received")
    return bytes(uid)


def init_from_process_group(ctx: Context, group=None, min_work: int | None = None) -> dict:
    """Join ctx to a partitioned world spanning the (initialised) torch process group."""
    import torch.distributed as tdist

    world, rank = tdist.get_world_size(group), tdist.get_rank(group)
    if world > 1:
        ctx.dist_init(world, rank, share_unique_id(rank, group=group))
    if min_work is not None:
        ctx.dist_set_min_work(min_work)
    return ctx.dist_info()


def plan(total: int, world: int, align: int = 128) -> list[tuple[int, int]]:
    """Every rank's slice of `total` (the library's partition, in rank order)."""
    return [dist_partition(total, world, r, align) for r in range(world)]
