"""Multi-process plumbing for the row-sharded path (one process per GPU).

torch.distributed is used only to broadcast librac's NCCL unique id and to
reduce timings; the per-pass exchange itself (ncclAllGather of the alive
bitvector slices) happens inside librac (include/rac.h, "Multi-GPU").
"""
from __future__ import annotations

from typing import Optional

from . import rac


def nccl_unique_id(group=None) -> bytes:
    """Rank 0 creates librac's NCCL unique id; every rank receives the same bytes."""
    import torch.distributed as dist
    obj = [rac.rac_get_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != rac.RAC_NCCL_ID_BYTES:
        raise RuntimeError("bad NCCL unique id broadcast")
    return bytes(uid)


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (multi-GPU timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def create_sharded_random(n_vars: int, d: int, dens_q32: int, t_q16: int, seed: int, device: int,
                          group=None, uid: Optional[bytes] = None) -> rac.RacContext:
    """Collective rac_create_random over the ranks of `group`: rank r keeps the
    masks of variables rac_shard_range(n, world, r)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if uid is None:
        uid = nccl_unique_id(group) if world > 1 else None
    return rac.RacContext.create_random(n_vars, d, dens_q32, t_q16, seed, device=device, rank=rank, world=world,
                                        nccl_unique_id=uid)
