"""Multi-process plumbing for the row-sharded path (one process per GPU).

torch.distributed is used only to exchange librac's setup tokens (the NCCL
unique id, or the peer regions' CUDA IPC handles) and to reduce timings; the
per-pass exchange itself happens inside librac (include/rac.h, "Multi-GPU"):
without RAC_OPT_PEER (the library's default for world > 1) an ncclAllGather of
the alive-bitvector slices between per-pass launches; with ``peer=True``
(RAC_OPT_PEER -- what ``bench.py --gpus N`` uses unless ``--exchange nccl``)
NVLink peer stores and a cross-rank barrier inside the one persistent
enforcement kernel.
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


def connect_peers(ctx: rac.RacContext, group=None) -> None:
    """All-gather every rank's IPC handle and open the peers' regions."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    handles = [None] * world
    dist.all_gather_object(handles, ctx.peer_handle(), group=group)
    ctx.connect_peers(handles)


def create_sharded_random(n_vars: int, d: int, dens_q32: int, t_q16: int, seed: int, device: int,
                          group=None, uid: Optional[bytes] = None, peer: bool = False) -> rac.RacContext:
    """Collective rac_create_random over the ranks of `group`: rank r keeps the
    masks of variables rac_shard_range(n, world, r).  peer=True: exchange
    through peer memory (RAC_OPT_PEER; IPC handles swapped here)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if peer and world > 1:
        ctx = rac.RacContext.create_random(n_vars, d, dens_q32, t_q16, seed, device=device, rank=rank, world=world,
                                           peer=True)
        connect_peers(ctx, group)
        return ctx
    if uid is None:
        uid = nccl_unique_id(group) if world > 1 else None
    return rac.RacContext.create_random(n_vars, d, dens_q32, t_q16, seed, device=device, rank=rank, world=world,
                                        nccl_unique_id=uid)
