"""Host-side sharding logic of the multi-GPU path (no arithmetic of the method here).

c4-style batches: frames are independent -> each rank owns a contiguous frame range,
no data-path collective.
c5-style single cube (BASELINE configs[4]): the L loops are sharded over ranks, each rank
computes the first-stage bitmaps of its loops (rsft_execute loop range), the per-loop
bitmaps are all-gathered over NCCL (2 KiB per loop at c5), then every rank votes on its own
dim-0 slab of locations (rsft_detect dim0 range).
"""
from __future__ import annotations


def frame_range(rank: int, world: int, frames: int):
    """Contiguous frame range [b, e) of `rank` when `frames` are split over `world` ranks."""
    b = rank * frames // world
    e = (rank + 1) * frames // world
    return b, e


def loop_range(rank: int, world: int, loops: int):
    """Loops [b, e) computed by `rank` (requires world | loops so the all-gather is even)."""
    if loops % world:
        raise ValueError(f"loops={loops} must divide evenly over {world} ranks")
    return rank * loops // world, (rank + 1) * loops // world


def slab_range(rank: int, world: int, n0: int, locs_per_row: int):
    """Dim-0 slab [b, e) voted by `rank`; slab sizes keep whole 32-bit detection words."""
    b = rank * n0 // world
    e = (rank + 1) * n0 // world
    if ((e - b) * locs_per_row) % 32:
        raise ValueError("slab must hold a multiple of 32 locations")
    return b, e


def gather_loop_bitmaps(local, world: int, group=None):
    """All-gather per-loop bitmaps.  local: int32 tensor [loops_per_rank, words] (contiguous).
    Returns [world * loops_per_rank, words] in loop order (rank-major = loop order because
    each rank owns a contiguous loop range)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    out = torch.empty((world * local.shape[0], local.shape[1]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out
