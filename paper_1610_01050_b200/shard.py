"""Host-side sharding logic of the multi-GPU path (no arithmetic of the method here).

c4-style batches: frames are independent -> each rank owns a contiguous frame range,
no data-path collective.
c5-style single cube (BASELINE configs[4]): the L loops are sharded over ranks and the
per-loop bitmaps are all-gathered over NCCL (2 KiB per loop at c5) before every rank votes on
its own dim-0 slab of locations (rsft_detect dim0 range).
  variant A: every rank reads the whole cube and computes the bitmaps of its loops
             (rsft_execute loop range);
  variant B: every rank folds only its dim-0 slab of the cube for all loops
             (rsft_bucketize_partial; the fold is linear in x), the partial folded spectra are
             reduce-scattered over loops (2 MiB at c5), and each rank finalizes its loops
             (rsft_finalize) -- HBM traffic per rank drops to cube/G.
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


def reduce_scatter_loops(partial, world: int, group=None):
    """Sum the slab partials [L, B_tot] over ranks and keep this rank's loop block
    [L / world, B_tot] (loop order = rank order).  NCCL: reduce_scatter_tensor; backends
    without it (gloo, CPU tests): all_reduce + slice."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return partial
    L = partial.shape[0]
    if L % world:
        raise ValueError(f"loops={L} must divide evenly over {world} ranks")
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((L // world,) + tuple(partial.shape[1:]), dtype=partial.dtype, device=partial.device)
        dist.reduce_scatter_tensor(out, partial.contiguous(), group=group)
        return out
    full = partial.clone()
    dist.all_reduce(full, group=group)
    return full[rank * L // world:(rank + 1) * L // world].contiguous()
