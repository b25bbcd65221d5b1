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


def _world(group):
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 0
    return dist.get_world_size(group)


def gather_loop_bitmaps(local, world: int = None, group=None):
    """All-gather per-loop bitmaps.  local: int32 tensor [loops_per_rank, words].
    Returns [world * loops_per_rank, words] in loop order (rank-major = loop order because
    each rank owns a contiguous loop range).  Runs the collective whenever a process group is
    initialised -- also with ONE rank (bench --force-collectives), so the NCCL path is the
    one measured on a 1-GPU lease; without a process group the input is returned."""
    import torch
    import torch.distributed as dist
    w = _world(group)
    if w == 0:
        return local
    if world is not None and world != w:
        raise ValueError(f"world={world} but the process group has {w} ranks")
    out = torch.empty((w * local.shape[0], local.shape[1]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


def reduce_scatter_loops(partial, world: int = None, group=None):
    """Sum the slab partials [L, ...] (complex64) over ranks and keep this rank's loop block
    [L / world, ...] (loop order = rank order) with ONE reduce_scatter_tensor.
    NCCL has no complex dtype and torch's reduce_scatter_tensor does not convert complex
    tensors, so the message is sent as its float32 view (torch.view_as_real: re/im summed
    independently, which is the complex sum).  The same call runs on gloo (CPU tests) and
    NCCL.  Without a process group the input is returned."""
    import torch
    import torch.distributed as dist
    w = _world(group)
    if w == 0:
        return partial
    if world is not None and world != w:
        raise ValueError(f"world={world} but the process group has {w} ranks")
    L = partial.shape[0]
    if L % w:
        raise ValueError(f"loops={L} must divide evenly over {w} ranks")
    src = partial.contiguous()
    out = torch.empty((L // w,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    if src.is_complex():
        dist.reduce_scatter_tensor(torch.view_as_real(out), torch.view_as_real(src), group=group)
    else:
        dist.reduce_scatter_tensor(out, src, group=group)
    return out
