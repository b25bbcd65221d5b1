"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: frame / loop / slab sharding
and the all-gather of per-loop bitmaps before voting (BASELINE configs[4]).
The per-rank first-stage bitmaps come from the oracle (CPU), so the test checks that the
sharded pipeline reassembles exactly the single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rsft_ref as R
import synth
from paper_1610_01050_b200 import shard


def pack(c):
    """bool bucket mask -> uint32 words (bit k of word w = flat bucket 32 w + k)."""
    bits = np.asarray(c, dtype=np.uint8).ravel()
    pad = (-bits.size) % 32
    bits = np.concatenate([bits, np.zeros(pad, np.uint8)])
    return np.packbits(bits, bitorder="little").view(np.uint32).astype(np.int64).astype(np.int32)


def unpack(words, n):
    return np.unpackbits(np.asarray(words, dtype=np.int32).view(np.uint8), bitorder="little")[:n].astype(bool)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, b, L = (32, 16, 64), (4, 4, 8), 4
        p = R.Params(n=n, b=b, loops=L, p_fa=1e-3, seed=17)
        tb = R.make_tables(p)
        wl = synth.Workload("mg", n, b, L, 1e-3, 1.0, (3, 6), (5.0, 20.0), 1, data_seed=4)
        x = synth.gen_frame(wl, 0)
        lb, le = shard.loop_range(rank, world, L)
        local = torch.from_numpy(np.stack([pack(R.first_stage(x, p, tb, l).c) for l in range(lb, le)]))
        full = shard.gather_loop_bitmaps(local, world)
        cs = [unpack(full[l].numpy(), int(np.prod(b))).reshape(b) for l in range(L)]
        d0b, d0e = shard.slab_range(rank, world, n[0], n[1] * n[2])
        abar = R.accumulate(cs, p, tb)
        mine = (abar >= p.mu)[d0b:d0e]
        gathered = [None] * world
        dist.all_gather_object(gathered, (d0b, d0e, mine))
        if rank == 0:
            ref = R.rsft_run(x, p, tb)
            det = np.zeros(n, dtype=bool)
            for bb, ee, m in gathered:
                det[bb:ee] = m
            ret["ok"] = bool(np.array_equal(det, ref.detect))
            ret["bits_ok"] = all(np.array_equal(cs[l], ref.stages[l].c) for l in range(L))
            ret["frames"] = [shard.frame_range(r, world, 4096) for r in range(world)]
    finally:
        dist.destroy_process_group()


def test_two_rank_loop_shard_allgather_vote():
    world = 2
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_worker, args=(world, free_port(), ret), nprocs=world, join=True)
        assert ret["bits_ok"] and ret["ok"]
        assert ret["frames"] == [(0, 2048), (2048, 4096)]


def test_shard_ranges_partition():
    for world in (1, 2, 4, 8):
        assert [shard.loop_range(r, world, 16) for r in range(world)] == [(16 // world * r, 16 // world * (r + 1)) for r in range(world)]
        sl = [shard.slab_range(r, world, 2048, 512 * 64) for r in range(world)]
        assert sl[0][0] == 0 and sl[-1][1] == 2048 and all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        shard.loop_range(0, 3, 16)


def _worker_b(rank, world, port, ret):
    """Variant B host logic: each rank's slab-masked frame -> oracle folded spectra (the fold
    is linear in x, Eqs. z, l P:272-279) -> reduce-scatter over loops -> this rank's loop rows
    equal the unsharded frame's."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, b, L = (32, 16, 64), (4, 4, 8), 4
        p = R.Params(n=n, b=b, loops=L, p_fa=1e-3, seed=19, random_tau=True)
        tb = R.make_tables(p)
        wl = synth.Workload("mgb", n, b, L, 1e-3, 1.0, (3, 6), (5.0, 20.0), 1, data_seed=6)
        x = synth.gen_frame(wl, 0)
        d0b, d0e = shard.slab_range(rank, world, n[0], n[1] * n[2])
        xs = np.zeros_like(x)
        xs[d0b:d0e] = x[d0b:d0e]
        part = torch.from_numpy(np.stack([R.first_stage(xs, p, tb, l).fhat.ravel() for l in range(L)]))
        mine = shard.reduce_scatter_loops(part, world)
        lb, le = shard.loop_range(rank, world, L)
        full = np.stack([R.first_stage(x, p, tb, l).fhat.ravel() for l in range(lb, le)])
        err = float(np.max(np.abs(mine.numpy() - full)) / np.max(np.abs(full)))
        gathered = [None] * world
        dist.all_gather_object(gathered, err)
        if rank == 0:
            ret["err"] = max(gathered)
    finally:
        dist.destroy_process_group()


def test_two_rank_slab_partials_reduce_scatter():
    world = 2
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_worker_b, args=(world, free_port(), ret), nprocs=world, join=True)
        assert ret["err"] < 1e-12


def _worker_c64(rank, world, port, ret):
    """The complex64 message of variant B (the GPU dtype) through the one reduce_scatter_tensor
    call shard.py also issues on NCCL (float32 view), at world 1 and 2."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, bt = 8, 96
        g = torch.Generator().manual_seed(5)
        parts = [torch.complex(torch.randn(L, bt, generator=g), torch.randn(L, bt, generator=g))
                 for _ in range(world)]
        mine = shard.reduce_scatter_loops(parts[rank], world)
        lb, le = shard.loop_range(rank, world, L)
        want = sum(p.to(torch.complex128) for p in parts)[lb:le]
        assert mine.dtype == torch.complex64 and mine.shape == (L // world, bt)
        err = float((mine.to(torch.complex128) - want).abs().max())
        bits = torch.arange(2 * 3, dtype=torch.int32).reshape(2, 3) + 100 * rank
        allb = shard.gather_loop_bitmaps(bits, world)
        okg = bool(torch.equal(allb, torch.cat([torch.arange(6, dtype=torch.int32).reshape(2, 3) + 100 * r
                                                for r in range(world)])))
        gathered = [None] * world
        dist.all_gather_object(gathered, (err, okg))
        if rank == 0:
            ret["err"] = max(e for e, _ in gathered)
            ret["gather_ok"] = all(o for _, o in gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_complex64_reduce_scatter_and_gather_through_collectives(world):
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_worker_c64, args=(world, free_port(), ret), nprocs=world, join=True)
        assert ret["err"] < 1e-5 and ret["gather_ok"]


def test_no_process_group_passthrough():
    x = torch.ones(4, 3, dtype=torch.complex64)
    assert shard.reduce_scatter_loops(x) is x and shard.gather_loop_bitmaps(x) is x
