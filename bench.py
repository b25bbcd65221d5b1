#!/usr/bin/env python
"""RSFT hot-path benchmark (BASELINE.json metric: RSFT frames/s and fused-bucketize HBM GB/s
as a fraction of the B200 peak, at 1/2/4/8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4_batched_2d|c5_cube]
                    [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...         (one rank per GPU, NCCL)

A step is one pass of the whole hot path (fold + FFT + threshold, vote + second stage, sorted index
list) over one batch of synthetic frames resident in HBM: ONE rsft_run call for fused-mode plans
(c4 / c2: k_fused2v folds and votes in one kernel; c1: k_gather1d with vote warps), rsft_execute +
rsft_detect_compact for split-mode plans (c3, c5) or with --two-calls.  Default
workload: c4 (BASELINE configs[3]: 1024x256 complex64 frames, B=32x16, L=6, P_fa=1e-6),
4096 frames per GPU (weak scaling: frames shard across GPUs, no collective in the data path).
`--workload c5_cube` runs the single 512 MiB cube with its L=16 loops sharded across ranks
and an NCCL all-gather of the per-loop bitmaps before voting.

Prints ONE JSON line on rank 0.  `--impl reference` times the fp64 CPU oracle (the only
reference this paper has: it publishes no code) on a bounded sample of the same workload.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "RSFT frames/sec and fused-bucketize HBM GB/s (% of B200 peak) at 1/2/4/8 GPUs"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(workload):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload)
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons with NVML (nvidia-smi fallback) in a thread."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- distributed
def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


# ----------------------------------------------------------------------------- reference arm
def oracle_worker(args):
    """Run the oracle on the given frames; inputs are generated before the clock starts."""
    wl_name, frame_ids = args
    from oracle import rsft_ref as R
    wl = synth.WORKLOADS[wl_name]
    op = R.Params(n=wl.n, b=wl.b, loops=wl.loops, support=wl.support, p_fa=wl.p_fa, noise_var=wl.noise_var,
                  seed=wl.sched_seed, random_tau=wl.random_tau, mu=wl.mu)
    tb = R.make_tables(op)
    xs = [synth.gen_frame(wl, f) for f in frame_ids]
    t = time.perf_counter()
    for x in xs:
        R.rsft_run(x, op, tb)
    return time.perf_counter() - t


def oracle_rate(wl, budget_s=12.0, max_cores=32):
    """Oracle frames/s on the host cores: a process pool (1 BLAS/OpenMP thread each) over a
    bounded sample of frames of the workload; rate = frames / slowest worker's oracle time.
    Returns (frames/s, cores, sample description)."""
    import multiprocessing as mp
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    cores = max(1, min(len(os.sched_getaffinity(0)), max_cores))
    one = oracle_worker((wl.name, [0]))                 # calibrate on one core
    if wl.name == "c5_cube":
        cores = 1
    per_core = max(1, int(budget_s / (2.0 * max(one, 1e-3))))
    nframes = per_core * cores
    chunks = [(wl.name, list(range(i, nframes, cores))) for i in range(cores)]
    if cores == 1:
        el = oracle_worker(chunks[0])
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(cores) as pool:
            el = max(pool.map(oracle_worker, chunks))
    return nframes / el, cores, (f"{nframes} frames of {wl.name}: oracle rsft_run (fp64, literal Alg. 1), "
                                 f"{cores} processes x 1 thread, input generation untimed"), one


def ref_config(wl, a):
    """Same config dict as the GPU arm's line for this workload (bench.py workload_config)."""
    if wl.name == "c5_cube":
        return workload_config(wl, 1, variant=a.c5_variant if a.gpus > 1 else "A", world=a.gpus)
    cfg = workload_config(wl, a.frames or wl.batch)
    cfg["mode"] = "fused" if len(wl.n) <= 2 else "split"
    return cfg


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    wl = synth.WORKLOADS[a.workload]
    rates = []
    sample = None
    cores = 1
    steps = max(1, a.steps)
    budget = max(2.0, min(20.0, 150.0 / steps))         # whole run within a few minutes
    ones = []
    for _ in range(steps):
        r, cores, sample, one = oracle_rate(wl, budget_s=budget)
        rates.append(r)
        ones.append(one)
    value = float(statistics.median(rates))
    frames_per_step = wl.batch
    unit = "cubes/s" if wl.name == "c5_cube" else "frames/s"
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": unit, "n_gpus": a.gpus,
        "steps": steps, "warmup": a.warmup, "ms_per_step": 1000.0 * frames_per_step / value,
        "higher_is_better": True, "scaling": "strong" if wl.name == "c5_cube" else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Eq. sig_model frames)",
        "config": ref_config(wl, a),
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "oracle", "sample": sample,
                         "one_core_s_per_frame": statistics.median(ones)},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def workload_config(wl, frames, mode=None, variant=None, world=1):
    """The `config` dict of a bench line; identical in both arms (ours / reference)."""
    cfg = {"workload": wl.name, "frames_per_gpu": frames, "n": list(wl.n), "b": list(wl.b), "loops": wl.loops,
           "p_fa": wl.p_fa, "mu": wl.mu or wl.loops}
    if wl.name == "c5_cube":
        cfg["variant"] = variant
        cfg["l2"] = "cube 512 MiB >> 126 MB L2 (no flush needed)"
    else:
        cfg["l2"] = f"inputs {frames * wl.ntot * 8 / 2**30:.1f} GiB per GPU >> 126 MB L2 (no flush needed)"
        cfg["parallelism"] = "frames sharded over the GPUs (weak scaling), no data-path collective"
    return cfg


def step_stats(step_ms):
    s = sorted(step_ms)
    p90 = s[min(len(s) - 1, int(math.ceil(0.9 * len(s))) - 1)]
    return {"median": statistics.median(s), "p90": p90, "min": s[0], "max": s[-1]}


def digest(*tensors):
    """sha1 over the bytes of device tensors (run-to-run / collective-vs-not bit identity)."""
    import hashlib
    h = hashlib.sha1()
    for t in tensors:
        h.update(t.contiguous().view(-1).view(__import__("torch").uint8).cpu().numpy().tobytes())
    return h.hexdigest()[:16]


def init_dist(a):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if a.gpus != world:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world} (launch with torchrun "
                         f"--nproc-per-node {a.gpus}, or without WORLD_SIZE to self-launch)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or a.force_collectives:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
    return rank, world, local, dev, dist.is_initialized()


def timed_steps(a, step, stream, local, pg):
    """W warm-up steps, then K timed steps between barrier + synchronize on both sides.
    Returns (elapsed ms max over ranks, per-step ms, per-step (k1 begin, k1 end) events,
    launches, clocks)."""
    import torch
    import torch.distributed as dist
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(a.steps)]
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    if pg:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    launches = 0
    for k in range(a.steps):
        marks[k].record(stream)
        launches += step(ev[k])
    marks[-1].record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if pg:
        dist.barrier()
    el = torch.tensor([marks[0].elapsed_time(marks[-1])], device="cuda")
    if pg:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    per_step = [marks[k].elapsed_time(marks[k + 1]) for k in range(a.steps)]
    return float(el.item()), per_step, ev, launches, clocks


def main_gpu(a):
    import torch
    import torch.distributed as dist
    from paper_1610_01050_b200 import rsft as B

    rank, world, local, dev, pg = init_dist(a)
    wl = synth.WORKLOADS[a.workload]
    stream = torch.cuda.current_stream()

    if a.bartlett:
        return bench_bartlett(a, wl, rank, world, dev)
    if a.segments:
        return bench_segments(a, wl, rank, world, dev)
    if wl.name == "c5_cube":
        return bench_c5(a, wl, rank, world, dev, pg)

    frames = a.frames or wl.batch
    plan = B.Plan(wl.n, wl.b, wl.loops, support=wl.support, p_fa=wl.p_fa, noise_var=wl.noise_var,
                  seed=wl.sched_seed, random_tau=wl.random_tau, mu=wl.mu, max_batch=frames).bind()
    pool = min(a.pool, frames)
    base = torch.from_numpy(synth.gen_batch(wl, range(rank * pool, rank * pool + pool)))
    x = torch.empty((frames,) + tuple(wl.n), dtype=torch.complex64, device=dev)
    base_d = base.to(dev)
    for f0 in range(0, frames, pool):                      # tile the pool on the device
        x[f0:f0 + pool].copy_(base_d[:frames - f0])
    del base_d
    bm = plan.new_bitmaps(frames)
    det = torch.empty((frames, plan.detect_words), dtype=torch.int32, device=dev)
    cap = frames * 4096
    idx = torch.empty(cap, dtype=torch.int64, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)

    # fused-mode plans: rsft_run is ONE fold kernel that also votes (D = 1 gather form, D = 2
    # warp-specialised k_fused2v) + the scan / index writer; split-mode plans: the fold, outer-FFT
    # and vote kernels, timed as two ABI calls so that the fold is the "dominant kernel"
    use_run = a.run or (plan.mode == 1 and not a.two_calls)

    def step(events=None):
        if use_run:
            # one rsft_run call (D = 1 gather plans: fold + vote in one kernel); the "dominant
            # kernel" events then bracket the whole call (conservative)
            if events is not None:
                events[0].record(stream)
            plan.run(x, cap, bitmaps=bm, detect=det, idx=idx, count=cnt)
            if events is not None:
                events[1].record(stream)
            return plan.last_launch_count()
        # == rsft_run (execute + detect_compact), as two ABI calls so that the fused
        # fold/FFT/threshold kernel can be timed alone on the launching stream
        if events is not None:
            events[0].record(stream)
        plan.execute(x, bitmaps=bm)
        n = plan.last_launch_count()
        if events is not None:
            events[1].record(stream)
        plan.detect_compact(bm, cap, detect=det, idx=idx, count=cnt)
        return n + plan.last_launch_count()

    elapsed_ms, per_step, ev, launches, clocks = timed_steps(a, step, stream, local, pg)
    k1_ms = [e[0].elapsed_time(e[1]) for e in ev]
    detections = int(cnt.item())
    dig = digest(bm, det, idx[:min(detections, cap)])

    # e2e through the C ABI on HOST buffers (H2D copy + kernels + D2H of count and indices)
    e2e = None
    if not a.no_e2e:
        hpin = torch.empty((frames,) + tuple(wl.n), dtype=torch.complex64, pin_memory=True)
        for f0 in range(0, frames, pool):
            hpin[f0:f0 + pool].copy_(base[:frames - f0])
        scratch = torch.empty(plan.host_scratch_bytes(frames, cap), dtype=torch.uint8, device=dev)
        plan.run_host(hpin, cap, scratch)
        e_steps = max(1, min(a.steps, 5))
        if pg:
            dist.barrier()
        tt0, tt1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        tt0.record(stream)
        nidx = 0
        for _ in range(e_steps):
            _, c = plan.run_host(hpin, cap, scratch)
            nidx = min(c, cap)
        tt1.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([tt0.elapsed_time(tt1) / e_steps], device=dev)
        if pg:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": world * frames / (float(e_ms.item()) / 1000.0), "unit": "frames/s",
               "h2d_bytes_per_step": int(hpin.numel() * 8), "d2h_bytes_per_step": int(8 + 8 * nidx)}
        del scratch, hpin

    ranks = None
    if pg:          # report gather (outside the timed region): per-rank detections and digests
        ranks = [None] * world
        dist.all_gather_object(ranks, {"rank": rank, "detections": detections, "digest": dig,
                                       "ms": elapsed_ms})
    if rank != 0:
        dist.destroy_process_group()
        return 0

    # roofline of the dominant kernel (fused fold + FFT + threshold, one launch per step):
    # algorithmic bytes = x read once + first-stage bitmaps written
    peak, peak_src = load_peaks()
    k1_avg = statistics.mean(k1_ms)
    algo_bytes = frames * (8 * plan.ntot + plan.loops * plan.bitmap_words * 4)
    if use_run:     # the whole call also writes the detection words (N/8 B per frame, §8(d)) + the index list
        algo_bytes += frames * plan.detect_words * 4 + 8 * min(detections, cap)
    achieved = algo_bytes / (k1_avg / 1000.0) / 1e9
    step_ms = elapsed_ms / a.steps
    value = world * frames / (step_ms / 1000.0)
    cpu = None
    if not a.no_cpu:
        cpu = cpu_baseline(wl, a.cpu_budget)
    cfg = workload_config(wl, frames)
    cfg["mode"] = {1: "fused", 2: "split"}.get(plan.mode, plan.mode)
    cfg["step_call"] = ("rsft_run (one call; roofline times the whole call)" if use_run
                        else "rsft_execute + rsft_detect_compact (roofline times rsft_execute)")
    out = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": step_ms, "step_ms": step_stats(per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic: {pool} distinct seeded Eq. sig_model frames per GPU tiled to {frames}",
        "config": cfg,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": load_traffic(wl.name),
                     "kernel": fold_kernel_label(plan, wl, use_run) + (" [whole rsft_run call]" if use_run else ""),
                     "algorithmic_bytes_per_launch": algo_bytes,
                     "avg_launch_ms": k1_avg, "share_of_step": k1_avg / step_ms, "peak_source": peak_src},
        "gpu_launches": launches,
        "clocks": clocks,
        "detections_per_step": detections,
        "digest": dig,
        "collectives": {"process_group": pg, "backend": "nccl" if pg else None, "ranks": ranks},
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(out), flush=True)
    if pg:
        dist.destroy_process_group()
    return 0


def fold_kernel_label(plan, wl, run=False):
    """The first-stage kernel(s) rsft_execute (run: rsft_run) launches for this plan (librsft's
    dispatch rules)."""
    if plan.mode == 2:
        mma = (len(wl.n) == 3 and wl.n[2] == 64 and not os.environ.get("RSFT_NO_MMA"))
        return ("k_split_mma (3xTF32 tcgen05)" if mma else "k_split_fold") + " + k_split_fft (fold + outer FFT + threshold)"
    w = (wl.support[0] if wl.support else 0) or wl.n[0]
    if len(wl.n) == 1 and w % 32 == 0 and w <= 1024 and not os.environ.get("RSFT_NO_GATHER1D"):
        return "k_gather1d (gather-form fold + FFT + threshold)"
    if run and len(wl.n) == 2 and max(wl.loops, 1) <= 8 and wl.b[0] <= 32 and wl.b[1] in (8, 16, 32) \
            and wl.n[1] in (128, 256) and wl.n[0] <= 1024 and not os.environ.get("RSFT_NO_FUSED2V"):
        return ("k_fused2v (fold warps + FFT/threshold/vote warps) + scan / index writer "
                "(k_region_scan_write for <= 8192 frames, else k_scan_tiles/k_scan_apply + k_region_write)")
    return "k_fused (pre-window+permute+flat window+fold+FFT+threshold)"


def cpu_baseline(wl, budget):
    r, cores, sample, one = oracle_rate(wl, budget_s=budget)
    return {"value": r, "unit": "frames/s", "cores": cores, "kind": "oracle", "sample": sample,
            "one_core_s_per_frame": one}


def bench_c5(a, wl, rank, world, dev, pg):
    """Single 512 MiB cube, L=16 loops sharded over ranks, NCCL all-gather of the per-loop
    bitmaps (2 KiB/loop), then voting on this rank's dim-0 slab (BASELINE configs[4]).
    Variant B (default): each rank folds only its dim-0 slab for all loops
    (rsft_bucketize_partial), the partial folded spectra are reduce-scattered over loops
    (NCCL), each rank finalizes its loops (rsft_finalize).  Variant A: each rank reads the
    whole cube for its loops (rsft_execute loop range).  Without a process group (one GPU,
    no --force-collectives) variant B's collectives are identities: B == A's computation
    is then run as A (rsft_execute), and the line says so."""
    import torch
    import torch.distributed as dist
    from paper_1610_01050_b200 import rsft as B
    from paper_1610_01050_b200 import shard

    stream = torch.cuda.current_stream()
    plan = B.Plan(wl.n, wl.b, wl.loops, p_fa=wl.p_fa, noise_var=wl.noise_var, seed=wl.sched_seed,
                  mu=wl.mu, max_batch=1).bind()
    L = wl.loops
    lb, le = shard.loop_range(rank, world, L)
    n0 = wl.n[0]
    d0b, d0e = shard.slab_range(rank, world, n0, plan.ntot // n0)
    hx = synth.gen_batch(wl, [0])
    variant = a.c5_variant
    if variant == "B" and not pg:
        variant = "A"
    if variant == "B":
        x = torch.from_numpy(np.ascontiguousarray(hx[0, d0b:d0e])).to(dev)     # this rank's slab only
        partial = torch.empty((L, plan.btot), dtype=torch.complex64, device=dev)
    else:
        x = torch.from_numpy(hx).to(dev)
    del hx
    mine = plan.new_bitmaps(1, le - lb)
    slab_words = (d0e - d0b) * (plan.ntot // n0) // 32
    det = torch.empty((1, slab_words), dtype=torch.int32, device=dev)
    keep = {}

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        if variant == "B":
            plan.bucketize_partial(x, d0b, partial=partial)
            n = plan.last_launch_count()
            folded = shard.reduce_scatter_loops(partial, world)
            plan.finalize(folded, loop_begin=lb, loop_end=le, bitmaps=mine[0])
            n += plan.last_launch_count()
        else:
            plan.execute(x, loop_begin=lb, loop_end=le, bitmaps=mine)
            n = plan.last_launch_count()
        if ev is not None:
            ev[1].record(stream)
        src = shard.gather_loop_bitmaps(mine[0], world).reshape(1, L, plan.bitmap_words)
        keep["src"] = src
        plan.detect(src, dim0=(d0b, d0e), detect=det)
        n += plan.last_launch_count()
        return n

    elapsed_ms, per_step, ev, launches, clocks = timed_steps(a, step, stream, int(os.environ.get("LOCAL_RANK", 0)), pg)
    dig = digest(keep["src"], det)
    ranks = None
    if pg:
        ranks = [None] * world
        dist.all_gather_object(ranks, {"rank": rank, "loops": [lb, le], "slab": [d0b, d0e], "digest": dig,
                                       "detections": int(B.bitmap_to_bool(det.cpu().numpy().ravel(), slab_words * 32).sum())})
    if rank != 0:
        dist.destroy_process_group()
        return 0
    step_ms = elapsed_ms / a.steps
    k1 = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    peak, peak_src = load_peaks()
    cube_bytes = 8 * plan.ntot
    algo = (cube_bytes // world if variant == "B" else cube_bytes) + (le - lb) * plan.bitmap_words * 4
    cfg = workload_config(wl, 1, variant=variant, world=world)
    cfg["parallelism"] = (f"dim-0 slabs over {world} GPU(s), partial folds reduce-scattered over loops "
                          f"(NCCL), loops finalized per rank, NCCL all-gather of bitmaps"
                          if variant == "B" else
                          f"loops sharded {world} way(s)" + (" + NCCL all-gather of bitmaps" if pg else
                                                               " (one GPU, no process group: no collective)"))
    mma = not os.environ.get("RSFT_NO_MMA")
    out = {
        "metric": METRIC, "value": 1000.0 / step_ms, "unit": "cubes/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": step_ms, "step_ms": step_stats(per_step),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (fold: 3xTF32 tcgen05, ~2^-20 rel.)" if mma else "f32",
        "data": "synthetic: 1 seeded Eq. sig_model cube",
        "config": cfg,
        "roofline": {"bound": "hbm", "achieved": algo / (k1 / 1000.0) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": algo / (k1 / 1000.0) / 1e9 / peak, "traffic": load_traffic(wl.name),
                     "kernel": ("k_split_mma (3xTF32 tcgen05)" if mma else "k_split_fold")
                               + " + k_split_fft (first stage of this rank)",
                     "algorithmic_bytes_per_launch": algo, "avg_launch_ms": k1,
                     "share_of_step": k1 / step_ms, "peak_source": peak_src},
        "gpu_launches": launches, "clocks": clocks, "digest": dig,
        "collectives": {"process_group": pg, "backend": "nccl" if pg else None, "ranks": ranks},
        "cpu_baseline": None, "e2e": None,
    }
    print(json.dumps(out), flush=True)
    if pg:
        dist.destroy_process_group()
    return 0


def bench_bartlett(a, wl, rank, world, dev):
    """Bartlett baseline (Alg. 2, App. A) on the workload's frame shape, batched: each frame is
    T = L segments (the paper's comparison of Tables I-II: T segments vs T RSFT iterations);
    one rsft_bartlett call per step over `frames` frames, CUDA events; reported beside the
    RSFT line, not as the headline."""
    import torch
    from paper_1610_01050_b200 import rsft as B
    stream = torch.cuda.current_stream()
    T = wl.loops
    per_frame = T * int(np.prod(wl.n)) * 8
    frames = a.frames or max(1, min(512, (4 << 30) // per_frame))
    plan = B.Plan(wl.n, wl.b, wl.loops, p_fa=wl.p_fa, noise_var=wl.noise_var, seed=wl.sched_seed).bind()
    pool = min(frames, 16)
    base = torch.from_numpy(synth.gen_batch(wl, range(pool * T)).reshape((pool, T) + tuple(wl.n))).to(dev)
    reps = (frames + pool - 1) // pool
    xs = base.repeat((reps,) + (1,) * (base.dim() - 1))[:frames].contiguous()
    g = plan.bartlett_threshold(T, wl.p_fa)
    power = torch.empty((frames,) + tuple(wl.n), dtype=torch.float32, device=dev)
    det = torch.empty((frames, plan.detect_words), dtype=torch.int32, device=dev)
    scratch = (torch.empty((frames, T) + tuple(wl.n), dtype=torch.complex64, device=dev)
               if int(np.prod(wl.n)) > 8192 else None)
    for _ in range(a.warmup):
        plan.bartlett(xs, gamma=g, power=power, detect=det, scratch=scratch)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    t0.record(stream)
    for _ in range(a.steps):
        plan.bartlett(xs, gamma=g, power=power, detect=det, scratch=scratch)
        launches += plan.last_launch_count()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.steps
    ntot = int(np.prod(wl.n))
    algo = frames * (T * ntot * 8 + ntot * 4)                 # segments read once, power written once
    passes = 1 if ntot <= 8192 else 3                         # two-pass: + scratch write + re-read
    moved = frames * (passes * T * ntot * 8 + ntot * 4)
    peak, _ = load_peaks()
    out = {"metric": "Bartlett baseline (Alg. 2) frames/s, T = L segments per frame", "value": frames * 1000.0 / ms,
           "unit": "frames/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
           "higher_is_better": True, "dtype": "f32", "data": "synthetic (seeded Eq. sig_model segments)",
           "config": {"workload": wl.name, "n": list(wl.n), "segments": T, "frames": frames, "impl": "bartlett"},
           "hbm": {"algorithmic_gbs": algo / (ms / 1e3) / 1e9, "design_bytes_gbs": moved / (ms / 1e3) / 1e9,
                   "design_frac": moved / (ms / 1e3) / 1e9 / peak, "passes_over_input": passes},
           "gpu_launches": launches}
    print(json.dumps(out), flush=True)
    return 0


def bench_segments(a, wl, rank, world, dev):
    """RSFT in segment mode: frames of T = L segments, loop l folds segment l
    (rsft_execute_segments + rsft_detect_compact); the like-for-like partner of the Bartlett
    baseline line (both read T x N samples per frame)."""
    import torch
    from paper_1610_01050_b200 import rsft as B
    stream = torch.cuda.current_stream()
    T = wl.loops
    per_frame = T * int(np.prod(wl.n)) * 8
    frames = a.frames or max(1, min(4096, (4 << 30) // per_frame))
    plan = B.Plan(wl.n, wl.b, wl.loops, support=wl.support, p_fa=wl.p_fa, noise_var=wl.noise_var,
                  seed=wl.sched_seed, random_tau=wl.random_tau, mu=wl.mu, max_batch=frames).bind()
    pool = min(frames, 16)
    base = torch.from_numpy(synth.gen_batch(wl, range(pool * T)).reshape((pool, T) + tuple(wl.n))).to(dev)
    reps = (frames + pool - 1) // pool
    xs = base.repeat((reps,) + (1,) * (base.dim() - 1))[:frames].contiguous()
    bm = plan.new_bitmaps(frames)
    cap = frames * 4096
    det = torch.empty((frames, plan.detect_words), dtype=torch.int32, device=dev)
    idx = torch.empty(cap, dtype=torch.int64, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)

    def step():
        plan.execute_segments(xs, bitmaps=bm)
        n = plan.last_launch_count()
        plan.detect_compact(bm, cap, detect=det, idx=idx, count=cnt)
        return n + plan.last_launch_count()

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    t0.record(stream)
    for _ in range(a.steps):
        launches += step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.steps
    out = {"metric": "RSFT segment mode frames/s, T = L segments per frame", "value": frames * 1000.0 / ms,
           "unit": "frames/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
           "higher_is_better": True, "dtype": "f32", "data": "synthetic (seeded Eq. sig_model segments)",
           "config": {"workload": wl.name, "n": list(wl.n), "segments": T, "frames": frames, "impl": "rsft-segments",
                      "hbm_read_gbs": frames * per_frame / (ms / 1000.0) / 1e9},
           "gpu_launches": launches}
    print(json.dumps(out), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c4_batched_2d", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=0, help="frames per GPU (default: the workload's batch)")
    ap.add_argument("--pool", type=int, default=256, help="distinct seeded frames per GPU (tiled)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--bartlett", action="store_true", help="time the Bartlett baseline (Alg. 2) instead")
    ap.add_argument("--segments", action="store_true", help="time the RSFT in segment mode (P:204)")
    ap.add_argument("--c5-variant", default="B", choices=["A", "B"], help="c5 multi-GPU scheme (DESIGN.md §8)")
    ap.add_argument("--run", action="store_true",
                    help="issue each step as ONE rsft_run call (the default for fused-mode plans, where the fold "
                         "kernel also votes); the roofline then times the whole call")
    ap.add_argument("--two-calls", action="store_true",
                    help="issue each step as rsft_execute + rsft_detect_compact (the fold kernel timed alone)")
    ap.add_argument("--force-collectives", action="store_true",
                    help="initialise an NCCL process group even with one rank, so the multi-GPU code path "
                         "(barriers, max-over-ranks timing, c5 reduce-scatter + all-gather) runs on a 1-GPU lease")
    a = ap.parse_args()
    if a.warmup < 3:
        a.warmup = 3
    if a.impl == "reference":
        return run_reference(a)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(a.gpus)
    return main_gpu(a)


def relaunch(n):
    """`python bench.py --gpus N` without torchrun: re-exec under torch.distributed.run with N
    ranks (one per GPU, rendezvous on 127.0.0.1) so --gpus N always measures N GPUs."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


if __name__ == "__main__":
    sys.exit(main())
