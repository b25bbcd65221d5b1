"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs
and the same seeded (sigma, tau).  Buckets within 1e-4 relative (noise-std floor), first-stage
bits exact outside the 1e-3 near-threshold band, detection sets inside the ambiguity envelope,
vote counts inside [abar_min, abar_max], index lists exact (BASELINE north_star)."""
import zlib

import numpy as np
import pytest

from oracle import rsft_ref as R
import synth
from gpu_helpers import check_frame, check_index_list, gpu_run, make_plan, oracle_params

pytestmark = pytest.mark.gpu


def frames(wl, batch, start=0):
    return synth.gen_batch(wl, range(start, start + batch))


def run_case(op, x, mode="auto", check=None, loops=None):
    import torch
    torch.cuda.init()
    plan = make_plan(op, max_batch=x.shape[0], mode=mode).bind()
    sig, _, tau = plan.schedule()
    tb = R.make_tables(op)
    np.testing.assert_array_equal(sig, tb.sigma)
    np.testing.assert_array_equal(tau, tb.tau)
    res = gpu_run(plan, x)
    check_index_list(res, plan.ntot, x.shape[0])
    reps = []
    for f in (range(x.shape[0]) if check is None else check):
        reps.append(check_frame(res, f, x[f], op, tb))
    return plan, res, reps


# ----------------------------------------------------------------------------- CI sizes
CASES = [
    # name, n, b, loops, extra oracle params, batch, mode
    ("1d_w256_tau", (1024,), (32,), 5, dict(support=(256,), random_tau=True, p_fa=1e-3), 3, "fused"),
    ("1d_b64_full", (2048,), (64,), 3, dict(p_fa=1e-3), 2, "fused"),
    # D = 1 gather-form fold (k_gather1d): W <= 1024, taps in registers
    ("1d_g_c1like", (4096,), (64,), 8, dict(support=(512,), random_tau=True, p_fa=1e-3), 5, "fused"),
    ("1d_g_b16_w128", (2048,), (16,), 6, dict(support=(128,), random_tau=True, p_fa=1e-3), 3, "fused"),
    ("1d_g_b8_w384", (1024,), (8,), 3, dict(support=(384,), p_fa=1e-3), 3, "fused"),
    ("1d_g_L20_w1024", (8192,), (64,), 20, dict(support=(1024,), random_tau=True, p_fa=1e-3, mu=15), 2, "fused"),
    ("1d_g_B_eq_N", (64,), (64,), 4, dict(p_fa=1e-2), 3, "fused"),
    ("1d_g_B1", (256,), (1,), 3, dict(p_fa=1e-2), 3, "fused"),
    ("1d_g_b32_dense", (512,), (32,), 7, dict(p_fa=1e-3, random_tau=True), 4, "fused"),
    # D = 1 with B = 128 / 256 (4 / 8 buckets per lane; P:558 B_opt = 128, Figs. ROC_K / ROC_CO
    # B = 256): full support, short support, two loops per warp, B = N, > 32 loops (two passes)
    ("1d_B128_full", (1024,), (128,), 6, dict(p_fa=1e-3, random_tau=True), 3, "fused"),
    ("1d_B256_full", (1024,), (256,), 5, dict(p_fa=1e-3), 2, "fused"),
    ("1d_B128_w512", (4096,), (128,), 8, dict(support=(512,), random_tau=True, p_fa=1e-3, mu=6), 3, "fused"),
    ("1d_B256_w512_L20", (2048,), (256,), 20, dict(support=(512,), p_fa=1e-2, mu=14), 2, "fused"),
    ("1d_B256_eq_N", (256,), (256,), 3, dict(p_fa=1e-2), 2, "fused"),
    ("1d_B128_L40", (1024,), (128,), 40, dict(support=(256,), p_fa=1e-2, mu=30, random_tau=True), 2, "fused"),
    # D = 1 warp-per-frame vote (k_vote1d): candidate mode (mu near L) and dense mode (mu small)
    ("1d_v_mu_half", (4096,), (64,), 8, dict(support=(512,), random_tau=True, p_fa=1e-2, mu=4), 6, "fused"),
    ("1d_v_mu1", (2048,), (32,), 4, dict(support=(256,), p_fa=1e-2, mu=1), 5, "fused"),
    ("1d_v_dense_pfa", (1024,), (64,), 6, dict(support=(512,), p_fa=0.3, mu=5), 4, "fused"),
    ("2d_fused", (128, 128), (16, 8), 6, dict(p_fa=1e-4, random_tau=True), 5, "fused"),
    ("2d_fused_mu", (128, 64), (8, 16), 7, dict(p_fa=1e-3, mu=4), 4, "fused"),
    ("2d_fused_mu1", (128, 64), (8, 16), 3, dict(p_fa=1e-3, mu=1), 2, "fused"),
    ("3d_split_mu1", (32, 32, 64), (4, 8, 8), 3, dict(p_fa=1e-3, mu=1), 1, "split"),
    ("3d_split_nlast32_B32", (16, 64, 32), (4, 8, 32), 4, dict(p_fa=1e-3), 1, "split"),
    ("2d_split_rpw1", (128, 64), (16, 16), 6, dict(p_fa=1e-4), 2, "split"),
    ("2d_split_rpw2", (256, 32), (16, 8), 4, dict(p_fa=1e-4, random_tau=True), 2, "split"),
    ("3d_split", (64, 32, 32), (8, 4, 8), 8, dict(p_fa=1e-5, random_tau=True), 2, "split"),
    ("3d_split_L12", (32, 16, 64), (4, 4, 8), 12, dict(p_fa=1e-4, mu=9), 1, "split"),
    ("3d_L1", (16, 16, 64), (4, 8, 16), 1, dict(p_fa=1e-3), 1, "split"),
    ("3d_c3like_mu", (64, 128, 32), (8, 16, 8), 8, dict(p_fa=1e-2, mu=5, random_tau=True), 3, "split"),
    ("3d_c3like_or", (32, 64, 32), (4, 8, 8), 4, dict(p_fa=1e-3, mu=1), 2, "split"),
    # warp-form outer FFT (B_0 = 32, B_1 in {8, 16})
    ("3d_w32_b16", (64, 32, 32), (32, 16, 8), 6, dict(p_fa=1e-3, random_tau=True), 2, "split"),
    ("3d_w32_b8_mu", (128, 64, 32), (32, 8, 4), 5, dict(p_fa=1e-2, mu=3), 2, "split"),
    # two-warp outer FFT (B_0 = 64, B_1 in {8, 16, 32}; c5's outer grid is 64 x 32)
    ("3d_w64_b32", (128, 64, 32), (64, 32, 8), 6, dict(p_fa=1e-3, random_tau=True), 2, "split"),
    ("3d_w64_b16_mma", (64, 256, 64), (64, 16, 8), 8, dict(p_fa=1e-3), 1, "split"),
    ("3d_w64_b8_mu", (64, 32, 64), (64, 8, 8), 5, dict(p_fa=1e-2, mu=3, random_tau=True), 2, "split"),
    # more than 32 loops (up to 63, the paper's T = 50 design point P:640): several fold passes
    ("2d_L40", (128, 64), (16, 8), 40, dict(p_fa=1e-2, mu=30, random_tau=True), 2, "fused"),
    ("1d_L50_w256", (1024,), (32,), 50, dict(support=(256,), p_fa=1e-2, mu=40), 2, "fused"),
    ("3d_L36", (16, 32, 32), (4, 8, 8), 36, dict(p_fa=1e-2, mu=20), 2, "split"),
    ("2d_B_eq_N_dim0", (64, 128), (64, 8), 3, dict(p_fa=1e-3), 3, "fused"),
    ("2d_B1_dim0", (64, 128), (1, 16), 3, dict(p_fa=1e-3), 2, "fused"),
    ("2d_Blast1", (64, 64), (16, 1), 3, dict(p_fa=1e-3), 2, "fused"),
    ("2d_Blast1_split", (64, 64), (16, 1), 3, dict(p_fa=1e-3), 2, "split"),
    ("2d_rect_cheb40", (128, 128), (16, 16), 4, dict(prewin="cheb", prewin_param=40.0, p_fa=1e-4), 2, "fused"),
    # D = 2 votes at N_1 = 128 / 256: c4's shape, dense spectra, every vote mode, B_0 = 64,
    # B_1 = 64 (two-word bucket rows)
    ("2d_v_c4like", (1024, 256), (32, 16), 6, dict(p_fa=1e-3), 2, "fused"),
    ("2d_v_dense_mu", (256, 256), (16, 16), 10, dict(p_fa=0.2, mu=3), 2, "fused"),
    ("2d_v_mu1_dense", (512, 128), (16, 8), 4, dict(p_fa=0.05, mu=1), 2, "fused"),
    ("2d_v_L12_B64", (256, 256), (64, 8), 12, dict(p_fa=1e-2, mu=9, random_tau=True), 2, "fused"),
    ("2d_v_B1_64", (128, 256), (8, 64), 5, dict(p_fa=1e-2), 2, "fused"),
    # k_fused2v corners (rsft_run on D = 2 fused plans): B_1 = 32 (one bucket row per bitmap word),
    # B_0 = 4 (lanes duplicate rows), L = 7 < LP = 8 with mu = 5 (bit-sliced counts)
    ("2d_f2v_b1_32", (128, 256), (8, 32), 5, dict(p_fa=1e-3, random_tau=True), 3, "fused"),
    ("2d_f2v_b0_4_mu", (64, 128), (4, 8), 7, dict(p_fa=1e-2, mu=5), 3, "fused"),
    ("3d_B_eq_N_last", (16, 32, 32), (4, 8, 32), 3, dict(p_fa=1e-3), 1, "split"),
    # tensor-core split fold (k_split_mma: N_last = 64, A_1 % 16 == 0, L <= 16, L % 4 == 0)
    ("3d_mma_A16", (16, 128, 64), (4, 8, 8), 8, dict(p_fa=1e-3, random_tau=True), 2, "split"),
    ("3d_mma_A32_L4", (8, 256, 64), (4, 8, 4), 4, dict(p_fa=1e-3), 1, "split"),
    ("3d_mma_L16_mu", (8, 128, 64), (2, 8, 8), 16, dict(p_fa=1e-4, mu=12), 1, "split"),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_parity_ci_sizes(case):
    name, n, b, loops, kw, batch, mode = case
    op = oracle_params(n, b, loops, seed=zlib.crc32(name.encode()) % 1000, noise_var=1.0, **kw)
    wl = synth.Workload(name, n, b, loops, op.p_fa, 1.0, (3, 8), (0.0, 20.0), batch, data_seed=77)
    x = frames(wl, batch)
    plan, res, reps = run_case(op, x, mode=mode)
    assert plan.mode == (1 if mode == "fused" else 2)
    assert max(r["max_ratio"] for r in reps) < 1e-4


MMA_CASES = [c for c in CASES if c[0].startswith("3d_mma")]


@pytest.mark.parametrize("case", MMA_CASES, ids=[c[0] for c in MMA_CASES])
def test_parity_ffma_fold_on_mma_shapes(case, monkeypatch):
    """The shapes the tensor-core fold (k_split_mma) takes, forced through the FFMA2 split
    fold (RSFT_NO_MMA=1, read per launch): both kernels stay parity-green."""
    monkeypatch.setenv("RSFT_NO_MMA", "1")
    name, n, b, loops, kw, batch, mode = case
    op = oracle_params(n, b, loops, seed=zlib.crc32(name.encode()) % 1000, noise_var=1.0, **kw)
    wl = synth.Workload(name, n, b, loops, op.p_fa, 1.0, (3, 8), (0.0, 20.0), batch, data_seed=77)
    x = frames(wl, batch)
    plan, res, reps = run_case(op, x, mode=mode)
    assert max(r["max_ratio"] for r in reps) < 1e-4


# the streaming kernel folds B <= 64 and frames whose tables fit (not 1d_g_L20_w1024)
G1_CASES = [c for c in CASES if c[0].startswith("1d_") and c[0] != "1d_g_L20_w1024" and c[2][0] <= 64]


@pytest.mark.parametrize("case", G1_CASES, ids=[c[0] for c in G1_CASES])
def test_parity_1d_streaming_fold_forced(case, monkeypatch):
    """The 1-D shapes forced through the streaming fused fold (RSFT_NO_GATHER1D=1) and the
    region vote (RSFT_NO_VOTE1D=1), both read per launch, instead of the gather-form fold and
    the warp-per-frame vote: both paths stay parity-green."""
    monkeypatch.setenv("RSFT_NO_GATHER1D", "1")
    monkeypatch.setenv("RSFT_NO_VOTE1D", "1")
    name, n, b, loops, kw, batch, mode = case
    op = oracle_params(n, b, loops, seed=zlib.crc32(name.encode()) % 1000, noise_var=1.0, **kw)
    wl = synth.Workload(name, n, b, loops, op.p_fa, 1.0, (3, 8), (0.0, 20.0), batch, data_seed=77)
    x = frames(wl, batch)
    plan, res, reps = run_case(op, x, mode=mode)
    assert max(r["max_ratio"] for r in reps) < 1e-4


V3_CASES = [c for c in CASES if c[0].startswith("3d_")]


@pytest.mark.parametrize("case", V3_CASES, ids=[c[0] for c in V3_CASES])
def test_parity_3d_region_vote_forced(case, monkeypatch):
    """The 3-D shapes with the CTA-per-region vote (RSFT_NO_VOTE3D=1, read per launch) instead
    of the warp-per-region vote on the k_etab expansions: both stay parity-green."""
    monkeypatch.setenv("RSFT_NO_VOTE3D", "1")
    name, n, b, loops, kw, batch, mode = case
    op = oracle_params(n, b, loops, seed=zlib.crc32(name.encode()) % 1000, noise_var=1.0, **kw)
    wl = synth.Workload(name, n, b, loops, op.p_fa, 1.0, (3, 8), (0.0, 20.0), batch, data_seed=77)
    x = frames(wl, batch)
    plan, res, reps = run_case(op, x, mode=mode)
    assert max(r["max_ratio"] for r in reps) < 1e-4


def _votes_all_kernels(plan, bm, cap, monkeypatch, envs):
    import torch
    outs = []
    for env in envs:
        for k in ("RSFT_VOTE3D", "RSFT_NO_VOTE3D", "RSFT_NO_ETAB8", "RSFT_VOTE3D_PK"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        det = plan.detect(bm)
        det_c, idx, cnt = plan.detect_compact(bm, cap)
        torch.cuda.synchronize()
        c = int(cnt.item())
        outs.append((det.cpu().numpy(), det_c.cpu().numpy(), idx.cpu().numpy()[:min(c, cap)], c))
    return outs


V3_ENVS = [{}, {"RSFT_NO_VOTE3D": "1"}, {"RSFT_NO_ETAB8": "1"}, {"RSFT_NO_ETAB8": "1", "RSFT_NO_VOTE3D": "1"},
           {"RSFT_VOTE3D_PK": "0"}]


@pytest.mark.parametrize("case", V3_CASES[:8], ids=[c[0] for c in V3_CASES[:8]])
def test_3d_votes_bit_identical(case, monkeypatch):
    """The 3-D votes (k_vote3d, warp per plane on the k_etab expansions; k_vote, CTA per region),
    each on the expansions of k_etab8 (nibble form, B_last = 8) and of k_etab (per-bit form),
    k_vote3d with packed per-lane offsets and with per-lookup index arithmetic,
    are integer work on the same bitmaps: their detection words, counts and index lists must be
    bit-identical."""
    import torch
    name, n, b, loops, kw, batch, mode = case
    op = oracle_params(n, b, loops, seed=zlib.crc32(name.encode()) % 1000, noise_var=1.0, **kw)
    wl = synth.Workload(name, n, b, loops, op.p_fa, 1.0, (3, 8), (0.0, 20.0), batch, data_seed=77)
    x = torch.from_numpy(frames(wl, batch)).cuda()
    plan = make_plan(op, max_batch=batch, mode=mode).bind()
    bm = plan.execute(x)
    outs = _votes_all_kernels(plan, bm, batch * plan.ntot, monkeypatch, V3_ENVS)
    for o in outs[1:]:
        for a_, b_ in zip(outs[0], o):
            np.testing.assert_array_equal(np.asarray(a_), np.asarray(b_))


@pytest.mark.parametrize("name", ["c3_3d", "c5_cube"])
def test_3d_votes_bit_identical_full_size(name, monkeypatch):
    """c3 (batched) and the c5 cube at full size: the 3-D votes bit-identical (the c5 planes of
    1024 words exceed k_vote3d's default limit; RSFT_VOTE3D=1 forces it there)."""
    import torch
    wl = synth.WORKLOADS[name]
    batch = 8 if name == "c3_3d" else 1
    x = torch.from_numpy(frames(wl.with_(batch=batch), batch)).cuda()
    op = wl_params(wl)
    plan = make_plan(op, max_batch=batch).bind()
    bm = plan.execute(x)
    envs = [{}, {"RSFT_VOTE3D": "1"}, {"RSFT_NO_VOTE3D": "1"}, {"RSFT_NO_ETAB8": "1"}, {"RSFT_VOTE3D_PK": "0"}]
    outs = _votes_all_kernels(plan, bm, 1 << 22, monkeypatch, envs)
    assert outs[0][3] > 0
    for o in outs[1:]:
        for a_, b_ in zip(outs[0], o):
            np.testing.assert_array_equal(np.asarray(a_), np.asarray(b_))


SW_CASES = [c for c in CASES if c[0] in ("1d_g_c1like", "1d_v_dense_pfa", "2d_fused", "2d_v_c4like", "2d_v_dense_mu",
                                          "2d_v_mu1_dense", "2d_split_rpw1", "3d_c3like_mu")]


@pytest.mark.parametrize("case", SW_CASES, ids=[c[0] for c in SW_CASES])
def test_scan_write_one_launch_vs_two_pass(case, monkeypatch):
    """The sorted index list through k_region_scan_write (scan + writer in one launch, default for
    <= 8192 vote regions) and through the two-pass scan + region writer (RSFT_NO_SCANWRITE=1, read
    per launch): integer work on the same counts, so count and list must be bit-identical -- with
    batches that span several writer CTAs and a ragged tail, dense spectra whose region lists
    overflow (the writer re-reads the detection words), and a capacity below the count."""
    import torch
    name, n, b, loops, kw, batch, mode = case
    batch = 37 if len(n) < 3 else 5
    op = oracle_params(n, b, loops, seed=zlib.crc32(name.encode()) % 1000, noise_var=1.0, **kw)
    wl = synth.Workload(name, n, b, loops, op.p_fa, 1.0, (3, 8), (0.0, 20.0), batch, data_seed=78)
    x = torch.from_numpy(frames(wl, batch)).cuda()
    plan = make_plan(op, max_batch=batch, mode=mode).bind()
    full = batch * plan.ntot
    outs = []
    for env in (None, "1"):
        monkeypatch.delenv("RSFT_NO_SCANWRITE", raising=False)
        if env:
            monkeypatch.setenv("RSFT_NO_SCANWRITE", env)
        for cap in (full, 7):
            idx0 = torch.full((cap + 5,), -1, dtype=torch.int64, device="cuda")
            _, det, idx, cnt = plan.run(x, cap, idx=idx0)
            _, idx2, cnt2 = plan.detect_compact(plan.execute(x), cap)
            torch.cuda.synchronize()
            c = int(cnt.item())
            assert int(cnt2.item()) == c
            assert (idx0[cap:] == -1).all()                # nothing written past the capacity
            outs.append((c, idx.cpu().numpy()[:min(c, cap)], idx2.cpu().numpy()[:min(c, cap)], det.cpu().numpy()))
    assert outs[0][0] > 0
    for k in (0, 1):
        for a_, b_ in zip(outs[k], outs[k + 2]):
            np.testing.assert_array_equal(np.asarray(a_), np.asarray(b_))
    c, idx, _, det = outs[0]
    bits = np.unpackbits(det.view(np.uint8), bitorder="little")
    np.testing.assert_array_equal(np.flatnonzero(bits), idx)   # ascending flat indices == the set bits


V2_CASES = [c for c in CASES if c[0].startswith("2d_") and c[6] == "fused"]


@pytest.mark.parametrize("case", V2_CASES, ids=[c[0] for c in V2_CASES])
@pytest.mark.parametrize("force", ["1", "0"])
def test_parity_2d_frame_vote_forced(case, force, monkeypatch):
    """The 2-D shapes with the persistent CTA-per-frame vote forced on / off (RSFT_VOTE2D=1/0,
    read per launch; default: on for N0 <= 256): both paths stay parity-green."""
    monkeypatch.setenv("RSFT_VOTE2D", force)
    name, n, b, loops, kw, batch, mode = case
    op = oracle_params(n, b, loops, seed=zlib.crc32(name.encode()) % 1000, noise_var=1.0, **kw)
    wl = synth.Workload(name, n, b, loops, op.p_fa, 1.0, (3, 8), (0.0, 20.0), batch, data_seed=77)
    x = frames(wl, batch)
    plan, res, reps = run_case(op, x, mode=mode)
    assert max(r["max_ratio"] for r in reps) < 1e-4


W32_CASES = [c for c in CASES if c[0].startswith(("3d_w32", "3d_w64"))]


@pytest.mark.parametrize("case", W32_CASES, ids=[c[0] for c in W32_CASES])
def test_outer_fft_warp_vs_cta_forms(case, monkeypatch):
    """The register-form outer FFT (k_split_fft_wr, default for B_0 = 32 / 64), the CTA form
    (RSFT_FFT_WARP=0) and, for B_0 = 32, the direct-DFT warp form (k_split_fft_w32,
    RSFT_FFT_W32DFT=1; env read per launch) on the same input: each within the oracle tolerance."""
    name, n, b, loops, kw, batch, mode = case
    op = oracle_params(n, b, loops, seed=zlib.crc32(name.encode()) % 1000, noise_var=1.0, **kw)
    wl = synth.Workload(name, n, b, loops, op.p_fa, 1.0, (3, 8), (0.0, 20.0), batch, data_seed=77)
    x = frames(wl, batch)
    monkeypatch.setenv("RSFT_FFT_WARP", "0")
    _, res_cta, reps = run_case(op, x, mode=mode)
    assert max(r["max_ratio"] for r in reps) < 1e-4
    monkeypatch.delenv("RSFT_FFT_WARP")
    if b[0] == 32:
        monkeypatch.setenv("RSFT_FFT_W32DFT", "1")
        _, _, reps = run_case(op, x, mode=mode)
        assert max(r["max_ratio"] for r in reps) < 1e-4
        monkeypatch.delenv("RSFT_FFT_W32DFT")
    _, res_w, reps = run_case(op, x, mode=mode)
    assert max(r["max_ratio"] for r in reps) < 1e-4


def test_parity_1d_gather_many_frames_ring_wrap():
    """c1's shape with many more frames than resident CTAs x ring slots: every CTA wraps its
    frame ring several times (producer/consumer phases); sampled frames vs the oracle."""
    wl = synth.C1.with_(batch=3000)
    x = frames(wl, 3000)
    plan, res, reps = run_case(wl_params(wl), x, check=[0, 1, 295, 296, 297, 1500, 2999])
    assert max(r["max_ratio"] for r in reps) < 1e-4


def test_parity_persistent_many_frames():
    """More frames than resident CTAs: each persistent CTA loops over several frames."""
    op = oracle_params((64, 64), (8, 8), 3, p_fa=1e-3, seed=5)
    wl = synth.Workload("many", (64, 64), (8, 8), 3, 1e-3, 1.0, (2, 6), (0.0, 20.0), 700, data_seed=9)
    x = frames(wl, 700)
    run_case(op, x, mode="fused", check=[0, 1, 2, 296, 297, 350, 591, 699])


def test_zero_and_noise_only_frames():
    op = oracle_params((128, 64), (16, 8), 4, p_fa=1e-2, seed=2)
    x = np.zeros((3, 128, 64), dtype=np.complex64)
    x[1] = synth.gen_noise_only((128, 64), 1.0, 4)
    plan, res, _ = run_case(op, x, mode="fused")
    assert not res["bm"][0].any() and not res["det"][0].any()


def test_gamma_override_noiseless_ongrid_truth():
    """Noiseless on-grid tones, tiny gamma: every tone cell detected (Prop. 3), GPU == oracle."""
    n, b = (128, 64), (16, 8)
    op = oracle_params(n, b, 4, gamma_override=1e-3, seed=5)
    rng = np.random.default_rng(4)
    bins = np.stack([rng.integers(0, n[0], 5), rng.integers(0, n[1], 5)], axis=1)
    x = synth.gen_ongrid(n, bins, np.exp(2j * np.pi * rng.random(5))).astype(np.complex64)[None]
    plan, res, _ = run_case(op, x, mode="fused")
    from paper_1610_01050_b200 import rsft as B
    det = B.bitmap_to_bool(res["det"][0], 128 * 64).reshape(n)
    for i0, i1 in bins:
        assert det[i0, i1]


def test_loop_range_and_slabs():
    """Loop-sharded execute (loops [lb, le)) equals the matching slice of the full run, and
    sharded voting over dim-0 slabs equals the matching slice of the full detection."""
    import torch
    for n, b, L in [((64, 32, 32), (8, 4, 8), 6), ((128, 64), (16, 8), 6)]:
        op = oracle_params(n, b, L, p_fa=1e-3, seed=11)
        wl = synth.Workload("lr", n, b, L, 1e-3, 1.0, (4, 8), (0.0, 20.0), 2, data_seed=3)
        x = frames(wl, 2)
        plan = make_plan(op, max_batch=2).bind()
        xt = torch.from_numpy(x).cuda()
        full = plan.execute(xt)
        parts = [plan.execute(xt, loop_begin=a, loop_end=e) for a, e in [(0, 2), (2, 5), (5, 6)]]
        torch.cuda.synchronize()
        np.testing.assert_array_equal(torch.cat(parts, dim=1).cpu().numpy(), full.cpu().numpy())
        det = plan.detect(full).cpu().numpy()
        per_row = plan.ntot // n[0] // 32
        for a, e in [(0, 8), (8, 40), (40, n[0])]:
            d = plan.detect(full, dim0=(a, e)).cpu().numpy()
            np.testing.assert_array_equal(d, det[:, a * per_row:e * per_row])


def test_run_host_end_to_end():
    import torch
    op = oracle_params((128, 64), (16, 8), 4, p_fa=1e-3, seed=6)
    wl = synth.Workload("rh", (128, 64), (16, 8), 4, 1e-3, 1.0, (4, 8), (0.0, 20.0), 3, data_seed=5)
    x = frames(wl, 3)
    plan = make_plan(op, max_batch=3).bind()
    cap = 1 << 16
    scratch = torch.empty(plan.host_scratch_bytes(3, cap), dtype=torch.uint8, device="cuda")
    hx = torch.from_numpy(x).pin_memory()
    idx, count = plan.run_host(hx, cap, scratch)
    res = gpu_run(plan, x)
    np.testing.assert_array_equal(idx, res["idx"])
    assert count == res["count"]
    tb = R.make_tables(op)
    for f in range(3):
        check_frame(res, f, x[f], op, tb)


def test_compaction_capacity_overflow():
    import torch
    op = oracle_params((64, 64), (8, 8), 2, p_fa=0.3, mu=1, seed=1)
    wl = synth.Workload("cap", (64, 64), (8, 8), 2, 0.3, 1.0, (4, 8), (0.0, 20.0), 2, data_seed=2)
    x = frames(wl, 2)
    plan = make_plan(op, max_batch=2).bind()
    res = gpu_run(plan, x, capacity=10)
    assert res["count"] > 10 and res["idx"].size == 10
    full = gpu_run(plan, x)
    np.testing.assert_array_equal(res["idx"], full["idx"][:10])


@pytest.mark.parametrize("n,b,L", [((64, 32, 32), (8, 4, 8), 4),       # FFMA2 split fold
                                   ((16, 128, 64), (4, 8, 8), 8)])    # tensor-core fold (k_split_mma)
def test_determinism_bitwise(n, b, L):
    """Bitwise-reproducible spectra (fixed reduction orders; the tensor-core fold sums its two
    worker groups' accumulators in a fixed order)."""
    import torch
    op = oracle_params(n, b, L, p_fa=1e-3, seed=3)
    wl = synth.Workload("det", n, b, L, 1e-3, 1.0, (4, 8), (0.0, 20.0), 1, data_seed=8)
    x = frames(wl, 1)
    plan = make_plan(op).bind()
    a = gpu_run(plan, x)
    b = gpu_run(plan, x)
    np.testing.assert_array_equal(a["spectra"].view(np.uint64), b["spectra"].view(np.uint64))


# ----------------------------------------------------------------------------- full sizes
def wl_params(wl):
    return oracle_params(wl.n, wl.b, wl.loops, support=wl.support, p_fa=wl.p_fa, noise_var=wl.noise_var,
                         seed=wl.sched_seed, random_tau=wl.random_tau, mu=wl.mu)


@pytest.mark.parametrize("name", ["c1_1d", "c2_2d", "c3_3d"])
def test_parity_full_size_single_frame(name):
    wl = synth.WORKLOADS[name]
    x = frames(wl, 1)
    _, _, reps = run_case(wl_params(wl), x)
    assert reps[0]["max_ratio"] < 1e-4


def test_parity_c4_full_batch_sampled():
    """c4 at full size in the bench launch configuration (4096 frames, fused persistent
    kernel).  The batch tiles 64 distinct seeded frames (bench.py uses the same recipe with a
    larger pool): every one of the 64 distinct frames is checked against the oracle (buckets,
    bits, vote counts, detection set), and every tiled copy f + 64 k must give bit-identical
    spectra, bitmaps, counts and detections on the GPU (all 4096 frames covered)."""
    wl = synth.C4
    pool = frames(wl, 64)
    x = np.concatenate([pool] * (wl.batch // 64), axis=0)
    _, res, reps = run_case(wl_params(wl), x, check=range(64))
    assert max(r["max_ratio"] for r in reps) < 1e-4
    for key in ("spectra", "bm", "det", "counts"):
        a = res[key].reshape((wl.batch // 64, 64) + res[key].shape[1:])
        assert (a == a[:1]).all(), key


@pytest.mark.parametrize("batch", [1, 8])
def test_parity_c2_shape_fused_batch(batch):
    """c2's exact shape (256x256, B=16x16, L=6, P_fa=1e-5) in FUSED mode (the kernel the c2
    batched bench line runs), multi-frame, every frame against the oracle."""
    wl = synth.C2.with_(batch=batch)
    x = frames(wl, batch)
    plan, _, reps = run_case(wl_params(wl), x, mode="fused")
    assert plan.mode == 1
    assert max(r["max_ratio"] for r in reps) < 1e-4


def test_fused2v_many_frames():
    """rsft_run's D = 2 warp-specialised kernel (k_fused2v) on c2's shape with more frames than
    CTAs: every CTA cycles its residue-sum slot(s) many times (Ffull / Fempty phases).  gpu_run
    compares its bitmaps, detections and index list with rsft_execute + rsft_detect_compact;
    sampled frames (CTA boundaries 147/148, the last frame) against the oracle."""
    wl = synth.C2.with_(batch=400)
    x = frames(wl, 400)
    plan, _, reps = run_case(wl_params(wl), x, mode="fused", check=[0, 1, 147, 148, 149, 296, 399])
    assert plan.mode == 1
    assert max(r["max_ratio"] for r in reps) < 1e-4


def test_parity_c5_full_cube():
    """c5 (512 MiB cube, L=16, split mode): every loop's buckets and bits, and the detection
    set, against the oracle (slow: the oracle runs Alg. 1 literally on 2^26 samples)."""
    wl = synth.C5
    x = frames(wl, 1)
    run_case(wl_params(wl), x)


# ----------------------------------------------------------------------------- variant B
def _slab_run(plan, x, slabs):
    import torch
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    folded = None
    for a, e in slabs:
        part = plan.bucketize_partial(xt[0, a:e].contiguous(), a)
        folded = part.clone() if folded is None else folded + part
    sp = torch.empty((plan.loops, plan.btot), dtype=torch.complex64, device="cuda")
    bm = plan.finalize(folded, spectra=sp)
    return folded, bm, sp


@pytest.mark.parametrize("n,b,L,slabs", [
    ((64, 32, 32), (8, 4, 8), 6, [(0, 16), (16, 40), (40, 64)]),
    ((128, 64), (16, 16), 4, [(0, 64), (64, 128)]),
    ((32, 16, 64), (4, 4, 8), 12, [(0, 8), (8, 12), (12, 32)]),
    ((16, 128, 64), (4, 8, 8), 8, [(0, 4), (4, 12), (12, 16)]),     # tensor-core fold
])
def test_variant_b_slab_partials(n, b, L, slabs):
    """Slab partial folds (linear in x) summed + rsft_finalize == the whole-frame first stage:
    buckets vs the oracle within 1e-4, bits exact outside the band; loop-sharded finalize
    returns the matching rows."""
    import torch
    op = oracle_params(n, b, L, p_fa=1e-3, seed=21, random_tau=True)
    wl = synth.Workload("vb", n, b, L, 1e-3, 1.0, (3, 8), (0.0, 20.0), 1, data_seed=12)
    x = frames(wl, 1)
    plan = make_plan(op, max_batch=1, mode="split").bind()
    folded, bm, sp = _slab_run(plan, x, slabs)
    torch.cuda.synchronize()
    res = {"bm": bm.cpu().numpy()[None], "spectra": sp.cpu().numpy()[None], "det": None}
    tb = R.make_tables(op)
    ref = R.rsft_run(x[0], op, tb)
    px = float(np.mean(np.abs(x[0].astype(np.complex128)) ** 2))
    from paper_1610_01050_b200 import rsft as B
    for l, st in enumerate(ref.stages):
        cb = R.compare_buckets(res["spectra"][0, l].reshape(b), st, px)
        assert cb["ok"], (l, cb)
        bits = B.bitmap_to_bool(res["bm"][0, l], plan.btot).reshape(b)
        assert R.compare_bits(bits, st)["ok"], l
    part = plan.finalize(folded[2:L - 1].contiguous(), loop_begin=2, loop_end=L - 1)
    np.testing.assert_array_equal(part.cpu().numpy(), bm.cpu().numpy()[2:L - 1])


def test_variant_b_c5_full_cube():
    """c5 at full size: 4 slabs of 512 planes (the 4-rank variant-B split) + finalize vs the
    unsharded rsft_execute: spectra within fp32 rounding, bits equal outside the 1e-3 band."""
    import torch
    wl = synth.C5
    x = frames(wl, 1)
    op = wl_params(wl)
    plan = make_plan(op, max_batch=1).bind()
    xt = torch.from_numpy(x).cuda()
    sp_full = torch.empty((1, plan.loops, plan.btot), dtype=torch.complex64, device="cuda")
    bm_full = plan.execute(xt, spectra=sp_full)
    del xt
    _, bm, sp = _slab_run(plan, x, [(0, 512), (512, 1024), (1024, 1536), (1536, 2048)])
    torch.cuda.synchronize()
    a, f = sp.cpu().numpy().astype(np.complex128), sp_full.cpu().numpy()[0].astype(np.complex128)
    beta, gamma = plan.thresholds()
    px = float(np.mean(np.abs(x[0].astype(np.complex128)) ** 2))
    floor = np.sqrt(beta * px)[:, None]
    assert np.max(np.abs(a - f) / np.maximum(np.abs(f), floor)) < 1e-4
    from paper_1610_01050_b200 import rsft as B
    for l in range(plan.loops):
        b1 = B.bitmap_to_bool(bm.cpu().numpy()[l], plan.btot)
        b2 = B.bitmap_to_bool(bm_full.cpu().numpy()[0, l], plan.btot)
        band = np.abs(np.abs(f[l]) ** 2 - gamma[l]) <= 1e-3 * gamma[l]
        assert np.all((b1 == b2) | band)


# ----------------------------------------------------------------------------- segment mode
@pytest.mark.parametrize("n,b,L,mode", [
    ((128, 64), (16, 8), 5, "fused"),
    ((1024,), (64,), 50, "fused"),                  # the paper's T = 50
    ((1024,), (32,), 4, "fused"),
    ((1024,), (128,), 6, "fused"),                  # gather-form segments, 4 buckets per lane
    ((1024,), (256,), 12, "fused"),                 # 8 buckets per lane
    ((4096,), (64,), 3, "fused"),                   # W = N > 1024: the streaming 1-D fold, per loop
    ((32, 16, 64), (4, 4, 8), 3, "split"),
    ((64, 128, 32), (8, 16, 8), 4, "split"),          # c3-like: multi-a0 boxes, batched segments
    ((128, 64), (16, 16), 3, "split"),                # D = 2 split, batched segments
    ((64, 32, 32), (32, 16, 8), 4, "split"),          # B_0 = 32: warp-form outer FFT, segments
])
def test_segment_mode_parity(n, b, L, mode):
    """Segment mode: loop l folds segment l of each frame (rsft_execute_segments);
    buckets, bits and the detection set against the oracle's rsft_run_segments."""
    import torch
    from paper_1610_01050_b200 import rsft as B
    batch = 3
    op = oracle_params(n, b, L, p_fa=1e-3, seed=41, random_tau=True, mu=max(1, L - 1))
    wl = synth.Workload("seg", n, b, L, 1e-3, 1.0, (3, 6), (0.0, 20.0), batch * L, data_seed=19)
    xs = frames(wl, batch * L).reshape((batch, L) + tuple(n))
    plan = make_plan(op, max_batch=batch, mode=mode).bind()
    xt = torch.from_numpy(np.ascontiguousarray(xs)).cuda()
    sp = torch.empty((batch, L, plan.btot), dtype=torch.complex64, device="cuda")
    bm = plan.execute_segments(xt, spectra=sp)
    det = plan.detect(bm)
    torch.cuda.synchronize()
    tb = R.make_tables(op)
    spn, bmn, detn = sp.cpu().numpy(), bm.cpu().numpy(), det.cpu().numpy()
    for f in range(batch):
        ref = R.rsft_run_segments(xs[f], op, tb)
        for l, st in enumerate(ref.stages):
            px = float(np.mean(np.abs(xs[f, l].astype(np.complex128)) ** 2))
            cb = R.compare_buckets(spn[f, l].reshape(b), st, px)
            assert cb["ok"], (f, l, cb)
            assert R.compare_bits(B.bitmap_to_bool(bmn[f, l], plan.btot).reshape(b), st)["ok"], (f, l)
        dset = B.bitmap_to_bool(detn[f], plan.ntot).reshape(n)
        assert R.compare_sets(dset, ref, op.mu)["ok"], f
