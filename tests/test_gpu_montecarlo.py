"""NEXT-2: segment mode + on-GPU Monte Carlo.
  * the GPU scene generator (rsft_synthesize) equals its NumPy mirror (same counter RNG);
  * the threshold design of Eq. opt (rsft_design_thresholds, NEXT-1) run in segment mode
    (Swerling amplitudes per segment) on GPU-generated trials: the measured
    per-location detection and false-alarm rates of the two-stage detector are compared with
    the design targets P_d, P_fa (Problem 1).  Claims 2-3 are asymptotic in T, so the
    check is a band, and the measured values are printed (recorded in DESIGN.md)."""
import math

import numpy as np
import pytest

import synth
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_generator_matches_numpy_mirror():
    import torch
    from paper_1610_01050_b200 import rsft as B
    rng = np.random.default_rng(3)
    for n in [(64,), (16, 32), (8, 4, 32)]:
        batch, T, K = 2, 3, 2
        om = rng.uniform(0, 1, (batch, K, len(n))) * np.asarray(n)[None, None, :]
        sb = rng.uniform(0.5, 2.0, (batch, K))
        x = B.synthesize(n, batch, T, torch.from_numpy(om).cuda(), torch.from_numpy(sb).cuda(), 0.7, 1234)
        torch.cuda.synchronize()
        ref = synth.synth_segments(n, batch, T, om, sb, 0.7, 1234)
        got = x.cpu().numpy().astype(np.complex128)
        assert np.max(np.abs(got - ref)) < 1e-5 * max(1.0, np.max(np.abs(ref)))
    # statistics of the noise stream: E|z|^2 = 1, circular
    z = synth.counter_normals(9, 2, np.arange(200000))
    assert abs(np.mean(np.abs(z) ** 2) - 1.0) < 0.01 and abs(np.mean(z)) < 0.01


def run_design_mc(n=(1024,), b=(64,), frames=2048, T=12, K=4, p_d=0.9, p_fa=1e-3, seed=77):
    import torch
    from paper_1610_01050_b200 import rsft as B
    probe = B.Plan(n, b, T, seed=seed)
    des = probe.design_thresholds(K=K, p_d=p_d, p_fa=p_fa, omega=(100.5,))
    plan = B.Plan(n, b, T, seed=seed, gamma_override=des["gamma"], mu=des["mu"], max_batch=frames).bind()
    rng = np.random.default_rng(seed)
    ks = np.zeros((frames, K), dtype=np.int64)
    for f in range(frames):                         # resolvable mid-bin tones (eta_m bins apart)
        ks[f] = np.sort(rng.choice(np.arange(0, n[0], 16), K, replace=False) + rng.integers(0, 8, K))
    om = (ks + 0.5).astype(np.float64)[:, :, None]
    sb = np.full((frames, K), math.sqrt(des["snr_min"]))      # every sinusoid at SNR_min* (eta_p = 1)
    x = B.synthesize(n, frames, T, torch.from_numpy(om).cuda(), torch.from_numpy(sb).cuda(), 1.0, seed)
    bm = plan.execute_segments(x)
    det = plan.detect(bm)
    # pure noise through the same plan: the first-stage law of Eq. tpd per loop
    xn = B.synthesize(n, frames, T, None, None, 1.0, seed + 1)
    bmn = plan.execute_segments(xn).cpu().numpy()
    torch.cuda.synchronize()
    d = np.unpackbits(det.cpu().numpy().view(np.uint8), bitorder="little").reshape(frames, -1)[:, : n[0]].astype(bool)
    hit = d[np.arange(frames)[:, None], ks]
    mask = np.ones_like(d)
    for j in range(-2, 4):                          # the tone's main lobe is not a false alarm
        mask[np.arange(frames)[:, None], (ks + j) % n[0]] = False
    bits = np.unpackbits(bmn.view(np.uint8), bitorder="little").reshape(frames, T, -1)[:, :, : plan.btot]
    beta, _ = plan.thresholds()
    fs_meas = bits.mean(axis=(0, 2))
    fs_law = np.exp(-des["gamma"] / beta)           # Eq. tpd with gamma* and this loop's beta
    return des, float(hit.mean()), float(d[mask].mean()), int(mask.sum()), fs_meas, fs_law


@pytest.mark.parametrize("b,T", [((64,), 12), ((32,), 24)])
def test_design_monte_carlo_segment_mode(b, T):
    des, pd_meas, pfa_meas, trials, fs_meas, fs_law = run_design_mc(b=b, T=T)
    print(f"B={b[0]} T={T}: design mu*={des['mu']} SNR*={des['snr_min_db']:.2f} dB gamma*={des['gamma']:.4g} "
          f"Pfa_bar={des['pfa_bar']:.4f}: measured P_d={pd_meas:.3f} (target 0.9), P_fa={pfa_meas:.2e} "
          f"(target 1e-3) over {trials} locations; first stage measured/law "
          f"{np.mean(fs_meas):.4f}/{np.mean(fs_law):.4f}")
    # first stage: Eq. tpd holds per loop (binomial error over frames x B buckets)
    tr = 2048 * b[0]
    assert np.all(np.abs(fs_meas - fs_law) <= 5 * np.sqrt(fs_law * (1 - fs_law) / tr) + 1e-4)
    # second stage: Claims 2-3 replace the vote counts by Normals (T -> infinity).  The same
    # model without that approximation -- per loop a location's bucket holds one of the K
    # sinusoids with probability q = K eta_m / B (Claim 3's F / T) and fires with Pd_bar, else
    # with Pfa_bar -- gives an exact Binomial(T, q Pd_bar + (1 - q) Pfa_bar) tail for P_fa and a
    # Binomial(T, Pd_bar) tail for P_d; the measurement must follow those within MC error.
    from scipy.stats import binom
    q = des["F"] / T
    pfa_exact = binom.sf(des["mu"] - 1, T, q * des["pd_bar"] + (1 - q) * des["pfa_bar"])
    pd_exact = binom.sf(des["mu"] - 1, T, des["pd_bar"])
    print(f"   exact-binomial model: P_d={pd_exact:.3f}, P_fa={pfa_exact:.2e}")
    assert 0.75 <= pd_meas <= 1.0 and abs(pd_meas - pd_exact) < 0.12   # alpha varies with sigma (Jensen)
    assert pfa_exact / 2 <= pfa_meas <= 2 * pfa_exact


# ----------------------------------------------------------------------------- T = 50
def test_per_sigma_first_stage_law_and_variance_bound():
    """The paper's design point (N = 1024, T = 50, B = 64, Dolph-Chebyshev 40 dB, omega_m = 64.5
    bins).  (a) For every odd sigma the GPU's first-stage detection rate of the tone's
    bucket follows Eq. tpd with the oracle's alpha(sigma), beta(sigma) (Eq.
    alpha_beta) -- binomial error, all 512 permutations.  (b) Fig. varAppErr: the
    approximation error of the variance bound T Pd_bar (1 - Pd_bar) from the measured
    per-permutation rates is a few percent (the paper: ~1.6 % at T = 10) and agrees with the
    closed form's."""
    import study_next2 as S
    des = S.design()
    sig, a, b = S.oracle_alpha_beta()
    law = S.tpd(a, b, des["gamma"], des["snr_min"])
    sig_g, p_hat, F = S.per_sigma_detection(des, frames=4096)
    assert np.array_equal(sig, sig_g)
    z = (p_hat - law) / np.sqrt(law * (1 - law) / F)
    print(f"per-sigma law: max |z| = {np.max(np.abs(z)):.2f} over {sig.size} sigmas, mean P~ "
          f"measured {p_hat.mean():.4f} / law {law.mean():.4f}")
    assert np.max(np.abs(z)) < 5.5
    pv = p_hat * (1 - p_hat) * F / (F - 1)
    for T in (10, 50):
        e_law, _ = S.approx_error(law, T)
        e_gpu, _ = S.approx_error(p_hat, T, var_unbiased=pv)
        print(f"T={T}: approximation error law {100 * e_law:.2f} %, GPU {100 * e_gpu:.2f} %")
        assert 0.0 <= e_law < 0.10 and abs(e_gpu - e_law) < 0.02


def test_fixed_schedule_vote_variance_T50():
    """Eq. var_a1 end to end at T = 50: for one schedule the tone location's vote
    count abar_i (rsft_detect counts, segment mode) has mean sum_s P~_d(sigma_s) and variance
    sum_s P~_d (1 - P~_d) <= T Pd_bar (1 - Pd_bar)."""
    import study_next2 as S
    des = S.design()
    sig, a, b = S.oracle_alpha_beta()
    law = S.tpd(a, b, des["gamma"], des["snr_min"])
    sg, ab = S.fixed_schedule_votes(des, frames=8192, batches=2)
    pl = law[(sg - 1) // 2]
    n = ab.size
    mean_ref, var_ref = pl.sum(), (pl * (1 - pl)).sum()
    m4 = np.mean((ab - ab.mean()) ** 4)
    se_var = math.sqrt(max(m4 - ab.var() ** 2, 1e-12) / n)
    print(f"abar: mean {ab.mean():.3f} (sum P~ {mean_ref:.3f}), var {ab.var(ddof=1):.3f} "
          f"(sum P~(1-P~) {var_ref:.3f} +- {se_var:.3f}; bound {S.T_PAPER * law.mean() * (1 - law.mean()):.3f})")
    assert abs(ab.mean() - mean_ref) < 5 * math.sqrt(var_ref / n)
    assert abs(ab.var(ddof=1) - var_ref) < 5 * se_var


def test_detector_at_paper_design_point_T50():
    """The two-stage detector with Eq. opt's (gamma*, mu*) at T = 50: P_d meets the
    target 0.9.  The false-detection rate is MEASURED and printed, not bounded: Claim 3's
    F = T K eta_m / B counts one bucket per sinusoid and loop, but a mid-bin Swerling tone under
    the 40 dB Chebyshev windows lights ~2.5 buckets per loop (first-stage rate ~0.17 per bucket
    instead of Pfa_bar = 0.044; the oracle on the same scenes agrees), so the vote counts of
    non-tone locations sit near 8 instead of ~4 and P_fa is far above the 1e-6 design target --
    reading L26 in DESIGN.md, profiles/r02_next2.md."""
    from scipy.stats import binom
    import study_next2 as S
    des = S.design()
    pd_m, fa, trials = S.detector_at_design(des, frames=4096, batches=1)
    q = des["F"] / S.T_PAPER
    pd_x = binom.sf(des["mu"] - 1, S.T_PAPER, des["pd_bar"])
    pfa_x = binom.sf(des["mu"] - 1, S.T_PAPER, q * des["pd_bar"] + (1 - q) * des["pfa_bar"])
    print(f"T=50 design mu*={des['mu']} SNR*={des['snr_min_db']:.2f} dB gamma*={des['gamma']:.4g}: P_d {pd_m:.3f} "
          f"(target 0.9, exact-binomial {pd_x:.3f}); false detections {fa} / {trials} "
          f"(exact-binomial expects {pfa_x * trials:.1f})")
    assert pd_m >= 0.9 - 5 * math.sqrt(0.09 / (4096 * 4))
    assert 0 < fa < trials
