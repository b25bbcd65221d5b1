"""NEXT-4: SRUR scenes (paper §VI, Tables III-IV) and their scoring; the RSFT
in segment mode (one burst per loop) on the Table IV scenarios (-m gpu)."""
import math

import numpy as np
import pytest

from synth import srur


def test_target_bins_closed_form():
    """Eq. s_u with Table III: target 1 (1000 m, 100 m/s, 30 deg) sits at range bin
    2 rho r / c / f_s * R = 999.02, angle bin N sin(30)/2 = 16, Doppler bin 2 v / lambda T_p M
    = 10.667."""
    kr, ka, kd = srur.target_bins(srur.table_iv(0)[0])
    assert kr == pytest.approx(2 * 3e12 * 1000 / 3e8 / 41e6 * 2048)
    assert kr == pytest.approx(999.0244, abs=1e-3)
    assert ka == pytest.approx(16.0)
    assert kd == pytest.approx(2 * 100 / 0.03 * 5e-5 * 32)


def test_noiseless_scene_peaks_at_target_bins():
    """A noiseless burst's 3-D DFT (Hann windowed) peaks at the nearest grid point of each
    target (Claim 4's on-grid/off-grid behaviour aside, the main lobe contains it)."""
    t = srur.Target(500.0, 50.0, 0.0, 0.0)
    shape = (256, 16, 32)
    x = srur.scene([t], 1, 3, shape=shape, noise=False)[0].astype(np.complex128)
    w = [np.sin(np.pi * np.arange(n) / n) ** 2 for n in shape]
    win = w[0][:, None, None] * w[1][None, :, None] * w[2][None, None, :]
    spec = np.abs(np.fft.fftn(x * win))
    peak = np.unravel_index(np.argmax(spec), shape)
    kb = srur.target_bins(t, shape)
    for p, k, n in zip(peak, kb, shape):
        d = abs(p - k) % n
        assert min(d, n - d) <= 1.0


def test_score_geometry():
    shape = (64, 16, 8)
    t = [srur.Target(0.0, 0.0, 0.0, 0.0)]              # bins (0, 0, 0)
    idx = [0 * 16 * 8 + 1 * 8 + 7, 30 * 16 * 8 + 5 * 8 + 4]   # (0, 1, 7): cyclic neighbour; (30, 5, 4): false
    found, nfalse, nalias = srur.score(idx, t, shape=shape)
    assert found.tolist() == [True] and nfalse == 1 and nalias == 0
    # (0, 0, 4): outside the main lobe, on the target's range/angle cell: a Doppler alias
    found, nfalse, nalias = srur.score([4], t, shape=shape)
    assert nfalse == 0 and nalias == 1


@pytest.mark.gpu
@pytest.mark.parametrize("setting", [0, 1])
def test_srur_table_iv_segment_mode(setting):
    """Table IV targets on the 2048 x 64 x 32 cube, T = 32 bursts (Swerling I per burst),
    RSFT in segment mode (one burst per loop) with B = 64 x 16 x 8, first-stage NP
    threshold gamma_l = beta_l ln(1 / P_fa_bar) with P_fa_bar = 0.05 (Eq. bpd) and mu = T / 2.
    Every target is recovered (the paper's RSFT recovers all four in both settings)
    and every detection outside the targets' main lobes is a single-dimension alias of a target
    (reading L25: the short angle / Doppler dimensions have only 32 / 16 odd permutations, so
    a cell on a strong target's range-angle cell collides with it in ~1/4 of the loops).

    Threshold choice (reading L25): at -20 dB the weakest target's peak bucket SNR is
    alpha_bar / beta_bar * 0.01 ~ 9.5 (library design, 29.8 dB window gain), so the per-loop
    detection rate is 0.05^(1 / 10.5) ~ 0.75 and P(Bin(32, 0.75) >= 16) > 0.999; a cell
    outside the targets is hit with probability <= 0.05 + (buckets lit by the four targets) /
    8192 ~ 0.065 per loop, and P(Bin(32, 0.065) >= 16) ~ 4e-11 per cell."""
    import torch
    from paper_1610_01050_b200 import rsft as B
    targets = srur.table_iv(setting)
    T = 32
    shape = (srur.R_BINS, srur.N_ELEM, srur.M_RI)
    design = B.Plan(shape, (64, 16, 8), T, seed=7).design_thresholds(
        K=4, p_d=0.9, p_fa=1e-6, omega=srur.target_bins(targets[2]), loops=T)
    gain = design["alpha_bar"] / design["beta_bar"]
    weakest = min(10 ** (t.snr_db / 10) for t in targets) * gain
    assert 0.05 ** (1.0 / (1.0 + weakest)) > 0.7
    xs = srur.scene(targets, T, seed=11 + setting)
    plan = B.Plan(shape, (64, 16, 8), T, p_fa=0.05, mu=T // 2, seed=7).bind()
    bm = plan.execute_segments(torch.from_numpy(xs[None]).cuda())
    det, idx, cnt = plan.detect_compact(bm, 1 << 20)
    torch.cuda.synchronize()
    got = idx.cpu().numpy()[: int(cnt.item())]
    found, nfalse, nalias = srur.score(got, targets)
    print(f"setting {setting}: window gain {10 * math.log10(gain):.1f} dB; found {found.tolist()}, "
          f"detections {got.size}, single-dimension aliases {nalias}, false {nfalse}")
    assert found.all()
    assert nfalse == 0
    assert nalias <= got.size // 2
