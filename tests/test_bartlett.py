"""NEXT-3: the Bartlett baseline.  Oracle pins on CPU (-m "not gpu") and the
CUDA implementation (rsft_bartlett, hand-written N-D FFTs) against the oracle (-m gpu)."""
import math

import numpy as np
import pytest
from scipy.stats import gamma as gamma_dist

from oracle import bartlett as BT
from oracle import rsft_ref as R
import synth


def test_hann_ongrid_tone_closed_form():
    """Periodic Hann on an on-grid unit tone: |u_hat|^2 = (N/2)^2 at k0, (N/4)^2 at k0 +- 1,
    0 elsewhere (the window's 3-term DFT); two segments add."""
    n = 256
    p = R.Params(n=(n,), b=(16,), loops=1)
    k0 = 41
    v = np.exp(2j * np.pi * k0 * np.arange(n) / n)
    x, l = BT.bartlett(np.stack([v, 1j * v]), p)
    want = np.zeros(n)
    want[k0] = 2 * (n / 2) ** 2
    want[k0 - 1] = want[k0 + 1] = 2 * (n / 4) ** 2
    np.testing.assert_allclose(x, want, atol=1e-6 * n * n)
    np.testing.assert_allclose(l, want / 2, atol=1e-6 * n * n)


def test_parseval_2d():
    rng = np.random.default_rng(1)
    p = R.Params(n=(32, 64), b=(4, 8), loops=1)
    xs = rng.standard_normal((3, 32, 64)) + 1j * rng.standard_normal((3, 32, 64))
    x, _ = BT.bartlett(xs, p)
    w = BT.compound_window(p)
    assert x.sum() == pytest.approx(32 * 64 * sum(np.sum(np.abs(w * s) ** 2) for s in xs), rel=1e-12)


def test_noise_statistic_is_gamma_and_threshold_semantics():
    """Under H'0 each bin of T l / (sigma_n^2 beta') is a sum of T unit exponentials
    (Gamma(T, 1)); the Normal-law threshold of Eq. bartlettROC maps P_fa to gamma."""
    n, T = 512, 8
    p = R.Params(n=(n,), b=(16,), loops=1, noise_var=2.0)
    rng = np.random.default_rng(5)
    bp = BT.beta_prime(p)
    stats = []
    for trial in range(200):
        xs = math.sqrt(2.0 / 2) * (rng.standard_normal((T, n)) + 1j * rng.standard_normal((T, n)))
        _, l = BT.bartlett(xs, p)
        stats.append(T * l / (2.0 * bp))
    s = np.concatenate(stats)
    # bins of a windowed FFT are correlated only between neighbours; test the marginal law
    for q in (0.5, 0.9, 0.99):
        assert abs(np.mean(s > gamma_dist.ppf(q, T)) - (1 - q)) < 0.01 + 0.1 * (1 - q)
    g = BT.threshold(p, T, 1e-3)
    assert g == pytest.approx(2.0 * bp * (1 + 3.090232306 / math.sqrt(T)), rel=1e-6)


def test_roc_monotone():
    pd = [BT.roc_pd(1e-6, snr, 1000.0, 100.0, 50) for snr in (0.05, 0.1, 0.2, 0.5)]
    assert all(a < b for a, b in zip(pd, pd[1:])) and pd[-1] > 0.99


@pytest.mark.gpu
@pytest.mark.parametrize("n,batch", [((1024,), 3), ((256, 128), 2), ((64, 32, 32), 2), ((4096,), 3), ((128, 64), 3),
                                     ((2048,), 2), ((512,), 2),
                                     ((1024, 256), 2), ((512, 128, 32), 1),
                                     # two-pass 2-D shapes for every transpose-FFT width: rows of 32 M
                                     # points (RW = 32 / M rows per warp), columns of 32 M0 points
                                     ((256, 256), 2), ((512, 64), 2), ((1024, 32), 2), ((128, 512), 2)])
def test_bartlett_gpu_parity(n, batch):
    """Single-pass (<= 8192 samples) and two-pass frames, several frames per call, against the
    oracle's literal Alg. 2 (numpy fftn) frame by frame."""
    import torch
    from paper_1610_01050_b200 import rsft as B
    T = 4
    b = tuple(min(16, v) for v in n)
    wl = synth.Workload("bart", n, b, 1, 1e-3, 1.0, (3, 6), (0.0, 20.0), T, data_seed=29)
    xs = synth.gen_batch(wl, range(batch * T)).reshape((batch, T) + tuple(n))
    p = R.Params(n=n, b=b, loops=1)
    plan = B.Plan(n, b, 1).bind()
    g = plan.bartlett_threshold(T, 1e-3)
    assert g == pytest.approx(BT.threshold(p, T, 1e-3), rel=1e-9)
    power, det = plan.bartlett(torch.from_numpy(np.ascontiguousarray(xs)).cuda(), gamma=g)
    torch.cuda.synchronize()
    pw, dt = power.cpu().numpy().astype(np.float64), det.cpu().numpy()
    for f in range(batch):
        x, l = BT.bartlett(xs[f], p)
        scale = max(float(np.max(x)), 1.0)
        assert np.max(np.abs(pw[f] - x)) <= 1e-5 * scale
        bits = B.bitmap_to_bool(dt[f], int(np.prod(n))).reshape(n)
        ref = l > g
        band = np.abs(l - g) <= 1e-3 * g
        assert np.all((bits == ref) | band)
