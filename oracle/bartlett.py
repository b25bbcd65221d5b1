"""Oracle of the Bartlett baseline (Algorithm 2, App. A; Eq. bartlettROC).
fp64 NumPy, literal: x = sum_s |NDFFT(W r_s)|^2, l = x / T, o = {k : l_k > gamma}.

*** TEST INFRASTRUCTURE ONLY *** (same rule as rsft_ref.py).
"""
from __future__ import annotations

import math

import numpy as np

from . import rsft_ref as R


def compound_window(p: R.Params) -> np.ndarray:
    """W = outer product of the per-dimension pre-windows."""
    return R.outer_nd([R.prewindow(p, d) for d in range(p.ndim)])


def bartlett(xs: np.ndarray, p: R.Params):
    """Alg. 2: returns (x, l) for segments xs [T][N...] (l = x / T)."""
    w = compound_window(p)
    x = np.zeros(p.n)
    for s in range(xs.shape[0]):
        u = w * xs[s].astype(np.complex128)          # l.4 windowing
        uh = np.fft.fftn(u)                          # l.5 N-D FFT (forward, unnormalised)
        x = x + np.abs(uh) ** 2                      # l.6 accumulation
    return x, x / xs.shape[0]


def beta_prime(p: R.Params) -> float:
    """beta' = ||w||^2 (App. A, below Eq. f_km)."""
    return float(np.sum(compound_window(p) ** 2))


def phi_inv(q: float) -> float:
    """Phi^{-1}(q) by bisection on the standard Normal CDF."""
    lo, hi = -40.0, 40.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if 0.5 * math.erfc(-mid / math.sqrt(2.0)) < q:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def threshold(p: R.Params, T: int, p_fa: float) -> float:
    """gamma for a per-bin P_fa under the Normal law of l under H'0 (App. A):
    N(sigma_n^2 beta', sigma_n^4 beta'^2 / T)."""
    return p.noise_var * beta_prime(p) * (1.0 + phi_inv(1.0 - p_fa) / math.sqrt(T))


def roc_pd(p_fa: float, snr: float, alpha_p: float, beta_p: float, T: int) -> float:
    """Eq. bartlettROC."""
    z = (beta_p * phi_inv(1.0 - p_fa) + math.sqrt(T) * (beta_p - snr * alpha_p)) / (snr * alpha_p)
    return 1.0 - 0.5 * math.erfc(-z / math.sqrt(2.0))
