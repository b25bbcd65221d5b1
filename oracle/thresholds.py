"""Oracle for the RSFT optimal threshold design: Eq. opt
with the first-stage laws of Eqs. tpd / bpd and the asymptotic Normal laws of
the accumulated votes, Claims 2-3.  fp64, plain Python/NumPy.

*** TEST INFRASTRUCTURE ONLY ***  (same rule as rsft_ref.py: only tests/, smoke() and
bench.py's CPU legs use it; the product's C++ design routine shares nothing with it).

Steps, in the paper's order and notation:
  alpha(p, sigma, omega) = |u_p^H V_sigma v(omega)|^2  and  beta(sigma) = ||Wbar P_sigma w||^2
      (Eq. alpha_beta), p = the peak bucket of Claim 1 (Eq. lemma13);
  alpha_bar, beta_bar = their expectations over the permutation (Eq. bpd), taken
      here as the mean over ALL odd sigma (and tau = 0);
  Claim 2: a1 ~ N(T Pd_bar, T Pd_bar (1 - Pd_bar))  (variance upper bound);
  Claim 3: a0 ~ N(F eta_p Pd_bar + (T - F) Pfa_bar,
                              F eta_p Pd_bar (1 - eta_p Pd_bar) + (T - F) Pfa_bar (1 - Pfa_bar)),
      F = T K eta_m / B;
  Eq. opt: for each mu in [T] solve P_d = int_mu^inf g_a1 for Pd_bar, then
      P_fa = int_mu^inf g_a0 for Pfa_bar, then SNR_min from Eq. bpd
      Pd_bar = Pfa_bar^(beta_bar / (alpha_bar SNR + beta_bar)); keep the mu with the
      smallest SNR_min; gamma* = sigma_n^2 beta_bar ln(1 / Pfa_bar) (Eq. bpd).
Readings: "int_mu^inf" of the Normal PDF is taken literally (continuous, no continuity
correction, L20); eta_p is an input (1 = lower bound, Remark 3 P:538-540), or the
co-existing sinusoids' first-stage detection rate at a given SNR offset (Fig. exHiBd P:661,
L21).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import rsft_ref as R


def q_normal(x: float) -> float:
    """Upper tail of N(0, 1): int_x^inf phi."""
    return 0.5 * math.erfc(x / math.sqrt(2.0))


def normal_tail(mu: float, mean: float, var: float) -> float:
    """int_mu^inf of the N(mean, var) PDF (var = 0: a point mass at mean)."""
    if var <= 0.0:
        return 1.0 if mean >= mu else 0.0
    return q_normal((mu - mean) / math.sqrt(var))


def bisect_increasing(f, target: float, lo: float = 0.0, hi: float = 1.0, iters: int = 200) -> float:
    """x in [lo, hi] with f(x) = target for f non-decreasing (plain bisection)."""
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if f(mid) < target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def eta_6db(w: np.ndarray, pad: int = 64) -> float:
    """6.0-dB main-lobe width of window w in DFT bins: width of the region
    around DC where |W(f)| >= |W(0)| / 2, from a `pad`-times zero-padded DFT."""
    n = w.size
    spec = np.abs(np.fft.fft(w, n * pad))
    half = spec[0] / 2.0
    k = 0
    while spec[k + 1] >= half:
        k += 1
    # linear interpolation of the crossing between k and k + 1 (one-sided), two-sided width
    x = k + (spec[k] - half) / (spec[k] - spec[k + 1])
    return 2.0 * x / pad


def alpha_beta_1d(p: R.Params, omega_bins: float, sigmas=None):
    """alpha(p(omega, sigma), sigma, omega) and beta(sigma) of a 1-D plan for every odd sigma
    (tau = 0), by running the oracle's first stage (Alg. 1 l.5-9) on the unit sinusoid
    v(omega)[n] = e^{j 2 pi omega_bins n / N} (Eq. sinusoid) and reading the Claim 1
    peak bucket.  Returns (alphas, betas) arrays over sigma."""
    n, b = p.n[0], p.b[0]
    v = np.exp(2j * np.pi * omega_bins * np.arange(n) / n)
    sigmas = list(range(1, n, 2)) if sigmas is None else list(sigmas)
    alphas, betas = [], []
    for s in sigmas:
        tb = R.make_tables(p, schedule_override=(np.array([[s]]), np.array([[0]])))
        st = R.first_stage(v, p, tb, 0)
        peak = int(b * ((s * int(math.floor(omega_bins))) % n) // n)   # Eq. lemma13
        alphas.append(abs(st.fhat[peak]) ** 2)
        betas.append(st.beta)
    return np.asarray(alphas), np.asarray(betas)


@dataclass
class Design:
    mu: int                 # second-stage vote threshold mu*
    snr_min: float          # SNR_min* (linear, per sample: sigma_bm^2 / sigma_n^2)
    snr_min_db: float
    pd_bar: float           # first-stage P_d_bar at the optimum
    pfa_bar: float          # first-stage P_fa_bar at the optimum
    gamma: float            # gamma* = sigma_n^2 beta_bar ln(1 / Pfa_bar) (Eq. bpd)
    table: list             # (mu, snr_min or None) for every mu in [T]


def optimize(T: int, K: int, B: int, eta_m: float, alpha_bar: float, beta_bar: float, p_d: float,
             p_fa: float, eta_p=1.0, noise_var: float = 1.0) -> Design:
    """Eq. opt by enumerating mu in [T] = {1, ..., T}.  eta_p: a number (>= 1),
    or a callable eta_p(pd_bar) returning the calibrated success rate eta_p * Pd_bar of the
    co-existing sinusoids (e.g. 1 for the upper bound of Remark 3)."""
    F = T * K * eta_m / B                                   # Claim 3
    if F >= T:
        raise ValueError("infeasible: K eta_m >= B (Remark 2, P:517)")
    best = None
    table = []
    for mu in range(1, T + 1):
        # P_d = int_mu^inf g_a1: Pd_bar (Claim 2 variance bound)
        pd_bar = bisect_increasing(lambda q: normal_tail(mu, T * q, T * q * (1.0 - q)), p_d)
        rate = eta_p(pd_bar) if callable(eta_p) else eta_p * pd_bar
        rate = min(rate, 1.0)

        def tail0(q):
            mean = F * rate + (T - F) * q
            var = F * rate * (1.0 - rate) + (T - F) * q * (1.0 - q)
            return normal_tail(mu, mean, var)

        if tail0(0.0) > p_fa:                              # even Pfa_bar = 0 exceeds P_fa
            table.append((mu, None))
            continue
        pfa_bar = bisect_increasing(tail0, p_fa)
        if not (0.0 < pfa_bar < pd_bar < 1.0):
            table.append((mu, None))
            continue
        snr = beta_bar / alpha_bar * (math.log(pfa_bar) / math.log(pd_bar) - 1.0)   # Eq. bpd inverted
        table.append((mu, snr))
        if best is None or snr < best[1]:
            best = (mu, snr, pd_bar, pfa_bar)
    if best is None:
        raise ValueError("no feasible mu")
    mu, snr, pd_bar, pfa_bar = best
    return Design(mu, snr, 10.0 * math.log10(snr), pd_bar, pfa_bar,
                  noise_var * beta_bar * math.log(1.0 / pfa_bar), table)
