"""NEXT-1: the optimal threshold design of Eq. opt.
Oracle pins (closed forms, an independent Normal-tail routine, the paper's worked design
of §V, Figs. exLowBd / exHiBd P:640-665) and the library's C++ design (rsft_design_thresholds)
against the oracle.  All host-side: -m "not gpu"."""
import math

import numpy as np
import pytest
from scipy.stats import norm

from oracle import rsft_ref as R
from oracle import thresholds as TH

# §V common parameters: N = 1024, T = 50, B = 64, eta_m = 1.8, P_d = 0.9,
# P_fa = 1e-6, omega_m = 64.5 bins, Dolph-Chebyshev 40 dB; K = 4 (Fig. exLowBd caption P:653)
SEC5 = dict(T=50, K=4, B=64, eta_m=1.8, p_d=0.9, p_fa=1e-6)


def test_eta_6db_closed_forms():
    """6-dB bandwidths (Harris 1978 [P:262 ref]): Hann 2.00 bins, rectangular 1.21 bins."""
    assert abs(TH.eta_6db(R.hann_periodic(1024)) - 2.0) < 0.01
    assert abs(TH.eta_6db(np.ones(1024)) - 1.207) < 0.01


def test_alpha_beta_brickwall_closed_form():
    """Rectangular pre-window + ideal brick-wall flat window (identity I4): an on-grid unit
    tone lands entirely in its Claim 1 bucket, |f_p|^2 = N^2 for every sigma, and
    beta = ||gbar||^2 = N A (Parseval)."""
    n, b = 256, 16
    p = R.Params(n=(n,), b=(b,), loops=1, prewin="rect")
    gb = R.brickwall_window(n, b)
    k0 = 37
    v = np.exp(2j * np.pi * k0 * np.arange(n) / n)
    for s in (1, 3, 77, 255):
        tb = R.make_tables(p, flat_override=[gb], schedule_override=(np.array([[s]]), np.array([[0]])))
        st = R.first_stage(v, p, tb, 0)
        pk = b * ((s * k0) % n) // n
        assert abs(abs(st.fhat[pk]) ** 2 - n * n) < 1e-6 * n * n
        assert abs(st.beta - n * (n // b)) < 1e-9 * n * n


def test_optimize_self_consistency():
    """At the optimum the asymptotic laws of Claims 2-3 reproduce the targets (checked with
    scipy's Normal survival function, an independent routine), and Eq. bpd maps SNR_min*
    back onto Pd_bar."""
    d = TH.optimize(alpha_bar=1.7, beta_bar=0.3, **SEC5)
    T, F = SEC5["T"], SEC5["T"] * SEC5["K"] * SEC5["eta_m"] / SEC5["B"]
    pd, pf = d.pd_bar, d.pfa_bar
    assert abs(norm.sf(d.mu, T * pd, math.sqrt(T * pd * (1 - pd))) - SEC5["p_d"]) < 1e-9
    m0 = F * pd + (T - F) * pf
    v0 = F * pd * (1 - pd) + (T - F) * pf * (1 - pf)
    assert abs(norm.sf(d.mu, m0, math.sqrt(v0)) - SEC5["p_fa"]) < 1e-12
    assert abs(pf ** (0.3 / (1.7 * d.snr_min + 0.3)) - pd) < 1e-9
    # every feasible mu is no better than the optimum
    assert all(s is None or s >= d.snr_min - 1e-15 for _, s in d.table)
    assert d.gamma == pytest.approx(0.3 * math.log(1 / pf))


def test_remark2_infeasible_and_monotone():
    """Remark 2: RSFT fails once K eta_m >= B; SNR_min* grows with K and falls with T."""
    with pytest.raises(ValueError):
        TH.optimize(50, 36, 64, 1.8, 1.0, 1.0, 0.9, 1e-6)
    s = [TH.optimize(50, k, 64, 1.8, 1.0, 1.0, 0.9, 1e-6).snr_min for k in (1, 4, 10, 20)]
    assert all(a < b for a, b in zip(s, s[1:]))
    s = [TH.optimize(t, 4, 64, 1.8, 1.0, 1.0, 0.9, 1e-6).snr_min for t in (10, 20, 50, 100)]
    assert all(a > b for a, b in zip(s, s[1:]))


def test_paper_worked_design_window_independent_parts():
    """§V design.  mu*/T and the lower-to-upper-bound SNR difference do not depend
    on the window gains alpha_bar / beta_bar (a common factor of SNR_min for every mu), so
    they pin Eq. opt itself: Fig. exLowBd mu*/T ~ 0.3, Fig. exHiBd mu*/T ~ 0.4 (read from the
    captions, +-0.1), SNR_min* -10.1 dB vs -9.1 dB (difference 1.0 dB, +-0.5 dB), and the two
    captions imply the same window gain ratio beta_bar/alpha_bar within 0.5 dB."""
    lo = TH.optimize(alpha_bar=1.0, beta_bar=1.0, eta_p=1.0, **SEC5)
    up = TH.optimize(alpha_bar=1.0, beta_bar=1.0, eta_p=lambda pd: 1.0, **SEC5)
    assert abs(lo.mu / SEC5["T"] - 0.3) <= 0.1
    assert abs(up.mu / SEC5["T"] - 0.4) <= 0.1
    assert abs((up.snr_min_db - lo.snr_min_db) - 1.0) <= 0.5
    ratio_lo = -10.1 - lo.snr_min_db
    ratio_up = -9.1 - up.snr_min_db
    assert abs(ratio_lo - ratio_up) <= 0.5


def _lib_plan(n, b, **kw):
    from paper_1610_01050_b200 import rsft as B
    return B.Plan(n, b, 1, **kw)


@pytest.mark.parametrize("n,b,prewin,param,flat,omega", [
    ((1024,), (64,), "cheb", 40.0, 40.0, (64.5,)),
    ((512,), (32,), "hann", 60.0, 60.0, (100.25,)),
    ((64, 32), (8, 4), "hann", 60.0, 60.0, (10.5, 3.0)),
])
def test_library_design_matches_oracle(n, b, prewin, param, flat, omega):
    """rsft_design_thresholds (C++, factored per-sample sums) == the oracle (literal first stage
    of a unit sinusoid for every odd sigma): alpha_bar, beta_bar to 1e-9, eta_m to 1e-3 bins,
    and the same mu*, SNR_min*, gamma*."""
    plan = _lib_plan(n, b, prewin=prewin, prewin_param=param, flat_atten_db=flat)
    got = plan.design_thresholds(K=3, p_d=0.9, p_fa=1e-5, omega=omega, loops=40)
    p = R.Params(n=n, b=b, loops=1, prewin=prewin, prewin_param=param, flat_atten_db=flat)
    ab = bb = eta = 1.0
    for d in range(len(n)):
        pd1 = R.Params(n=(n[d],), b=(b[d],), loops=1, prewin=prewin, prewin_param=param, flat_atten_db=flat)
        al, be = TH.alpha_beta_1d(pd1, omega[d])
        ab *= al.mean()
        bb *= be.mean()
        eta *= TH.eta_6db(R.prewindow(p, d))
    assert got["alpha_bar"] == pytest.approx(ab, rel=1e-9)
    assert got["beta_bar"] == pytest.approx(bb, rel=1e-9)
    assert abs(got["eta_m"] - eta) < 1e-3
    ref = TH.optimize(40, 3, int(np.prod(b)), got["eta_m"], ab, bb, 0.9, 1e-5)
    assert got["mu"] == ref.mu
    assert got["snr_min"] == pytest.approx(ref.snr_min, rel=1e-9)
    assert got["gamma"] == pytest.approx(ref.gamma, rel=1e-9)
    up = plan.design_thresholds(K=3, p_d=0.9, p_fa=1e-5, eta_p=0.0, omega=omega, loops=40)
    ref_up = TH.optimize(40, 3, int(np.prod(b)), got["eta_m"], ab, bb, 0.9, 1e-5, eta_p=lambda q: 1.0)
    assert up["mu"] == ref_up.mu and up["snr_min"] == pytest.approx(ref_up.snr_min, rel=1e-9)
