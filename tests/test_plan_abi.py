"""CPU tests of the C ABI (no GPU): the library loads, exports every symbol include/rsft.h
declares, validates arguments, and its host plan (C++ fp64) agrees with the oracle's
independently written NumPy tables (windows, schedule, beta, gamma, weights)."""
import math
import os
import re

import numpy as np
import pytest

from oracle import rsft_ref as R
import synth

P = pytest.importorskip("paper_1610_01050_b200")
from paper_1610_01050_b200 import rsft as B  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "rsft.h")) as f:
        txt = f.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rsft_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = B.lib()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(B.EXPORTED) == syms


def oracle_params(wl, **kw):
    d = dict(n=wl.n, b=wl.b, loops=wl.loops, support=wl.support, p_fa=wl.p_fa, noise_var=wl.noise_var,
             seed=wl.sched_seed, random_tau=wl.random_tau, mu=wl.mu)
    d.update(kw)
    return R.Params(**d)


def plan_for(wl, **kw):
    d = dict(support=wl.support, p_fa=wl.p_fa, noise_var=wl.noise_var, seed=wl.sched_seed,
             random_tau=wl.random_tau, mu=wl.mu, max_batch=wl.batch)
    d.update(kw)
    return B.Plan(wl.n, wl.b, wl.loops, **d)


@pytest.mark.parametrize("wl", list(synth.WORKLOADS.values()), ids=list(synth.WORKLOADS))
def test_plan_tables_match_oracle(wl):
    """T2: C++ plan vs NumPy oracle, both fp64, to 1e-12 (windows, beta, gamma) and exact
    (schedule); fp32 weight tables equal the oracle-derived h_{l,d}[s] after fp32 rounding."""
    if wl.name == "c5_cube":
        wl = wl.with_(loops=4)
    p = plan_for(wl)
    op = oracle_params(wl)
    tb = R.make_tables(op)
    sig, sinv, tau = p.schedule()
    np.testing.assert_array_equal(sig, tb.sigma)
    np.testing.assert_array_equal(sinv, tb.sigma_inv)
    np.testing.assert_array_equal(tau, tb.tau)
    for d in range(len(wl.n)):
        np.testing.assert_allclose(p.window(d, 0), tb.prewin[d], rtol=0, atol=1e-10)
        g = R.flat_prototype(wl.n[d], wl.b[d], op.support[d], op.flat_atten_db)
        np.testing.assert_allclose(p.window(d, 1), g, rtol=0, atol=1e-10)
        # I3 weights from the oracle's pieces: h[s] = w[s] g[t] (-1)^floor(t/B), t = sinv (s - tau)
        h = p.window(d, 2)
        n, b = wl.n[d], wl.b[d]
        s = np.arange(n)
        for l in range(wl.loops):
            t = (int(tb.sigma_inv[l, d]) * (s - int(tb.tau[l, d]))) % n
            sign = np.where((t // b) % 2 == 1, -1.0, 1.0) if b < n else np.ones(n)
            want = (tb.prewin[d] * g[t] * sign).astype(np.float32).astype(np.float64)
            np.testing.assert_allclose(h[l], want, rtol=2e-7, atol=1e-12)
    be, ga = p.thresholds()
    for l in range(wl.loops):
        assert math.isclose(be[l], R.beta(op, tb, l), rel_tol=1e-12)
        assert math.isclose(ga[l], R.gamma(op, tb, l), rel_tol=1e-12)


def test_cheb_prewindow_and_gamma_override():
    p = B.Plan((256, 64), (16, 8), 3, prewin="cheb", prewin_param=40.0, gamma_override=7.5, seed=3)
    op = R.Params(n=(256, 64), b=(16, 8), loops=3, prewin="cheb", prewin_param=40.0, gamma_override=7.5, seed=3)
    tb = R.make_tables(op)
    for d in range(2):
        np.testing.assert_allclose(p.window(d, 0), tb.prewin[d], rtol=0, atol=1e-10)
    assert np.all(p.thresholds()[1] == 7.5)


def test_set_schedule_roundtrip_and_errors():
    p = B.Plan((64, 32), (8, 4), 2, seed=1)
    p.set_schedule([[3, 5], [7, 9]], [[1, 2], [3, 4]])
    s, si, t = p.schedule()
    assert s.tolist() == [[3, 5], [7, 9]] and t.tolist() == [[1, 2], [3, 4]]
    assert ((s * si) % np.array([64, 32]) == 1).all()
    with pytest.raises(B.RsftError) as e:
        p.set_schedule([[4, 5], [7, 9]])
    assert e.value.status == 3                                        # RSFT_E_SIGMA
    op = R.Params(n=(64, 32), b=(8, 4), loops=2)
    tb = R.make_tables(op, schedule_override=([[3, 5], [7, 9]], [[1, 2], [3, 4]]))
    be, _ = p.thresholds()
    assert math.isclose(be[1], R.beta(op, tb, 1), rel_tol=1e-12)


@pytest.mark.parametrize("kw,status", [
    (dict(n=(100,), b=(4,), loops=1), 2),                   # N not a power of two
    (dict(n=(64,), b=(128,), loops=1), 2),                  # B > N
    (dict(n=(4096,), b=(128,), loops=1), 4),                # D = 1, B > 64 needs the gather form (W <= 1024)
    (dict(n=(2048,), b=(512,), loops=1, support=(1024,)), 4),   # D = 1, B > 256
    (dict(n=(256, 256), b=(128, 8), loops=1), 4),           # D = 2, B_d > 64
    (dict(n=(64,), b=(8,), loops=1, support=(24,)), 2),     # 2B does not divide W
    (dict(n=(64,), b=(8,), loops=0), 1),
    (dict(n=(64,), b=(8,), loops=64), 4),                   # L > 63 (6 vote bit planes)
    (dict(n=(64,), b=(8,), loops=4, mu=5), 1),              # mu > L
    (dict(n=(64,), b=(8,), loops=4, p_fa=1.5), 1),
    (dict(n=(16,), b=(8,), loops=1), 4),                    # N_last < 32
    (dict(n=(8, 8, 8, 8), b=(2, 2, 2, 2), loops=1), 4),     # D > 3
])
def test_plan_argument_errors(kw, status):
    n = kw.pop("n")
    b = kw.pop("b")
    loops = kw.pop("loops")
    with pytest.raises(B.RsftError) as e:
        B.Plan(n, b, loops, **kw)
    assert e.value.status == status


@pytest.mark.parametrize("n,b,w", [((1024,), (128,), 0), ((1024,), (256,), 0), ((4096,), (256,), 1024),
                                   ((256,), (256,), 0)])
def test_plan_1d_large_b(n, b, w):
    """D = 1 with B = 128 / 256 (the paper's B_opt = 128 at K = 100; B = 256 in Figs.
    ROC_K / ROC_CO): planned in the gather form (support W <= 1024); the schedule,
    windows and thresholds match the oracle's tables."""
    kw = dict(support=(w,)) if w else {}
    p = B.Plan(n, b, 4, seed=5, random_tau=True, **kw)
    assert p.mode == 1
    op = R.Params(n=n, b=b, loops=4, seed=5, random_tau=True, **kw)
    tb = R.make_tables(op)
    sig, _, tau = p.schedule()
    np.testing.assert_array_equal(sig, tb.sigma)
    np.testing.assert_array_equal(tau, tb.tau)
    be, ga = p.thresholds()
    for l in range(4):
        assert math.isclose(be[l], R.beta(op, tb, l), rel_tol=1e-9)


def test_device_calls_require_bind():
    p = B.Plan((64, 64), (8, 8), 2)
    with pytest.raises(B.RsftError) as e:
        p._need_bind()
    assert e.value.status == 7


def test_mode_resolution():
    assert B.Plan((1024, 256), (32, 16), 6, max_batch=4096).mode == 1          # fused
    assert B.Plan((2048, 512, 64), (64, 32, 8), 16).mode == 2                  # split
    assert B.Plan((4096,), (64,), 8, support=(512,)).mode == 1
    assert B.Plan((256, 256), (16, 16), 6, max_batch=1).mode == 2
    assert B.Plan((512, 128, 32), (32, 16, 8), 8).mode == 2


def test_new_entry_points_validate_before_any_launch():
    """rsft_run / rsft_bucketize_partial / rsft_finalize / rsft_design_thresholds: argument and
    state errors are returned before any CUDA call (no GPU needed)."""
    import ctypes
    L = B.lib()
    p = B.Plan((64, 32, 64), (8, 4, 8), 4)
    h = p.handle
    dummy = ctypes.c_void_p(256)
    assert L.rsft_bucketize_partial(h, None, 0, 8, dummy, None) == 1            # E_ARG
    assert L.rsft_bucketize_partial(h, dummy, 0, 8, dummy, None) == 7           # E_STATE (unbound)
    assert L.rsft_finalize(h, None, 0, 4, dummy, None, None) == 1
    assert L.rsft_finalize(h, dummy, 0, 4, dummy, None, None) == 7
    assert L.rsft_run(h, None, 1, dummy, dummy, dummy, 10, dummy, None) == 1
    assert L.rsft_run(h, dummy, 1, dummy, dummy, dummy, 10, dummy, None) == 7
    with pytest.raises(B.RsftError) as e:
        p.design_thresholds(K=100, loops=20)                                    # K eta_m >= B (Remark 2)
    assert e.value.status == 1
    with pytest.raises(B.RsftError):
        p.design_thresholds(K=2, p_d=1.5)
    r = p.design_thresholds(K=2, loops=20, omega=(3.5, 1.0, 7.25))
    assert 1 <= r["mu"] <= 20 and r["pfa_bar"] < r["pd_bar"] and r["gamma"] > 0


def test_survey_spelling_plan_and_destroy():
    """rsft_plan(params, device, out) / rsft_destroy (SURVEY §8(b) names) behave like
    rsft_plan_create / rsft_plan_destroy; bad device ids are argument errors."""
    import ctypes
    L = B.lib()
    p = B.RsftParams()
    L.rsft_default_params(ctypes.byref(p))
    p.ndim, p.n[0], p.b[0], p.loops = 1, 1024, 32, 4
    h = ctypes.c_void_p()
    assert L.rsft_plan(ctypes.byref(p), 0, ctypes.byref(h)) == 0 and h.value
    info = B.RsftInfo()
    assert L.rsft_get_info(h, ctypes.byref(info)) == 0 and info.ntot == 1024 and info.btot == 32
    L.rsft_destroy(h)
    h2 = ctypes.c_void_p()
    assert L.rsft_plan(ctypes.byref(p), -2, ctypes.byref(h2)) == 1
