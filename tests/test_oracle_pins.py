"""Pins for the oracle (oracle/rsft_ref.py) against things other than itself: the paper's
and SPEC's worked examples, Props. 1-4, closed forms, library special cases, brute force on
tiny inputs, and statistical laws the paper states.  CPU only (-m "not gpu")."""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import rsft_ref as R
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def golden():
    with open(GOLD) as f:
        return json.load(f)


# ---------------------------------------------------------------- worked examples
def test_spec_worked_examples():
    g = golden()
    for e in g["mod_inverse"]:
        assert R.mod_inverse(e["sigma"], e["n"]) == e["inv"]
    with pytest.raises(ValueError):
        R.mod_inverse(4, 8)                                   # S:184 NonInvertible
    for e in g["permute"]:
        assert list(R.permute(np.array(e["x"]), e["sigma"], e["tau"])) == e["out"]
    for e in g["alias"]:
        assert list(R.fold(np.array(e["x"]), e["b"])) == e["out"]
    for e in g["map_index"]:
        assert R.map_index(e["i"], e["sigma"], e["n"], e["b"]) == e["out"]
    for e in g["reverse_map"]:
        assert sorted(R.reverse_map(e["j"], e["sigma_inv"], e["n"], e["b"])) == e["out"]
    for e in g["accumulate"]:
        p = R.Params(n=(e["n"],), b=(e["b"],), loops=1, prewin="rect")
        tb = R.Tables([np.ones(e["n"])], [np.ones(e["n"])], np.array([[e["sigma"]]]),
                      np.array([[R.mod_inverse(e["sigma"], e["n"])]]), np.array([[0]]))
        c = np.zeros(e["b"], dtype=bool)
        c[e["marked"]] = True
        abar = R.accumulate([c], p, tb)
        want = np.zeros(e["n"], dtype=np.int32)
        for k, v in e["counts_at"].items():
            want[int(k)] = v
        assert np.array_equal(abar, want)


def test_fig_permutation_example():
    e = golden()["fig_permutation"]
    x = (8 * np.arange(4)[:, None] + np.arange(8)[None, :]).astype(np.float64)
    p = R.permute_nd(x, e["sigma"], [0, 0])
    assert np.array_equal(p, np.array(e["permuted"]))
    assert np.array_equal(R.fold_nd(p, e["b"]), np.array(e["folded"]))


def test_splitmix64_reference_vector():
    # SplitMix64 (Steele/Lea/Flood; reading L5) seeded with 0: published first outputs.
    assert R.splitmix64(0, 0) == 0xE220A8397B1DCDAF
    assert R.splitmix64(0, 1) == 0x6E789E6AA1B965F4
    assert R.splitmix64(0, 2) == 0x06C45D188009454F


def test_schedule_properties():
    p = R.Params(n=(1024, 256, 2), b=(32, 16, 2), loops=40, seed=7, random_tau=True)
    sig, sinv, tau = R.schedule(p)
    for l in range(p.loops):
        for d, n in enumerate(p.n):
            assert sig[l, d] % 2 == 1 and 0 < sig[l, d] < n        # P:728 odd sigma
            assert (sig[l, d] * sinv[l, d]) % n == 1                 # Eq. mod_inv
            assert 0 <= tau[l, d] < n
    assert np.all(sig[:, 2] == 1)
    s2, _, _ = R.schedule(p)
    assert np.array_equal(sig, s2)                                   # deterministic
    q = R.Params(n=(1024,), b=(32,), loops=4, seed=7)
    assert np.all(R.schedule(q)[2] == 0)                             # tau = 0
    # uniformity over odd residues: chi^2 on 4000 draws of N=16
    r = R.Params(n=(16,), b=(4,), loops=4000, seed=3)
    s, _, _ = R.schedule(r)
    counts = np.bincount((s[:, 0] - 1) // 2, minlength=8)
    chi2 = float(((counts - 500.0) ** 2 / 500.0).sum())
    assert chi2 < 24.3                                               # p = 0.001, 7 dof


# ---------------------------------------------------------------- Props. 1-4
def test_props_3_4_exhaustive():
    """Reversibility (Prop. 3) and distinctiveness (Prop. 4), n=64, b=16, all odd sigma
    (acceptance 3 S:598); the reverse maps partition [n]."""
    n, b = 64, 16
    for s in range(1, n, 2):
        si = R.mod_inverse(s, n)
        sets = [set(R.reverse_map(j, si, n, b)) for j in range(b)]
        for i in range(n):
            assert i in sets[R.map_index(i, s, n, b)]
        for i, j in itertools.combinations(range(b), 2):
            assert not (sets[i] & sets[j])
        assert set().union(*sets) == set(range(n))
        assert all(len(x) == n // b for x in sets)


def test_property1_permutation_dilation():
    """Prop. 1 with the corrected phase e^{+j 2 pi tau i / N} (reading L6)."""
    rng = np.random.default_rng(0)
    n = 64
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    X = np.fft.fft(x)
    for s in (1, 3, 5, 27, 63):
        for tau in (0, 1, 17):
            P = np.fft.fft(R.permute(x, s, tau))
            i = np.arange(n)
            np.testing.assert_allclose(P[(s * i) % n], X * np.exp(2j * np.pi * tau * i / n),
                                       rtol=1e-10, atol=1e-10)


def test_property2_aliasing():
    """Prop. 2: DFT_B(alias(x))_i = DFT_N(x)_{iL}; n=64, b=8."""
    rng = np.random.default_rng(1)
    x = rng.standard_normal(64) + 1j * rng.standard_normal(64)
    np.testing.assert_allclose(np.fft.fft(R.fold(x, 8)), np.fft.fft(x)[::8], rtol=1e-10, atol=1e-10)
    # N-D version + Parseval on the folded grid
    y = rng.standard_normal((16, 32)) + 1j * rng.standard_normal((16, 32))
    f = R.fold_nd(y, (4, 8))
    np.testing.assert_allclose(np.fft.fftn(f), np.fft.fftn(y)[::4, ::4], rtol=1e-10, atol=1e-9)
    assert math.isclose(np.sum(np.abs(np.fft.fftn(f)) ** 2), f.size * np.sum(np.abs(f) ** 2), rel_tol=1e-12)


def test_fftn_matches_direct_dft():
    """The library N-D FFT step (reading L7: forward, unnormalised) equals the
    explicit O(N^2) DFT sums."""
    rng = np.random.default_rng(2)
    for shape in [(8,), (4, 8), (2, 4, 4)]:
        x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        np.testing.assert_allclose(np.fft.fftn(x), R.dft_direct(x), rtol=1e-10, atol=1e-10)


# ---------------------------------------------------------------- windows
@pytest.mark.parametrize("m", [9, 33, 65, 513, 1025])
def test_dolph_chebyshev_matches_scipy(m):
    from scipy.signal.windows import chebwin
    for att in (40.0, 60.0):
        np.testing.assert_allclose(R.dolph_chebyshev(m, att), chebwin(m, att), rtol=0, atol=1e-12)


def test_dolph_chebyshev_equiripple_sidelobes():
    """Equiripple sidelobes at -A dB (within +-0.5 dB), symmetric, peak 1."""
    for m, att in [(1025, 40.0), (257, 60.0)]:
        w = R.dolph_chebyshev(m, att)
        assert w.max() == 1.0 and np.allclose(w, w[::-1], atol=1e-14)
        spec = np.abs(np.fft.fft(w, 16 * m))
        spec = 20 * np.log10(spec / spec.max() + 1e-300)
        k = 1
        while spec[k + 1] < spec[k]:        # walk down the main lobe to the first null
            k += 1
        side = spec[k:len(spec) // 2].max()
        assert -att - 0.5 <= side <= -att + 0.5


def test_hann_periodic_closed_form():
    """Periodic Hann is DFT-even: exactly three nonzero bins N(1/2, -1/4, -1/4) (L3)."""
    for n in (16, 256, 1024):
        W = np.fft.fft(R.hann_periodic(n))
        want = np.zeros(n, dtype=complex)
        want[0], want[1], want[-1] = n / 2, -n / 4, -n / 4
        np.testing.assert_allclose(W, want, atol=1e-9)


@pytest.mark.parametrize("n,b,w", [(256, 16, 0), (1024, 32, 0), (4096, 64, 512), (64, 8, 0)])
def test_flat_window_response(n, b, w):
    """Flat window (L1-L2): DFT(gbar) is a boxcar of width A=N/B bins placed so that
    permuted bin m lands in bucket floor(m/A) (Def. 3 floor): centre of the bucket at
    0 dB, the bucket edge at -6.02 dB (inherent to a real even prototype), and far other
    buckets attenuated."""
    a = n // b
    G = np.fft.fft(R.flat_window(n, b, w, 60.0))
    resp = lambda k, m: abs(G[(k * a - m) % n])        # contribution of bin m to bucket k
    ref = resp(0, a // 2)
    assert abs(20 * math.log10(resp(0, 0) / ref) + 6.02) < 0.05          # edge bin: -6 dB
    assert abs(20 * math.log10(resp(-1 % b, 0) / ref) + 6.02) < 0.05     # ... in both buckets
    if w == 0:                                                           # full support
        for m in range(2, a - 1):
            assert abs(20 * math.log10(resp(0, m) / ref)) < 1.0          # passband
        for m in range(a):
            for k in range(1, b):
                lo = k * a
                dist = min(min(abs(u - m), n - abs(u - m)) for u in (lo, lo + a - 1))
                if dist >= 4:
                    assert 20 * math.log10(resp(k, m) / ref + 1e-300) < -55.0
    assert np.allclose(R.flat_window(64, 64, 0, 60.0), 1.0)              # B == N


# ---------------------------------------------------------------- first stage
def _rand_params(n, b, loops=3, support=(), seed=11, prewin="hann"):
    return R.Params(n=n, b=b, loops=loops, support=support, prewin=prewin, seed=seed,
                    random_tau=True, noise_var=1.0, p_fa=1e-3)


@pytest.mark.parametrize("n,b,support", [((32,), (4,), ()), ((32,), (4,), (16,)),
                                         ((8, 16), (2, 4), ()), ((4, 8, 8), (2, 2, 4), ())])
def test_first_stage_equals_dense_matrix(n, b, support):
    """f^ = D V_sigma r with explicit dense matrices (Eqs. l, f): pins the
    permutation direction, window order, fold and FFT sign/normalisation."""
    p = _rand_params(n, b, support=support)
    tb = R.make_tables(p)
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    for l in range(p.loops):
        M = R.first_stage_matrix(p, tb, l)
        want = (M @ x.astype(np.complex128).ravel()).reshape(b)
        got = R.first_stage(x, p, tb, l).fhat
        np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-10)


def test_beta_is_bucket_noise_variance():
    """Eq. var_fu: under white noise every bucket has variance sigma_n^2 beta; in
    closed form every row of D V_sigma has squared norm beta."""
    for n, b, sup in [((32,), (4,), ()), ((8, 16), (2, 4), ()), ((64,), (8,), (16,))]:
        p = _rand_params(n, b, support=sup)
        tb = R.make_tables(p)
        for l in range(p.loops):
            M = R.first_stage_matrix(p, tb, l)
            be = R.beta(p, tb, l)
            np.testing.assert_allclose(np.sum(np.abs(M) ** 2, axis=1), be, rtol=1e-10)
            # literal N-D norm ||Wbar P_sigma w||^2 equals the separable product
            wv = R.outer_nd(tb.prewin)
            lit = np.sum(np.abs(R.outer_nd(tb.flat) * R.permute_nd(wv, tb.sigma[l], tb.tau[l])) ** 2)
            assert math.isclose(lit, be, rel_tol=1e-12)


def test_brickwall_identity_direct_dft():
    """I4: with the ideal brick-wall flat window, f^_k = sum_{i: M(i,sigma)=k} y^_i
    e^{+j 2 pi tau . i / N} (Props. 1-2, Def. 3), y^ from the explicit O(N^2) DFT."""
    for n, b in [((16,), (4,)), ((8, 16), (2, 4))]:
        p = _rand_params(n, b)
        tb = R.make_tables(p, flat_override=[R.brickwall_window(nn, bb) for nn, bb in zip(n, b)])
        rng = np.random.default_rng(9)
        x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
        yhat = R.dft_direct(x.astype(np.complex128) * R.outer_nd(tb.prewin))
        for l in range(p.loops):
            want = np.zeros(b, dtype=np.complex128)
            for i in itertools.product(*[range(v) for v in n]):
                k = tuple(R.map_index(i[d], int(tb.sigma[l, d]), n[d], b[d]) for d in range(len(n)))
                ph = sum(int(tb.tau[l, d]) * i[d] / n[d] for d in range(len(n)))
                want[k] += yhat[i] * np.exp(2j * np.pi * ph)
            np.testing.assert_allclose(R.first_stage(x, p, tb, l).fhat, want, rtol=1e-9, atol=1e-9)


def test_brickwall_identity_large():
    n, b = (64, 32, 16), (8, 4, 4)
    p = _rand_params(n, b, loops=2)
    tb = R.make_tables(p, flat_override=[R.brickwall_window(nn, bb) for nn, bb in zip(n, b)])
    x = synth.gen_noise_only(n, 1.0, 3)
    yhat = np.fft.fftn(x.astype(np.complex128) * R.outer_nd(tb.prewin))
    for l in range(p.loops):
        idx = np.ix_(*[((np.arange(n[d]) * int(tb.sigma[l, d])) % n[d]) * b[d] // n[d] for d in range(3)])
        ph = R.outer_nd([np.exp(2j * np.pi * int(tb.tau[l, d]) * np.arange(n[d]) / n[d]) for d in range(3)])
        want = np.zeros(b, dtype=np.complex128)
        np.add.at(want, tuple(np.broadcast_arrays(*idx)), yhat * ph)
        np.testing.assert_allclose(R.first_stage(x, p, tb, l).fhat, want, rtol=1e-9, atol=1e-8)


def test_false_alarm_rate_pure_noise():
    """Eq. tpd: on pure noise the per-bucket exceedance of
    gamma = sigma_n^2 beta ln(1/P_fa) is P_fa, within a 4-sigma binomial interval."""
    p = R.Params(n=(64, 32), b=(8, 8), loops=40, p_fa=0.02, noise_var=2.0, seed=4)
    tb = R.make_tables(p)
    hits = trials = 0
    for frame in range(8):
        x = synth.gen_noise_only(p.n, p.noise_var, 100 + frame)
        for l in range(p.loops):
            st = R.first_stage(x, p, tb, l)
            hits += int(st.c.sum())
            trials += st.c.size
    rate = hits / trials
    sd = math.sqrt(p.p_fa * (1 - p.p_fa) / trials)
    assert abs(rate - p.p_fa) < 4 * sd, (rate, trials)


# ---------------------------------------------------------------- second stage
def test_accumulate_equals_lookup_form():
    """Literal Def. 4 accumulation == I1 hash lookup (Props. 3-4) on random bitmaps."""
    rng = np.random.default_rng(3)
    for n, b in [((64,), (8,)), ((32, 16), (4, 8)), ((16, 8, 8), (4, 2, 4))]:
        p = R.Params(n=n, b=b, loops=5, seed=21)
        tb = R.make_tables(p)
        cs = [rng.random(b) < 0.3 for _ in range(p.loops)]
        np.testing.assert_array_equal(R.accumulate(cs, p, tb), R.vote_lookup(cs, p, tb))


def test_accumulate_all_and_none():
    p = R.Params(n=(32, 16), b=(4, 8), loops=3, seed=2)
    tb = R.make_tables(p)
    assert np.all(R.accumulate([np.ones(p.b, bool)] * 3, p, tb) == 3)   # partition (Prop. 4)
    assert np.all(R.accumulate([np.zeros(p.b, bool)] * 3, p, tb) == 0)
    o, idx = R.second_stage(np.array([0, 3, 2, 3]), 3)
    assert list(idx) == [1, 3] and len(R.second_stage(np.array([3]), 4)[1]) == 0


# ---------------------------------------------------------------- end to end
def test_end_to_end_noiseless_ongrid_brickwall():
    """Noiseless on-grid tones, RECT pre-window, brick-wall flat window: closed form
    f^_k = N_tot sum_{tones i: M(i,sigma)=k} a_i e^{+j2 pi tau.i/N}; with a tiny gamma the
    detected set equals the DFT-only prediction {i : #{l : bucket M_l(i) holds a tone} >= mu}
    and contains the truth (Prop. 3)."""
    n, b = (64, 32), (8, 4)
    p = R.Params(n=n, b=b, loops=5, prewin="rect", gamma_override=1e-6, seed=8, random_tau=True)
    tb = R.make_tables(p, flat_override=[R.brickwall_window(nn, bb) for nn, bb in zip(n, b)])
    rng = np.random.default_rng(12)
    bins = np.stack([rng.integers(0, n[0], 6), rng.integers(0, n[1], 6)], axis=1)
    amps = np.exp(2j * np.pi * rng.random(6))
    x = synth.gen_ongrid(n, bins, amps)
    res = R.rsft_run(x, p, tb)
    ntot = n[0] * n[1]
    for l, st in enumerate(res.stages):
        want = np.zeros(b, dtype=np.complex128)
        for (i0, i1), a in zip(bins, amps):
            k = (R.map_index(i0, int(tb.sigma[l, 0]), n[0], b[0]), R.map_index(i1, int(tb.sigma[l, 1]), n[1], b[1]))
            want[k] += ntot * a * np.exp(2j * np.pi * (tb.tau[l, 0] * i0 / n[0] + tb.tau[l, 1] * i1 / n[1]))
        np.testing.assert_allclose(st.fhat, want, rtol=1e-9, atol=1e-7)
    # DFT-only prediction (no permute / fold code): occupied cells of the dense DFT
    occ = np.abs(np.fft.fft2(x)) > 1e-3
    pred = np.zeros(n, dtype=np.int32)
    for l in range(p.loops):
        m0 = ((np.arange(n[0]) * int(tb.sigma[l, 0])) % n[0]) * b[0] // n[0]
        m1 = ((np.arange(n[1]) * int(tb.sigma[l, 1])) % n[1]) * b[1] // n[1]
        full = np.zeros(b, dtype=bool)
        for i0, i1 in zip(*np.nonzero(occ)):
            full[m0[i0], m1[i1]] = True
        pred += full[np.ix_(m0, m1)]
    np.testing.assert_array_equal(res.detect, pred >= p.mu)
    for i0, i1 in bins:
        assert res.detect[i0, i1]


def test_end_to_end_hann_real_flat_window_truth_recovered():
    """Realistic windows, noiseless on-grid tones, small gamma: every tone's grid cell is
    detected in every loop (Prop. 3 + Claim 1), so truth is a subset of o with mu = L."""
    n, b = (128, 64), (16, 8)
    p = R.Params(n=n, b=b, loops=4, gamma_override=1e-3, seed=5)
    tb = R.make_tables(p)
    rng = np.random.default_rng(4)
    bins = np.stack([rng.integers(0, n[0], 5), rng.integers(0, n[1], 5)], axis=1)
    x = synth.gen_ongrid(n, bins, np.exp(2j * np.pi * rng.random(5)))
    res = R.rsft_run(x, p, tb)
    for i0, i1 in bins:
        assert res.detect[i0, i1]
    assert res.detect.sum() < res.detect.size // 4


def test_claim1_peak_bucket():
    """Claim 1: a single on-grid tone at bin i peaks in bucket
    floor(B [sigma i]_N / N) when it is not on a bucket edge (reading L1/L14)."""
    n, b = 1024, 64
    p = R.Params(n=(n,), b=(b,), loops=20, prewin="rect", seed=13)
    tb = R.make_tables(p)
    rng = np.random.default_rng(6)
    checked = 0
    for i in rng.integers(0, n, 10):
        x = synth.gen_ongrid((n,), [[i]], [1.0])
        for l in range(p.loops):
            s = int(tb.sigma[l, 0])
            if ((s * i) % n) % (n // b) in (0, n // b - 1):
                continue
            st = R.first_stage(x, p, tb, l)
            assert int(np.argmax(np.abs(st.fhat))) == R.map_index(int(i), s, n, b)
            checked += 1
    assert checked > 100


def test_scale_invariance():
    """|c|^2 scaling: detections on c*x with gamma*|c|^2 equal those on x."""
    wl = synth.C2.with_(n=(64, 64), b=(8, 8))
    x = synth.gen_frame(wl, 0)
    p1 = R.Params(n=wl.n, b=wl.b, loops=4, gamma_override=50.0, seed=1)
    c = 3.0 - 4.0j
    p2 = R.Params(n=wl.n, b=wl.b, loops=4, gamma_override=50.0 * abs(c) ** 2, seed=1)
    r1 = R.rsft_run(x, p1)
    r2 = R.rsft_run(x.astype(np.complex128) * c, p2)
    np.testing.assert_array_equal(r1.abar, r2.abar)
