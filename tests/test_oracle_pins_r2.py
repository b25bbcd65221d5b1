"""Round-2 pins for the oracle functions the round-1 review found unpinned (VERDICT r1
"What's weak" 1): the periodic Chebyshev pre-window, segment mode, and the comparators
themselves (each must REJECT a wrong answer, not only accept a right one).  CPU only."""
import numpy as np
import pytest

from oracle import rsft_ref as R
import synth


# ---------------------------------------------------------------- cheb_periodic
@pytest.mark.parametrize("n,at", [(16, 40.0), (64, 60.0), (256, 40.0), (1024, 60.0), (4096, 80.0)])
def test_cheb_periodic_equals_scipy_periodic_chebwin(n, at):
    """The paper's pre-window is a Dolph-Chebyshev window; the DFT-even
    (periodic) form is the (N+1)-point symmetric window with its last sample dropped, which is
    exactly scipy's ``chebwin(N, at, sym=False)`` (an independent implementation)."""
    from scipy.signal.windows import chebwin
    got = R.cheb_periodic(n, at)
    want = chebwin(n, at, sym=False)
    assert got.shape == (n,)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


def test_cheb_periodic_is_dft_even():
    """Periodic window: w[n] == w[N - n] for n = 1..N-1 (a one-sample shift breaks it) and
    the peak (1.0) sits at n = N/2."""
    for n in (32, 512):
        w = R.cheb_periodic(n, 60.0)
        np.testing.assert_allclose(w[1:], w[1:][::-1], rtol=0, atol=1e-13)
        assert int(np.argmax(w)) == n // 2 and abs(w[n // 2] - 1.0) < 1e-15


def test_prewindow_cheb_routes_to_periodic_chebwin():
    from scipy.signal.windows import chebwin
    p = R.Params(n=(64, 32), b=(8, 4), loops=2, prewin="cheb", prewin_param=50.0)
    for d in range(2):
        np.testing.assert_allclose(R.prewindow(p, d), chebwin(p.n[d], 50.0, sym=False), atol=1e-12)


# ---------------------------------------------------------------- rsft_run_segments
def _seg_case(seed=3, n=(64, 32), b=(8, 4), L=5):
    p = R.Params(n=n, b=b, loops=L, p_fa=1e-3, seed=seed, random_tau=True, mu=3)
    tb = R.make_tables(p)
    wl = synth.Workload("segpin", n, b, L, 1e-3, 1.0, (2, 4), (5.0, 20.0), L, data_seed=seed)
    xs = synth.gen_batch(wl, range(L))
    return p, tb, xs


def test_segments_identical_equal_same_frame_run():
    """with every segment equal to r, "iterations on different segments" IS the
    same-frame algorithm -> identical stages, votes and detections."""
    p, tb, xs = _seg_case()
    same = np.stack([xs[0]] * p.loops)
    a = R.rsft_run_segments(same, p, tb)
    b = R.rsft_run(xs[0], p, tb)
    for sa, sb in zip(a.stages, b.stages):
        assert np.array_equal(sa.fhat, sb.fhat) and np.array_equal(sa.c, sb.c)
    assert np.array_equal(a.abar, b.abar) and np.array_equal(a.detect, b.detect)
    assert np.array_equal(a.idx, b.idx)


def test_segments_loop_l_reads_segment_l():
    """Swapping segments i and j changes only loops i and j, and loop i then equals the
    same-frame first stage of loop i on segment j (the segment index follows the loop)."""
    p, tb, xs = _seg_case(seed=5)
    i, j = 1, 3
    sw = xs.copy()
    sw[[i, j]] = sw[[j, i]]
    a = R.rsft_run_segments(xs, p, tb)
    b = R.rsft_run_segments(sw, p, tb)
    for l in range(p.loops):
        if l in (i, j):
            continue
        assert np.array_equal(a.stages[l].fhat, b.stages[l].fhat)
    ri = R.rsft_run(xs[j], p, tb)
    assert np.array_equal(b.stages[i].fhat, ri.stages[i].fhat)
    assert not np.allclose(a.stages[i].fhat, b.stages[i].fhat)


def test_segments_votes_are_sum_of_per_loop_votes():
    """Eq. a_i: the segment-mode vote count is the sum over loops of the Def. 4
    reverse-maps of each loop's bits; check against the I1 lookup form per loop."""
    p, tb, xs = _seg_case(seed=7)
    a = R.rsft_run_segments(xs, p, tb)
    total = np.zeros(p.n, dtype=np.int32)
    for l, st in enumerate(a.stages):
        one = R.Tables(tb.prewin, tb.flat, tb.sigma[l:l + 1], tb.sigma_inv[l:l + 1], tb.tau[l:l + 1])
        pl = R.Params(n=p.n, b=p.b, loops=1, p_fa=p.p_fa, seed=p.seed)
        total += R.vote_lookup([st.c], pl, one)
    assert np.array_equal(a.abar, total)
    assert np.array_equal(a.detect, total >= p.mu)


# ---------------------------------------------------------------- comparators must reject
def _run_case():
    p = R.Params(n=(64, 32), b=(8, 4), loops=4, p_fa=1e-2, seed=11, mu=3)
    tb = R.make_tables(p)
    wl = synth.Workload("cmp", p.n, p.b, p.loops, 1e-2, 1.0, (3, 5), (5.0, 20.0), 1, data_seed=9)
    x = synth.gen_frame(wl, 0)
    return p, tb, x, R.rsft_run(x, p, tb)


def test_compare_buckets_rejects_perturbation():
    p, tb, x, res = _run_case()
    st = res.stages[0]
    px = float(np.mean(np.abs(x.astype(np.complex128)) ** 2))
    scale = np.maximum(np.abs(st.fhat), np.sqrt(st.beta * px))
    assert R.compare_buckets(st.fhat.copy(), st, px)["ok"]
    k = np.unravel_index(int(np.argmax(np.abs(st.fhat))), st.fhat.shape)
    for rel, ok in ((0.5e-4, True), (2e-4, False)):
        g = st.fhat.copy()
        g[k] += rel * scale[k]
        assert R.compare_buckets(g, st, px)["ok"] is ok, rel
    g = st.fhat.copy()                                      # a wrong sign on one small bucket
    kk = np.unravel_index(int(np.argmin(np.abs(st.fhat))), st.fhat.shape)
    g[kk] = -g[kk] + 3e-4 * scale[kk]
    assert not R.compare_buckets(g, st, px)["ok"]


def test_compare_bits_rejects_flip_outside_band_only():
    p, tb, x, res = _run_case()
    st = res.stages[1]
    assert R.compare_bits(st.c.copy(), st)["ok"]
    clear = np.flatnonzero(~st.ambiguous.ravel())
    g = st.c.copy().ravel()
    g[clear[0]] = ~g[clear[0]]
    r = R.compare_bits(g.reshape(st.c.shape), st)
    assert not r["ok"] and r["mismatch"] == 1
    # a bucket exactly on the threshold is ambiguous: flipping it is allowed (L16)
    pw = np.abs(st.fhat) ** 2
    k = int(np.argmax(pw.ravel()))
    on = R.FirstStage(st.f, st.fhat, st.beta, float(pw.ravel()[k]), pw > pw.ravel()[k],
                      np.abs(pw - pw.ravel()[k]) <= R.AMBIGUITY_REL * pw.ravel()[k])
    g2 = on.c.copy().ravel()
    g2[k] = ~g2[k]
    assert on.ambiguous.ravel()[k] and R.compare_bits(g2.reshape(st.c.shape), on)["ok"]


def test_compare_sets_rejects_missing_and_extra():
    p, tb, x, res = _run_case()
    assert R.compare_sets(res.detect.copy(), res, p.mu)["ok"]
    sure = np.flatnonzero((res.abar_min >= p.mu).ravel())
    never = np.flatnonzero((res.abar_max < p.mu).ravel())
    assert sure.size and never.size
    g = res.detect.copy().ravel()
    g[sure[0]] = False
    r = R.compare_sets(g.reshape(p.n), res, p.mu)
    assert not r["ok"] and r["missing"] == 1
    g = res.detect.copy().ravel()
    g[never[0]] = True
    r = R.compare_sets(g.reshape(p.n), res, p.mu)
    assert not r["ok"] and r["extra"] == 1
