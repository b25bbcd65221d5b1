"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI and compare
with the oracle frame by frame (SURVEY §8(c) comparison rules)."""
import numpy as np

from oracle import rsft_ref as R
from paper_1610_01050_b200 import rsft as B


def oracle_params(n, b, loops, **kw):
    return R.Params(n=tuple(n), b=tuple(b), loops=loops, **kw)


def make_plan(op: R.Params, max_batch=1, mode="auto"):
    return B.Plan(op.n, op.b, op.loops, support=op.support, prewin=op.prewin, prewin_param=op.prewin_param,
                  flat_atten_db=op.flat_atten_db, p_fa=op.p_fa, noise_var=op.noise_var,
                  gamma_override=op.gamma_override, mu=op.mu, seed=op.seed, random_tau=op.random_tau,
                  max_batch=max_batch, mode=mode)


def gpu_run(plan, x_np, spectra=True, counts=True, capacity=None):
    import torch
    x = torch.from_numpy(np.ascontiguousarray(x_np)).cuda()
    batch = x.shape[0]
    sp = torch.empty((batch, plan.loops, plan.btot), dtype=torch.complex64, device="cuda") if spectra else None
    bm = plan.execute(x, spectra=sp)
    ct = torch.empty((batch, plan.ntot), dtype=torch.uint8, device="cuda") if counts else None
    det = plan.detect(bm, counts=ct)
    det_fast = plan.detect(bm)              # no counts: AND (mu = L) / OR (mu = 1) fast paths
    cap = capacity if capacity is not None else batch * plan.ntot
    idx, cnt = plan.compact(det, cap)
    det_f, idx_f, cnt_f = plan.detect_compact(bm, cap)      # vote + compaction in one call
    bm_r, det_r, idx_r, cnt_r = plan.run(x, cap)             # whole path (fused vote in fused mode)
    torch.cuda.synchronize()
    count = int(cnt.item())
    assert int(cnt_f.item()) == count
    np.testing.assert_array_equal(det_f.cpu().numpy(), det.cpu().numpy())
    np.testing.assert_array_equal(idx_f.cpu().numpy()[:min(count, cap)], idx.cpu().numpy()[:min(count, cap)])
    # rsft_run: fused-mode plans fold + FFT + vote in one kernel whose FFT order differs from
    # rsft_execute's (equal to fp32 rounding).  Its bits must equal execute's except inside the
    # 1e-3 near-threshold band; with equal bits, every output must be identical.
    bm_np, bmr_np = bm.cpu().numpy(), bm_r.cpu().numpy()
    if not np.array_equal(bmr_np, bm_np):
        assert sp is not None, "rsft_run bitmaps differ from rsft_execute's (no spectra to check the band)"
        _, gam = plan.thresholds()
        diff = B.bitmap_to_bool((bmr_np ^ bm_np).reshape(-1), bm_np.size * 32).reshape(batch, plan.loops, -1)
        diff = diff[:, :, :plan.btot]
        f_, l_, k_ = np.nonzero(diff)
        pw = np.abs(sp.cpu().numpy()[f_, l_, k_].astype(np.complex128)) ** 2
        rel = np.abs(pw / gam[l_] - 1.0)
        assert (rel < 1e-3).all(), ("rsft_run bits outside the near-threshold band", rel.max())
    else:
        assert int(cnt_r.item()) == count
        np.testing.assert_array_equal(det_r.cpu().numpy(), det.cpu().numpy())
        np.testing.assert_array_equal(idx_r.cpu().numpy()[:min(count, cap)], idx.cpu().numpy()[:min(count, cap)])
    return {
        "bm": bm.cpu().numpy(),
        "spectra": sp.cpu().numpy() if sp is not None else None,
        "det": det.cpu().numpy(),
        "det_fast": det_fast.cpu().numpy(),
        "counts": ct.cpu().numpy() if ct is not None else None,
        "idx": idx.cpu().numpy()[:min(count, cap)],
        "count": count,
    }


def check_frame(res, f, x, op, tb, loops=None, check_counts=True):
    """Element-wise parity of frame f: buckets (1e-4 rel. with noise floor), first-stage bits
    outside the 1e-3 band, vote counts within [abar_min, abar_max], detection set envelope.
    Returns a small report dict."""
    ref = R.rsft_run(x, op, tb, loops=loops)
    px = float(np.mean(np.abs(x.astype(np.complex128)) ** 2))
    rep = {"max_ratio": 0.0, "ambiguous": 0, "bit_mismatch": 0}
    for i, st in enumerate(ref.stages):
        l = i if loops is None else list(loops)[i]
        if res["spectra"] is not None:
            got = res["spectra"][f, l].reshape(op.b)
            if px == 0.0:
                assert np.all(got == 0)
            else:
                cb = R.compare_buckets(got, st, px)
                rep["max_ratio"] = max(rep["max_ratio"], cb["max_ratio"])
                assert cb["ok"], (f, l, cb)
        bits = B.bitmap_to_bool(res["bm"][f, l], int(np.prod(op.b))).reshape(op.b)
        cbits = R.compare_bits(bits, st)
        rep["ambiguous"] += cbits["ambiguous"]
        assert cbits["ok"], (f, l, cbits)
    if loops is None:
        ntot = int(np.prod(op.n))
        det = B.bitmap_to_bool(res["det"][f], ntot).reshape(op.n)
        cs = R.compare_sets(det, ref, op.mu)
        assert cs["ok"], (f, cs)
        if check_counts and res["counts"] is not None:
            c = res["counts"][f].reshape(op.n).astype(np.int32)
            assert np.all(c >= ref.abar_min) and np.all(c <= ref.abar_max)
            assert np.array_equal(det, c >= op.mu)
        rep["detections"] = int(det.sum())
    return rep


def check_index_list(res, ntot, batch):
    """The compacted list equals the set bits of the detection bitmap, ascending."""
    np.testing.assert_array_equal(res["det"], res["det_fast"])
    bits = B.bitmap_to_bool(res["det"].reshape(-1), ntot * batch)
    want = np.flatnonzero(bits).astype(np.int64)
    assert res["count"] == want.size
    np.testing.assert_array_equal(res["idx"], want[: res["idx"].size])
