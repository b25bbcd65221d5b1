"""T4 statistical tests on the GPU: properties the paper fixes that hold at full
size and that the oracle cannot check element by element at scale.
  * Eq. tpd (reading L8): on pure noise every loop's per-bucket exceedance rate
    is P_fa -- a binomial check over ~1.6e6 bucket trials;
  * K = 0 end to end: no location survives the second stage at the c4 design (P_fa = 1e-6,
    mu = L);
  * noiseless on-grid tones at full c4 / c2 sizes with a tiny gamma: every tone cell is
    detected (Prop. 3, reversibility P:437-441)."""
import math

import numpy as np
import pytest

import synth
from gpu_helpers import make_plan, oracle_params

pytestmark = pytest.mark.gpu


def test_pure_noise_first_stage_false_alarm_rate():
    import torch
    n, b, L, pfa = (1024, 256), (32, 16), 6, 1e-3
    frames = 512
    op = oracle_params(n, b, L, p_fa=pfa, noise_var=2.0, seed=31)
    plan = make_plan(op, max_batch=frames).bind()
    x = torch.from_numpy(synth.gen_noise_only((frames,) + n, 2.0, 17)).cuda()
    bm = plan.execute(x)
    torch.cuda.synchronize()
    words = bm.cpu().numpy().view(np.uint32)
    hits = np.unpackbits(words.view(np.uint8), bitorder="little").reshape(frames, L, -1)[:, :, : plan.btot]
    trials = frames * plan.btot
    for l in range(L):
        k = int(hits[:, l].sum())
        sd = math.sqrt(trials * pfa * (1 - pfa))
        assert abs(k - trials * pfa) <= 4.5 * sd, (l, k, trials * pfa, sd)
    k = int(hits.sum())
    assert abs(k - L * trials * pfa) <= 4.5 * math.sqrt(L * trials * pfa * (1 - pfa))


def test_pure_noise_no_detections_at_design_point():
    import torch
    wl = synth.C4
    frames = 256
    op = oracle_params(wl.n, wl.b, wl.loops, p_fa=wl.p_fa, noise_var=1.0, seed=wl.sched_seed)
    plan = make_plan(op, max_batch=frames).bind()
    x = torch.from_numpy(synth.gen_noise_only((frames,) + wl.n, 1.0, 23)).cuda()
    _, _, _, cnt = plan.run(x, 1 << 20)
    torch.cuda.synchronize()
    # per location P(all L loops fire) ~ P_fa^L ~ 1e-36: nothing may survive
    assert int(cnt.item()) == 0


@pytest.mark.parametrize("n,b,L", [((1024, 256), (32, 16), 6), ((256, 256), (16, 16), 6)])
def test_noiseless_ongrid_tones_all_detected_full_size(n, b, L):
    import torch
    rng = np.random.default_rng(8)
    K = 30
    bins = np.stack([rng.integers(0, n[0], K), rng.integers(0, n[1], K)], axis=1)
    amps = np.exp(2j * np.pi * rng.random(K))
    x = synth.gen_ongrid(n, bins, amps).astype(np.complex64)[None]
    op = oracle_params(n, b, L, gamma_override=1e-4, seed=13)   # below any non-cancelled tone bucket
    plan = make_plan(op, max_batch=1).bind()
    _, det, idx, cnt = plan.run(torch.from_numpy(x).cuda(), 1 << 20)
    torch.cuda.synchronize()
    got = set(idx.cpu().numpy()[: int(cnt.item())].tolist())
    for i0, i1 in bins:
        assert int(i0) * n[1] + int(i1) in got
