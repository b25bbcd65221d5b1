"""NEXT-2 studies at the paper's design point, on the GPU path.

Setting (§V): N = 1024, T = 50, B = 64, P_d = 0.9, P_fa = 1e-6, the weakest
sinusoid at omega_m = 64.5 bins, Dolph-Chebyshev 40 dB pre-window, flat window built on the same
taper (L2 with a 40 dB taper), sigma_n^2 = 1, Swerling amplitudes per segment in segment
mode.  (gamma*, mu*, SNR_min*) come from Eq. opt (rsft_design_thresholds, NEXT-1).

  per_sigma_detection -- the first-stage detection probability of the tone's bucket for EVERY
      odd sigma (all 512), measured by Monte Carlo; Eq. tpd predicts
      P~_d(omega_m, sigma) = exp(-gamma / (sigma_n^2 beta(sigma) + SNR alpha(p, omega_m, sigma)))
      with alpha, beta of Eq. alpha_beta -- the oracle computes those.
  approx_error -- Fig. varAppErr: (T Pd_bar (1 - Pd_bar) - sigma_a1^2) / sigma_a1^2,
      sigma_a1^2 = sum_s P~_d(sigma_s) (1 - P~_d(sigma_s)) (Eq. var_a1) for T random
      permutations, averaged over 100 draws, T in {10, 50, 100, 200}; Pd_bar = E_sigma P~_d.
  fixed_schedule_votes -- Eq. var_a1 end to end: one seeded T = 50 schedule, the vote count
      abar_i of the tone's location (rsft_detect counts) over many frames; its sample mean and
      variance against sum_s P~_d and sum_s P~_d (1 - P~_d) and the bound T Pd_bar (1 - Pd_bar).
  detector_at_design -- the two-stage detector with (gamma*, mu*) at T = 50, K = 4 tones at
      SNR_min*: measured P_d and P_fa against the targets and the exact-Binomial model.

`python tests/study_next2.py` (GPU) writes profiles/r02_next2.{md,json}; tests/test_gpu_montecarlo.py
runs reduced versions with assertions.  The oracle (closed forms) is test infrastructure.
"""
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

N, BK, T_PAPER, OMEGA, LOC = 1024, 64, 50, 64.5, 64
WIN = dict(prewin="cheb", prewin_param=40.0, flat_atten_db=40.0)


def design(T=T_PAPER, K=4, p_d=0.9, p_fa=1e-6):
    from paper_1610_01050_b200 import rsft as B
    probe = B.Plan((N,), (BK,), T, **WIN)
    return probe.design_thresholds(K=K, p_d=p_d, p_fa=p_fa, omega=(OMEGA,), loops=T)


def oracle_alpha_beta():
    """alpha(p, omega_m, sigma), beta(sigma) for every odd sigma (oracle first stage)."""
    from oracle import rsft_ref as R
    from oracle import thresholds as TH
    p = R.Params(n=(N,), b=(BK,), loops=1, prewin="cheb", prewin_param=40.0, flat_atten_db=40.0)
    sig = np.arange(1, N, 2)
    a, b = TH.alpha_beta_1d(p, OMEGA, sig)
    return sig, a, b


def tpd(alpha, beta, gamma, snr):
    """Eq. tpd with sigma_n^2 = 1."""
    return np.exp(-gamma / (beta + snr * alpha))


def bucket_of(sig, loc=LOC):
    """M_sigma(loc) = floor(B [sigma loc]_N / N) (Def. 3)."""
    return ((np.asarray(sig) * loc) % N) * BK // N


def _tone(frames, K=1, omega=OMEGA, snr=1.0):
    import torch
    om = torch.full((frames, K, 1), float(omega), dtype=torch.float64, device="cuda")
    sb = torch.full((frames, K), math.sqrt(snr), dtype=torch.float64, device="cuda")
    return om, sb


def per_sigma_detection(des, frames=8192, seed=11):
    """Measured P(c_sigma[M_sigma(LOC)] = 1) for every odd sigma (32 sigmas per plan, one
    segment per sigma and frame).  Returns (sigmas, p_hat, frames)."""
    import torch
    from paper_1610_01050_b200 import rsft as B
    sig_all = np.arange(1, N, 2)
    p_hat = np.zeros(sig_all.size)
    om, sb = _tone(frames, snr=des["snr_min"])
    for c in range(0, sig_all.size, 32):
        sg = sig_all[c:c + 32]
        L = sg.size
        plan = B.Plan((N,), (BK,), L, gamma_override=des["gamma"], mu=1, max_batch=frames, **WIN)
        plan.set_schedule(sg[:, None], np.zeros((L, 1), np.int64))
        plan.bind()
        x = B.synthesize((N,), frames, L, om, sb, 1.0, seed * 1000 + c)
        bm = plan.execute_segments(x)                                   # [frames, L, 2]
        j = torch.from_numpy(bucket_of(sg)).cuda()
        w = bm.gather(2, (j // 32).view(1, L, 1).expand(frames, L, 1)).squeeze(2)
        bits = (w.to(torch.int64) >> (j % 32).view(1, L)) & 1
        p_hat[c:c + L] = bits.double().mean(0).cpu().numpy()
        del x, bm
    torch.cuda.synchronize()
    return sig_all, p_hat, frames


def approx_error(P, T, draws=100, seed=5, var_unbiased=None):
    """Fig. varAppErr: mean over `draws` sets of T permutations (uniform over the odd sigma,
    with replacement) of (T Pd_bar (1 - Pd_bar) - sigma_a1^2) / sigma_a1^2, Eq. var_a1."""
    rng = np.random.default_rng(seed)
    P = np.asarray(P, dtype=np.float64)
    pv = P * (1 - P) if var_unbiased is None else var_unbiased
    pbar = P.mean()
    errs = []
    for _ in range(draws):
        s = rng.integers(0, P.size, T)
        sa = pv[s].sum()
        errs.append((T * pbar * (1 - pbar) - sa) / sa)
    return float(np.mean(errs)), float(np.std(errs))


def fixed_schedule_votes(des, frames=8192, batches=8, T=T_PAPER, seed=21):
    """abar at the tone's location over frames for one seeded T-loop schedule (segment mode,
    rsft_detect counts).  Returns (sigmas [T], abar values [frames * batches])."""
    import torch
    from paper_1610_01050_b200 import rsft as B
    plan = B.Plan((N,), (BK,), T, gamma_override=des["gamma"], mu=1, seed=seed, max_batch=frames, **WIN)
    plan.bind()
    sig = plan.schedule()[0][:, 0]
    om, sb = _tone(frames, snr=des["snr_min"])
    counts = torch.empty((frames, N), dtype=torch.uint8, device="cuda")
    vals = []
    for k in range(batches):
        x = B.synthesize((N,), frames, T, om, sb, 1.0, seed * 7919 + k)
        bm = plan.execute_segments(x)
        plan.detect(bm, counts=counts)
        vals.append(counts[:, LOC].to(torch.int32).cpu().numpy())
        del x, bm
    return sig, np.concatenate(vals)


def detector_at_design(des, frames=4096, batches=2, T=T_PAPER, K=4, seed=77):
    """Two-stage detector with (gamma*, mu*): K resolvable mid-bin tones per frame at SNR_min*
    (eta_p = 1), Swerling per segment.  Returns (P_d measured, false detections, trials)."""
    import torch
    from paper_1610_01050_b200 import rsft as B
    plan = B.Plan((N,), (BK,), T, gamma_override=des["gamma"], mu=des["mu"], seed=seed, max_batch=frames, **WIN)
    plan.bind()
    rng = np.random.default_rng(seed)
    hits = tot = fa = trials = 0
    for k in range(batches):
        ks = np.zeros((frames, K), dtype=np.int64)
        for f in range(frames):                      # resolvable tones (>= 16 bins apart)
            ks[f] = np.sort(rng.choice(np.arange(0, N, 16), K, replace=False) + rng.integers(0, 8, K))
        om = torch.from_numpy((ks + 0.5).astype(np.float64)[:, :, None]).cuda()
        sb = torch.full((frames, K), math.sqrt(des["snr_min"]), dtype=torch.float64, device="cuda")
        x = B.synthesize((N,), frames, T, om, sb, 1.0, seed * 31 + k)
        det = plan.detect(plan.execute_segments(x)).cpu().numpy()
        d = np.unpackbits(det.view(np.uint8), bitorder="little").reshape(frames, -1)[:, :N].astype(bool)
        hits += int(d[np.arange(frames)[:, None], ks].sum())
        tot += ks.size
        mask = np.ones_like(d)
        for j in range(-3, 5):                       # the tones' main lobes are not false alarms
            mask[np.arange(frames)[:, None], (ks + j) % N] = False
        fa += int(d[mask].sum())
        trials += int(mask.sum())
        del x
    return hits / tot, fa, trials


def main():
    import torch
    from scipy.stats import binom
    torch.cuda.init()
    out = {"setting": {"N": N, "B": BK, "T": T_PAPER, "omega_m_bins": OMEGA, "window": "Dolph-Chebyshev 40 dB",
                       "P_d": 0.9, "P_fa": 1e-6, "K": 4}}
    t0 = time.time()
    des = design()
    out["design"] = {k: float(v) for k, v in des.items()}
    sig, a, b = oracle_alpha_beta()
    law = tpd(a, b, des["gamma"], des["snr_min"])
    sig_g, p_hat, F = per_sigma_detection(des, frames=16384)
    z = (p_hat - law) / np.sqrt(law * (1 - law) / F)
    out["per_sigma"] = {"frames_per_sigma": F, "sigmas": int(sig.size), "max_abs_z": float(np.max(np.abs(z))),
                        "mean_measured": float(p_hat.mean()), "mean_law": float(law.mean()),
                        "min_law": float(law.min()), "max_law": float(law.max())}
    pv_hat = p_hat * (1 - p_hat) * F / (F - 1)                        # unbiased P(1-P)
    rows = []
    for T in (10, 50, 100, 200):
        e_law, s_law = approx_error(law, T)
        e_gpu, s_gpu = approx_error(p_hat, T, var_unbiased=pv_hat)
        rows.append({"T": T, "err_law": e_law, "err_law_std": s_law, "err_gpu": e_gpu, "err_gpu_std": s_gpu})
    out["approx_error"] = rows
    sg, ab = fixed_schedule_votes(des, frames=8192, batches=8)
    idx = (sg - 1) // 2
    pl = law[idx]
    out["fixed_schedule"] = {"frames": int(ab.size), "abar_mean": float(ab.mean()), "sum_P": float(pl.sum()),
                             "abar_var": float(ab.var(ddof=1)), "sum_P1mP": float((pl * (1 - pl)).sum()),
                             "bound_T_Pbar_1mPbar": float(T_PAPER * law.mean() * (1 - law.mean()))}
    pd_m, fa, trials = detector_at_design(des, frames=4096, batches=4)
    q = des["F"] / T_PAPER
    out["detector"] = {"P_d_measured": pd_m, "false_detections": fa, "trials": trials,
                       "P_fa_measured": fa / trials,
                       "P_d_exact_binomial": float(binom.sf(des["mu"] - 1, T_PAPER, des["pd_bar"])),
                       "P_fa_exact_binomial": float(binom.sf(des["mu"] - 1, T_PAPER,
                                                             q * des["pd_bar"] + (1 - q) * des["pfa_bar"]))}
    out["wall_s"] = time.time() - t0
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r02_next2.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
