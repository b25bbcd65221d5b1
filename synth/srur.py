"""SRUR scene generator and scoring (paper §VI).

Short-range ubiquitous radar (Table III): LFMCW bursts of M repetition intervals
(RIs) received on an N-element half-wavelength ULA and de-chirped (Eq. trsig, Eq. r_i
P:788-793): each target k contributes a sinusoid whose fast-time frequency encodes range,
f_r = 2 rho r / c (Eq. s_u), whose element-to-element phase step is pi sin(theta), and
whose RI-to-RI phase step is 2 pi f_d T_p with f_d = 2 v / lambda (Eq. s_u).  Complex
baseband cube per burst s: x[r][i][v] (R fast-time samples x N elements x M RIs), amplitude
a_k(s) ~ CN(0, sigma_k^2) static within a burst and independent between bursts
(Swerling I), plus CN(0, 1) noise.  Reading L24: the complex (IQ) form of Eq. r_i with
the slow-time Doppler phase that the 3-D FFT of Fig. MIMO_Bart resolves;
the paper omits constant phases only.

Input generation and geometry only: none of the RSFT arithmetic lives here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# Table III
R_BINS, N_ELEM, M_RI = 2048, 64, 32
LAMBDA, C_LIGHT, T_P, RHO, F_S = 0.03, 3e8, 5e-5, 3e12, 41e6


@dataclass
class Target:
    range_m: float
    velocity_mps: float
    doa_deg: float
    snr_db: float


# Table IV: range, velocity, DOA, SNR for the two settings
TABLE_IV = [(1000.0, 100.0, 30.0, (-10.0, 0.0)), (500.0, 50.0, 0.0, (-10.0, -10.0)),
            (350.0, 240.0, -16.0, (-10.0, -20.0)), (350.0, 240.0, -20.0, (-10.0, -20.0))]


def table_iv(setting: int):
    """The four targets of Table IV; setting 0: equal SNR (-10 dB), 1: mixed SNR."""
    return [Target(r, v, a, s[setting]) for r, v, a, s in TABLE_IV]


def target_bins(t: Target, shape=(R_BINS, N_ELEM, M_RI)):
    """Continuous DFT-bin position (range, angle, Doppler) of a target (Eq. s_u):
    range: f_r / f_s * R; angle: N sin(theta) / 2 (half-wavelength spacing); Doppler:
    f_d T_p M, all modulo the dimension."""
    R, N, M = shape
    f_r = 2.0 * RHO * t.range_m / C_LIGHT
    f_d = 2.0 * t.velocity_mps / LAMBDA
    kr = f_r / F_S * R
    ka = N * math.sin(math.radians(t.doa_deg)) / 2.0
    kd = f_d * T_P * M
    return (kr % R, ka % N, kd % M)


def scene(targets, bursts: int, seed: int, shape=(R_BINS, N_ELEM, M_RI), noise: bool = True) -> np.ndarray:
    """Complex64 bursts [bursts][R][N][M] of Eq. r_i in complex baseband (reading L24)."""
    R, N, M = shape
    rng = np.random.default_rng([seed, 5])
    r = np.arange(R)[:, None, None]
    i = np.arange(N)[None, :, None]
    v = np.arange(M)[None, None, :]
    out = np.empty((bursts, R, N, M), dtype=np.complex64)
    steer = []
    for t in targets:
        kr, ka, kd = target_bins(t, shape)
        steer.append(np.exp(2j * np.pi * (kr * r / R + ka * i / N + kd * v / M)))
    for s in range(bursts):
        x = np.zeros((R, N, M), dtype=np.complex128)
        if noise:
            x = x + math.sqrt(0.5) * (rng.standard_normal((R, N, M)) + 1j * rng.standard_normal((R, N, M)))
        for t, st in zip(targets, steer):
            sig = math.sqrt(10.0 ** (t.snr_db / 10.0))
            a = sig * math.sqrt(0.5) * (rng.standard_normal() + 1j * rng.standard_normal())
            x = x + a * st
        out[s] = x.astype(np.complex64)
    return out


def score(det_idx, targets, shape=(R_BINS, N_ELEM, M_RI), tol=1, lobe=(3, 3, 3)):
    """Scoring as SPEC S:530: a target counts as found when a detection lies within +-tol bins
    (cyclic, per dimension) of its nearest grid point.  Detections farther than `lobe` bins
    from every target split into single-dimension aliases (within +-tol of a target in all
    dimensions but one: cells that share a strong target's bucket whenever one short
    dimension's permutation collides, reading L25) and false detections (the rest).
    Returns (found [K] bool, n_false, n_alias)."""
    R, N, M = shape
    idx = np.asarray(det_idx, dtype=np.int64)
    pos = np.stack([idx // (N * M), (idx // M) % N, idx % M], axis=1) if idx.size else np.zeros((0, 3), np.int64)
    dims = np.array(shape)
    found = []
    near_any = np.zeros(len(pos), dtype=bool)
    alias = np.zeros(len(pos), dtype=bool)
    for t in targets:
        g = np.array([round(b) % d for b, d in zip(target_bins(t, shape), shape)])
        dd = np.abs(pos - g[None, :])
        dd = np.minimum(dd, dims[None, :] - dd)
        found.append(bool(np.any(np.all(dd <= tol, axis=1))))
        near_any |= np.all(dd <= np.array(lobe)[None, :], axis=1)
        alias |= (dd <= tol).sum(axis=1) >= len(shape) - 1
    alias &= ~near_any
    return np.array(found), int((~near_any & ~alias).sum()), int(alias.sum())
