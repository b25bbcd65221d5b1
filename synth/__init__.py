"""Seeded synthetic radar-shaped inputs for the RSFT hot path.

This module holds NONE of the RSFT method's arithmetic (no windows, permutations, folds,
FFTs, thresholds or votes).  It only draws the input frames of the paper's signal model,
Eq. sig_model / sinusoid, extended separably to N-D (Sec. III-C):

    x[n] = sum_k a_k prod_d exp(j 2 pi f_{k,d} n_d) + nu[n],   nu ~ CN(0, sigma_n^2) iid,

with off-grid frequencies f_{k,d} ~ U[0,1) (cycles/sample, "frequencies are continuous")
and a_k = sigma_n 10^{SNR_k/20} e^{j phi_k} (per-sample SNR), phi_k ~ U[0, 2 pi).
BASELINE c1 instead fixes |a_k| = 1 with sigma_n^2 = 0.1 (10 dB).

It is the one module shared by the oracle side (tests) and the product side (bench, smoke):
both consume the same complex64 bits.  The paper measures on no public dataset; these
seeded frames stand in for its simulations.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    n: tuple            # frame shape N_0 x ... (row-major, last dim contiguous)
    b: tuple            # buckets per dim B_d
    loops: int          # L permutation loops (paper T)
    p_fa: float         # first-stage per-bucket false-alarm probability (DESIGN L8)
    noise_var: float    # sigma_n^2
    k_range: tuple      # (K_min, K_max) targets per frame, uniform integer
    snr_db: tuple       # (lo, hi) per-target SNR in dB, uniform; None -> unit amplitude
    batch: int = 1      # frames per call
    support: tuple = () # flat-window support W_d (0 -> N_d)
    random_tau: bool = False
    data_seed: int = 0
    sched_seed: int = 0
    mu: int = 0         # 0 -> L (DESIGN L9)

    @property
    def ntot(self):
        return int(np.prod(self.n))

    def with_(self, **kw):
        return replace(self, **kw)


# BASELINE.json configs[0..4].  Seeds: data 100+c, schedule 200+c.
C1 = Workload("c1_1d", (4096,), (64,), 8, 1e-4, 0.1, (4, 4), None, 1, (512,), True, 101, 201)
C2 = Workload("c2_2d", (256, 256), (16, 16), 6, 1e-5, 1.0, (10, 10), (0.0, 20.0), 1, (), False, 102, 202)
C3 = Workload("c3_3d", (512, 128, 32), (32, 16, 8), 8, 1e-6, 1.0, (20, 20), (5.0, 25.0), 1, (), False, 103, 203)
C4 = Workload("c4_batched_2d", (1024, 256), (32, 16), 6, 1e-6, 1.0, (5, 30), (0.0, 20.0), 4096, (), False, 104, 204)
C5 = Workload("c5_cube", (2048, 512, 64), (64, 32, 8), 16, 1e-7, 1.0, (64, 64), (0.0, 20.0), 1, (), False, 105, 205)
WORKLOADS = {w.name: w for w in (C1, C2, C3, C4, C5)}


@dataclass
class Truth:
    freqs: np.ndarray   # [K, D] cycles/sample in [0, 1)
    amps: np.ndarray    # [K] complex


def draw_truth(wl: Workload, frame: int) -> Truth:
    rng = np.random.default_rng([wl.data_seed, frame, 1])
    k = int(rng.integers(wl.k_range[0], wl.k_range[1] + 1))
    freqs = rng.random((k, len(wl.n)))
    phase = np.exp(2j * np.pi * rng.random(k))
    if wl.snr_db is None:
        amps = phase
    else:
        snr = rng.uniform(wl.snr_db[0], wl.snr_db[1], k)
        amps = np.sqrt(wl.noise_var) * 10.0 ** (snr / 20.0) * phase
    return Truth(freqs, amps)


def tones(shape, truth: Truth) -> np.ndarray:
    """sum_k a_k prod_d e^{j 2 pi f_{k,d} n_d} as complex128 (separable outer products)."""
    k = truth.amps.shape[0]
    if k == 0:
        return np.zeros(shape, dtype=np.complex128)
    e = [np.exp(2j * np.pi * np.outer(np.arange(n), truth.freqs[:, d])) for d, n in enumerate(shape)]
    if len(shape) == 1:
        return e[0] @ truth.amps
    left = e[0] * truth.amps[None, :]                  # [N0, K]
    right = e[1]                                       # [N1, K]
    for d in range(2, len(shape)):                     # Khatri-Rao of the trailing dims
        right = (right[:, None, :] * e[d][None, :, :]).reshape(-1, k)
    return (left @ right.T).reshape(shape)


def gen_frame(wl: Workload, frame: int, noise: bool = True) -> np.ndarray:
    """Frame #frame of workload wl as complex64 (deterministic in (data_seed, frame))."""
    x = tones(wl.n, draw_truth(wl, frame))
    if noise and wl.noise_var > 0:
        rng = np.random.default_rng([wl.data_seed, frame, 2])
        s = np.sqrt(wl.noise_var / 2.0)
        nr = rng.standard_normal(x.shape)
        ni = rng.standard_normal(x.shape)
        x = x + s * (nr + 1j * ni)
    return x.astype(np.complex64)


def gen_batch(wl: Workload, frames, noise: bool = True) -> np.ndarray:
    frames = list(frames)
    out = np.empty((len(frames),) + tuple(wl.n), dtype=np.complex64)
    for i, f in enumerate(frames):
        out[i] = gen_frame(wl, f, noise)
    return out


def gen_noise_only(shape, noise_var: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng([seed, 7])
    s = np.sqrt(noise_var / 2.0)
    return (s * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))).astype(np.complex64)


def gen_ongrid(shape, bins, amps) -> np.ndarray:
    """Noiseless on-grid tones at integer bins (rows of `bins`), complex128."""
    bins = np.asarray(bins, dtype=np.float64).reshape(len(amps), len(shape))
    tr = Truth(bins / np.asarray(shape, dtype=np.float64)[None, :], np.asarray(amps, dtype=np.complex128))
    return tones(tuple(shape), tr)


# ----------------------------------------------------------------------------- counter RNG
# NumPy mirror of the library's Monte Carlo scene generator (rsft_synthesize): SplitMix64 of
# (seed, stream, counter) -> two 32-bit uniforms -> Box-Muller, E|z|^2 = 1.  Pure input
# generation (no arithmetic of the method).
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64_np(z):
    with np.errstate(over="ignore"):
        z = (z + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def counter_normals(seed: int, stream: int, ctr) -> np.ndarray:
    """CN(0, 1) samples (complex128) for counters ctr (array of non-negative ints)."""
    ctr = np.asarray(ctr, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = np.uint64(seed) ^ ((np.uint64(stream) * np.uint64(0xD1B54A32D192ED03)) & _M64)
    r = _splitmix64_np(key ^ _splitmix64_np(ctr))
    u1 = ((r >> np.uint64(32)).astype(np.float64) + 1.0) / 4294967296.0
    u2 = (r & np.uint64(0xFFFFFFFF)).astype(np.float64) / 4294967296.0
    rad = np.sqrt(-np.log(u1))
    return rad * np.exp(2j * np.pi * u2)


def synth_segments(n, batch: int, segments: int, omega: np.ndarray, sigma_b: np.ndarray, sigma_n: float,
                   seed: int) -> np.ndarray:
    """NumPy reference of rsft_synthesize: [batch][segments][*n] complex128."""
    n = tuple(int(v) for v in n)
    D = len(n)
    K = omega.shape[1] if omega.size else 0
    ntot = int(np.prod(n))
    grids = np.meshgrid(*[np.arange(v) for v in n], indexing="ij")
    out = np.zeros((batch, segments) + n, dtype=np.complex128)
    for f in range(batch):
        for s in range(segments):
            x = np.zeros(n, dtype=np.complex128)
            for k in range(K):
                b = counter_normals(seed, 1, [(f * K + k) * segments + s])[0] * sigma_b[f, k]
                ph = np.zeros(n)
                for d in range(D):
                    ph = ph + 2.0 * np.fmod(omega[f, k, d] * grids[d], n[d]) / n[d]
                x = x + b * np.exp(1j * np.pi * ph)
            ctr = (f * segments + s) * ntot + np.arange(ntot)
            x = x + sigma_n * counter_normals(seed, 2, ctr).reshape(n)
            out[f, s] = x
    return out
