"""RSFT oracle: a plain, slow, obviously-correct fp64 CPU implementation of Algorithm 1
of Wang, Patel, Petropulu, "An Efficient High-Dimensional Sparse Fourier Transform"
(arXiv 1610.01050, the "Realistic Sparse Fourier Transform", RSFT).

*** TEST INFRASTRUCTURE ONLY. ***
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path
(``paper_1610_01050_b200``, ``include/rsft.h``, the CUDA kernels) never imports, links
or calls anything here, and this module imports nothing from the product path.  The two
share no code, tables or constants; the only shared module is ``synth`` (seeded input
generation, which holds none of the method's arithmetic).

Citation convention: ``P:<line>`` is a line of ``/root/reference/PAPER.md`` (the paper's
LaTeX source) with the section / equation / algorithm it falls in.  ``L<n>`` is a reading
listed in DESIGN.md ("Readings of the paper"), used where the paper is silent or garbled.

Everything is computed in float64 / complex128 on the exact complex64 input bits.  Steps
follow Algorithm 1 in order: pre-permutation window -> permutation ->
flat window -> aliasing -> N-D FFT -> first-stage NP test -> reverse mapping ->
accumulation -> second-stage test.  Library primitives used as single steps:
``numpy.fft.fftn`` (the N-D DFT) and numpy fancy indexing / reshape-sum.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): SPEC/paper worked examples, Props. 1-4
(exhaustive), dense brute-force D*V_sigma*r matrices (Eqs. l, f), the
brick-wall identity against a direct O(N^2) DFT, closed-form noise variance beta (Eq.
var_fu), the Eq. tpd false-alarm law on pure noise, scipy's chebwin, Hann's
closed-form spectrum, Parseval, on-grid noiseless exact recovery.
Parity unpinned (a chosen design, pinned only by its own response properties): the exact
flat-window prototype shape (L2), the default mu (L9), absolute gamma vs. the paper (L15).
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

MASK64 = (1 << 64) - 1
AMBIGUITY_REL = 1e-3      # first-stage near-threshold band (BASELINE north_star; L16)
BUCKET_REL_TOL = 1e-4     # bucket value tolerance fp32 vs fp64 (BASELINE north_star)


# ----------------------------------------------------------------------------------
# Parameters (mirrors the C ABI rsft_params; SPEC RsftConfig S:255-260)
# ----------------------------------------------------------------------------------
@dataclass
class Params:
    n: tuple                      # N_d, powers of two
    b: tuple                      # B_d, powers of two, B_d | N_d (Def. 2)
    loops: int                    # L (the paper's T, Alg. 1)
    support: tuple = ()           # flat-window support W_d (0 -> N_d)
    prewin: str = "hann"          # "hann" | "rect" | "cheb"
    prewin_param: float = 60.0    # Chebyshev attenuation in dB when prewin == "cheb"
    flat_atten_db: float = 60.0   # Dolph-Chebyshev taper of the flat window
    p_fa: float = 1e-6            # first-stage per-bucket false-alarm prob. (L8)
    noise_var: float = 1.0        # sigma_n^2
    gamma_override: float = 0.0   # > 0: one gamma for all loops (SPEC RsftConfig.gamma)
    mu: int = 0                   # second-stage vote threshold; 0 -> L (L9)
    seed: int = 0                 # sigma/tau schedule seed (L5)
    random_tau: bool = False      # tau = 0 unless set

    def __post_init__(self):
        self.n = tuple(int(v) for v in self.n)
        self.b = tuple(int(v) for v in self.b)
        if not self.support:
            self.support = tuple(0 for _ in self.n)
        self.support = tuple(int(v) for v in self.support)
        if self.mu == 0:
            self.mu = self.loops

    @property
    def ndim(self):
        return len(self.n)

    @property
    def a(self):  # fold factors N_d / B_d (the paper's L = N/B)
        return tuple(n // b for n, b in zip(self.n, self.b))


def validate(p: Params):
    """Argument rules (S:172 AliasShape, S:259 RsftConfig, S:180 NonInvertible)."""
    if not (1 <= p.ndim <= 3):
        raise ValueError("ndim must be 1..3")
    for n, b, w in zip(p.n, p.b, p.support):
        if n < 1 or n & (n - 1) or b < 1 or b & (b - 1) or b > n:
            raise ValueError("N_d, B_d must be powers of two with B_d <= N_d (P:57, P:88)")
        if b < n:
            w = n if w == 0 else w
            if w > n or w % 2 or (w // 2) % b:
                raise ValueError("flat-window support W_d must satisfy 2B_d | W_d <= N_d (L2)")
    if p.loops < 1 or not (1 <= p.mu <= p.loops):
        raise ValueError("need L >= 1 and 1 <= mu <= L (S:259)")
    if not (0.0 < p.p_fa < 1.0):
        raise ValueError("0 < P_fa < 1")


# ----------------------------------------------------------------------------------
# Modular machinery: Defs. 1-4
# ----------------------------------------------------------------------------------
def splitmix64(seed: int, ctr: int) -> int:
    """Counter-based SplitMix64 draw #ctr of stream ``seed`` (reading L5; the paper only
    says "Generate a set of sigma randomly for each dimension", Alg. 1 l.2)."""
    z = (seed + (ctr + 1) * 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def mod_inverse(sigma: int, n: int) -> int:
    """sigma^{-1} with sigma*sigma^{-1} = [1]_N, Eq. mod_inv."""
    if math.gcd(sigma, n) != 1:
        raise ValueError("sigma not invertible mod N (S:180 NonInvertible)")
    return pow(sigma, -1, n) if n > 1 else 0


def schedule(p: Params):
    """sigma, sigma^{-1}, tau as [L][D] int arrays.  sigma uniform over odd [N_d]
    ("a valid sigma can be any odd integer"); reading L5 fixes the generator:
    sigma = 2*(SplitMix64(seed, 2(lD+d)) & (N_d/2-1)) + 1,
    tau   = SplitMix64(seed, 2(lD+d)+1) & (N_d-1) if random_tau else 0."""
    D, L = p.ndim, p.loops
    sig = np.zeros((L, D), dtype=np.int64)
    sinv = np.zeros((L, D), dtype=np.int64)
    tau = np.zeros((L, D), dtype=np.int64)
    for l in range(L):
        for d in range(D):
            n = p.n[d]
            ctr = 2 * (l * D + d)
            s = 2 * (splitmix64(p.seed, ctr) & (n // 2 - 1)) + 1 if n >= 2 else 1
            t = (splitmix64(p.seed, ctr + 1) & (n - 1)) if (p.random_tau and n > 1) else 0
            sig[l, d] = s
            sinv[l, d] = mod_inverse(s, n)
            tau[l, d] = t
    return sig, sinv, tau


def permute(y: np.ndarray, sigma: int, tau: int) -> np.ndarray:
    """Def. 1, Eq. permutation: (P_{sigma,tau} y)_i = y_{sigma i + tau}."""
    n = y.shape[0]
    return y[(sigma * np.arange(n) + tau) % n]


def permute_nd(y: np.ndarray, sigmas: Sequence[int], taus: Sequence[int]) -> np.ndarray:
    """Per-dimension permutation carried out on each dimension sequentially."""
    out = y
    for d, (s, t) in enumerate(zip(sigmas, taus)):
        n = y.shape[d]
        idx = (int(s) * np.arange(n) + int(t)) % n
        out = np.take(out, idx, axis=d)
    return out


def fold(z: np.ndarray, b: int) -> np.ndarray:
    """Def. 2, Eq. aliasing: y_i = sum_{j in [N/B]} z_{i+Bj}, i in [B]."""
    n = z.shape[0]
    return z.reshape(n // b, b).sum(axis=0)


def fold_nd(z: np.ndarray, bs: Sequence[int]) -> np.ndarray:
    """N-D aliasing: periodic extension with basic period B_0 x ...."""
    shape = []
    for n, b in zip(z.shape, bs):
        shape += [n // b, b]
    axes = tuple(range(0, 2 * len(bs), 2))
    return z.reshape(shape).sum(axis=axes)


def map_index(i: int, sigma: int, n: int, b: int) -> int:
    """Def. 3: M(i, sigma) = floor(B/N * [i sigma]_N)."""
    return ((i * sigma) % n) * b // n


def reverse_map(j: int, sigma_inv: int, n: int, b: int) -> list:
    """Def. 4: R(j, sigma^{-1}) = {[sigma^{-1} u]_N : jN/B <= u < (j+1)N/B}."""
    a = n // b
    return [(sigma_inv * u) % n for u in range(j * a, (j + 1) * a)]


# ----------------------------------------------------------------------------------
# Windows
# ----------------------------------------------------------------------------------
def hann_periodic(n: int) -> np.ndarray:
    """Periodic Hann w[n] = sin^2(pi n / N) (BASELINE c1/c2 "Hann"; reading L3)."""
    return np.sin(np.pi * np.arange(n) / n) ** 2


def dolph_chebyshev(m: int, atten_db: float) -> np.ndarray:
    """Symmetric Dolph-Chebyshev taper of odd length M, peak 1.
    Chebyshev-polynomial frequency definition + inverse DFT:
      r = 10^(A/20), x0 = cosh(arccosh(r)/(M-1)),
      What[k] = T_{M-1}(x0 cos(pi k / M)),  k in [M],
      taper[m] = Re(IDFT_M(What))[(m - (M-1)/2) mod M] / max   (centre at m=(M-1)/2).
    (Reading L19: SURVEY's index "(m + (M-1)/2)" is off by one; the centred form is used.)"""
    if m < 1 or m % 2 == 0:
        raise ValueError("odd M required")
    if m == 1:
        return np.ones(1)
    order = m - 1
    r = 10.0 ** (atten_db / 20.0)
    x0 = np.cosh(np.arccosh(r) / order)
    x = x0 * np.cos(np.pi * np.arange(m) / m)
    ax = np.abs(x)
    inside = ax <= 1.0
    t = np.empty(m)
    t[inside] = np.cos(order * np.arccos(x[inside]))
    t[~inside] = np.cosh(order * np.arccosh(ax[~inside])) * np.sign(x[~inside]) ** order
    w = np.real(np.fft.ifft(t))
    k = (np.arange(m) - (m - 1) // 2) % m
    taper = w[k]
    return taper / taper.max()


def cheb_periodic(n: int, atten_db: float) -> np.ndarray:
    """Periodic Chebyshev pre-window: N+1-point symmetric taper, last point dropped."""
    return dolph_chebyshev(n + 1, atten_db)[:n]


def prewindow(p: Params, d: int) -> np.ndarray:
    """Pre-permutation window w_d (Alg. 1 l.5)."""
    n = p.n[d]
    if p.prewin == "hann":
        return hann_periodic(n)
    if p.prewin == "rect":
        return np.ones(n)
    if p.prewin == "cheb":
        return cheb_periodic(n, p.prewin_param)
    raise ValueError(p.prewin)


def flat_prototype(n: int, b: int, w: int, atten_db: float) -> np.ndarray:
    """Real, even, cyclic flat-window prototype g (reading L2; "main-lobe width
    2 pi / B, length N"; "based on this [Dolph-Chebyshev] window, passband 1/B"):
        g[t] = sinc(t_c / B) * T_{W+1}(t_c)   for |t_c| <= W/2, else 0,
    t_c the centred representative of t in [-N/2, N/2); T the symmetric Dolph-Chebyshev
    taper of length W+1 centred at t_c = 0.  B == N: no flat window (g = 1)."""
    if b == n:
        return np.ones(n)
    w = n if w == 0 else w
    t = np.arange(n)
    tc = np.where(t < n // 2, t, t - n)
    taper = dolph_chebyshev(w + 1, atten_db)
    g = np.zeros(n)
    sel = np.abs(tc) <= w // 2
    g[sel] = np.sinc(tc[sel] / b) * taper[tc[sel] + w // 2]
    return g


def flat_window(n: int, b: int, w: int, atten_db: float) -> np.ndarray:
    """Complex flat window gbar[t] = g[t] e^{-j pi t / B} (reading L1: the half-bucket
    shift realises Def. 3's floor mapping, P:104 / Claim 1 P:325).  B == N: gbar = 1."""
    if b == n:
        return np.ones(n, dtype=np.complex128)
    g = flat_prototype(n, b, w, atten_db)
    return g * np.exp(-1j * np.pi * np.arange(n) / b)


def brickwall_window(n: int, b: int) -> np.ndarray:
    """Ideal complex brick-wall flat window gbar[t] = sum_{q in [N/B]} e^{-j 2 pi q t / N}
    (used only by pins: with it f^_k = sum_{i: M(i,sigma)=k} y^_i e^{+j2pi tau i/N}, I4)."""
    a = n // b
    t = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(np.arange(a), t) / n).sum(axis=0)


def outer_nd(vecs: Sequence[np.ndarray]) -> np.ndarray:
    """Compound N-D window W_xy = w_x w_y^H generalised; real windows, so the
    conjugate is immaterial for w; for the complex flat window the product is used as is."""
    out = np.asarray(vecs[0])
    for v in vecs[1:]:
        out = np.multiply.outer(out, np.asarray(v))
    return out


# ----------------------------------------------------------------------------------
# The RSFT first stage (Alg. 1 lines 5-10; Eqs. z, l, f, alpha_beta, tpd; P:220-225,
# P:267-316) and the second stage (Alg. 1 lines 11-14; Eq. a_i).
# ----------------------------------------------------------------------------------
@dataclass
class Tables:
    prewin: list            # w_d, float64 [N_d]
    flat: list              # gbar_d, complex128 [N_d]
    sigma: np.ndarray       # [L][D]
    sigma_inv: np.ndarray
    tau: np.ndarray


def make_tables(p: Params, flat_override=None, schedule_override=None) -> Tables:
    validate(p)
    w = [prewindow(p, d) for d in range(p.ndim)]
    if flat_override is not None:
        gb = list(flat_override)
    else:
        gb = [flat_window(p.n[d], p.b[d], p.support[d], p.flat_atten_db) for d in range(p.ndim)]
    if schedule_override is not None:
        sig, tau = (np.asarray(v, dtype=np.int64) for v in schedule_override)
        sinv = np.array([[mod_inverse(int(s), n) for s, n in zip(row, p.n)] for row in sig],
                        dtype=np.int64)
    else:
        sig, sinv, tau = schedule(p)
    return Tables(w, gb, sig, sinv, tau)


def beta(p: Params, tb: Tables, l: int) -> float:
    """beta(sigma) = ||Wbar P_sigma w||^2, Eq. alpha_beta.  The compound windows
    are outer products, so the squared norm of the N-D vector is the product
    of the per-dimension squared norms."""
    out = 1.0
    for d in range(p.ndim):
        pw = permute(tb.prewin[d], int(tb.sigma[l, d]), int(tb.tau[l, d]))
        out *= float(np.sum(np.abs(tb.flat[d] * pw) ** 2))
    return out


def gamma(p: Params, tb: Tables, l: int) -> float:
    """First-stage threshold.  Eq. tpd: P~_fa(sigma) = exp(-gamma/(sigma_n^2
    beta(sigma))); reading L8 sets P~_fa = P_fa exactly per loop:
    gamma_l = sigma_n^2 beta_l ln(1/P_fa).  gamma_override > 0 replaces it."""
    if p.gamma_override > 0:
        return float(p.gamma_override)
    return p.noise_var * beta(p, tb, l) * math.log(1.0 / p.p_fa)


@dataclass
class FirstStage:
    f: np.ndarray           # aliased buckets (complex128, shape B)
    fhat: np.ndarray        # B-point N-D FFT (complex128, shape B)
    beta: float
    gamma: float
    c: np.ndarray           # bool, shape B: |fhat|^2 > gamma
    ambiguous: np.ndarray   # bool: | |fhat|^2 - gamma | <= 1e-3 gamma (L16)


def first_stage(x: np.ndarray, p: Params, tb: Tables, l: int) -> FirstStage:
    """One iteration of Algorithm 1 on frame x (shape N_0 x ... row-major)."""
    x = np.asarray(x).astype(np.complex128)
    y = x * outer_nd(tb.prewin)                                   # l.5  y <- W r
    pz = permute_nd(y, tb.sigma[l], tb.tau[l])                    # l.6  p <- P_sigma y
    z = pz * outer_nd(tb.flat)                                    # l.7  z <- Wbar p
    f = fold_nd(z, p.b)                                           # l.8  Aliasing
    fhat = np.fft.fftn(f)                                         # l.9  N-D FFT
    be = beta(p, tb, l)
    ga = gamma(p, tb, l)
    pw = np.abs(fhat) ** 2                                        # "Square" (Table II)
    c = pw > ga                                                   # l.10 NPdet1
    amb = np.abs(pw - ga) <= AMBIGUITY_REL * ga
    return FirstStage(f, fhat, be, ga, c, amb)


def reverse_map_nd(k: Sequence[int], sinv: Sequence[int], p: Params) -> list:
    """N-D reverse map: Cartesian product of the per-dimension Def. 4 sets."""
    return [reverse_map(int(k[d]), int(sinv[d]), p.n[d], p.b[d]) for d in range(p.ndim)]


def accumulate(cs: Sequence[np.ndarray], p: Params, tb: Tables) -> np.ndarray:
    """Reverse-mapping + accumulation (Alg. 1 l.11-12; Eq. a_i):
    every set bucket k of loop l adds 1 at each location of R(k, sigma_l^{-1}) (Def. 4),
    literally, one set bucket at a time."""
    abar = np.zeros(p.n, dtype=np.int32)
    for l, c in enumerate(cs):
        for k in zip(*np.nonzero(c)):
            sets = reverse_map_nd(k, tb.sigma_inv[l], p)
            abar[np.ix_(*sets)] += 1
    return abar


def second_stage(abar: np.ndarray, mu: int):
    """Alg. 1 l.14: o = {i : abar_i >= mu} (reading L10: '>=' per P:530's integral
    from mu).  Returns (bool mask, sorted flat index list)."""
    o = abar >= mu
    return o, np.flatnonzero(o.ravel()).astype(np.int64)


def vote_lookup(cs: Sequence[np.ndarray], p: Params, tb: Tables) -> np.ndarray:
    """Hash-lookup form of the accumulation (identity I1 from Props. 3-4):
    abar[i] = sum_l c_l[M_l(i)], M_l(i)_d = Def. 3 per dimension.  Used only as a pin."""
    abar = np.zeros(p.n, dtype=np.int32)
    for l, c in enumerate(cs):
        idx = []
        for d in range(p.ndim):
            i = np.arange(p.n[d])
            idx.append(((i * int(tb.sigma[l, d])) % p.n[d]) * p.b[d] // p.n[d])
        abar += c[np.ix_(*idx)].astype(np.int32)
    return abar


@dataclass
class RsftResult:
    stages: list            # FirstStage per loop
    abar: np.ndarray        # vote counts (exact oracle bits)
    abar_min: np.ndarray    # ambiguous votes counted as 0
    abar_max: np.ndarray    # ambiguous votes counted as 1
    detect: np.ndarray      # bool mask abar >= mu
    idx: np.ndarray         # sorted flat indices


def rsft_run(x: np.ndarray, p: Params, tb: Tables | None = None, loops=None) -> RsftResult:
    """Algorithm 1 end to end on one frame."""
    tb = make_tables(p) if tb is None else tb
    loops = range(p.loops) if loops is None else loops
    st = [first_stage(x, p, tb, l) for l in loops]
    abar = accumulate([s.c for s in st], p, tb)
    amin = accumulate([s.c & ~s.ambiguous for s in st], p, tb)
    amax = accumulate([s.c | s.ambiguous for s in st], p, tb)
    det, idx = second_stage(abar, p.mu)
    return RsftResult(st, abar, amin, amax, det, idx)


def rsft_run_segments(xs: np.ndarray, p: Params, tb: Tables | None = None) -> RsftResult:
    """Algorithm 1 with "iterations on different segments": loop l runs the first stage
    on segment r_l (Eq. sig_model: fresh amplitudes and noise per segment), the
    reverse-mapped votes accumulate over the loops as in Eq. a_i and the second stage
    is unchanged.  xs: [L][N_0]...[N_{D-1}]."""
    tb = make_tables(p) if tb is None else tb
    st = [first_stage(xs[l], p, tb, l) for l in range(p.loops)]
    abar = accumulate([s.c for s in st], p, tb)
    amin = accumulate([s.c & ~s.ambiguous for s in st], p, tb)
    amax = accumulate([s.c | s.ambiguous for s in st], p, tb)
    det, idx = second_stage(abar, p.mu)
    return RsftResult(st, abar, amin, amax, det, idx)


# ----------------------------------------------------------------------------------
# Brute-force references (pins only; tiny sizes)
# ----------------------------------------------------------------------------------
def dft_direct(x: np.ndarray) -> np.ndarray:
    """N-D DFT by explicit sums over all n for every k (O(N^2)), forward, unnormalised."""
    x = np.asarray(x, dtype=np.complex128)
    shape = x.shape
    out = np.zeros(shape, dtype=np.complex128)
    for k in itertools.product(*[range(s) for s in shape]):
        acc = 0j
        for nidx in itertools.product(*[range(s) for s in shape]):
            ph = sum(k[d] * nidx[d] / shape[d] for d in range(len(shape)))
            acc += x[nidx] * np.exp(-2j * np.pi * ph)
        out[k] = acc
    return out


def first_stage_matrix(p: Params, tb: Tables, l: int) -> np.ndarray:
    """Dense B_tot x N_tot matrix D V_sigma of Eqs. l and f, built from explicit
    matrices on the row-major flattening: W = diag(w), P_sigma a 0/1 permutation matrix,
    Wbar = diag(gbar), the aliasing sum of row blocks Wbar_i (Eq. l), and the N-D DFT
    matrix D[k, b] = exp(-j 2 pi sum_d k_d b_d / B_d)."""
    ntot = int(np.prod(p.n))
    btot = int(np.prod(p.b))
    locs = list(itertools.product(*[range(n) for n in p.n]))
    flat_of = {loc: i for i, loc in enumerate(locs)}
    W = np.diag(outer_nd(tb.prewin).ravel().astype(np.complex128))
    Wb = np.diag(outer_nd(tb.flat).ravel())
    P = np.zeros((ntot, ntot))
    for t, loc in enumerate(locs):
        src = tuple((int(tb.sigma[l, d]) * loc[d] + int(tb.tau[l, d])) % p.n[d]
                    for d in range(p.ndim))
        P[t, flat_of[src]] = 1.0
    bl = list(itertools.product(*[range(b) for b in p.b]))
    bflat = {loc: i for i, loc in enumerate(bl)}
    Al = np.zeros((btot, ntot))
    for t, loc in enumerate(locs):
        Al[bflat[tuple(loc[d] % p.b[d] for d in range(p.ndim))], t] = 1.0
    V = Al @ Wb @ P @ W
    Dm = np.zeros((btot, btot), dtype=np.complex128)
    for i, k in enumerate(bl):
        for j, bb in enumerate(bl):
            Dm[i, j] = np.exp(-2j * np.pi * sum(k[d] * bb[d] / p.b[d] for d in range(p.ndim)))
    return Dm @ V


# ----------------------------------------------------------------------------------
# Comparison utility (the BASELINE tolerances made precise)
# ----------------------------------------------------------------------------------
def compare_buckets(fhat_gpu: np.ndarray, st: FirstStage, frame_power: float) -> dict:
    """|f_gpu - f_orc| <= 1e-4 max(|f_orc|, sqrt(beta P_x)) per bucket."""
    ref = st.fhat
    floor = math.sqrt(st.beta * frame_power)
    err = np.abs(np.asarray(fhat_gpu, dtype=np.complex128) - ref)
    scale = np.maximum(np.abs(ref), floor)
    ratio = err / scale
    return {"max_ratio": float(ratio.max()), "ok": bool(ratio.max() <= BUCKET_REL_TOL)}


def compare_bits(c_gpu: np.ndarray, st: FirstStage) -> dict:
    """First-stage bits must equal the oracle's outside the 1e-3 near-threshold band."""
    c_gpu = np.asarray(c_gpu, dtype=bool)
    bad = (c_gpu != st.c) & ~st.ambiguous
    return {"mismatch": int(bad.sum()), "ambiguous": int(st.ambiguous.sum()),
            "ok": not bad.any()}


def compare_sets(det_gpu: np.ndarray, res: RsftResult, mu: int) -> dict:
    """{count_min >= mu} subset o_gpu subset {count_max >= mu}."""
    det_gpu = np.asarray(det_gpu, dtype=bool)
    lo = res.abar_min >= mu
    hi = res.abar_max >= mu
    miss = lo & ~det_gpu
    extra = det_gpu & ~hi
    return {"missing": int(miss.sum()), "extra": int(extra.sum()),
            "ok": not (miss.any() or extra.any())}
