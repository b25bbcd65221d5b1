"""Thin ctypes binding of the C ABI in include/rsft.h (argument marshalling only).

Every step of the RSFT hot path runs in librsft.so's CUDA kernels; this module only converts
Python/PyTorch arguments to plain pointers and sizes.  PyTorch supplies device memory and
streams (plumbing).  There is no CPU fallback: if librsft.so is missing or a call fails,
an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int32, c_int64, c_size_t, c_uint8, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RSFT_LIB") or os.path.join(HERE, "librsft.so")   # RSFT_LIB: tuning variants

WIN = {"rect": 0, "hann": 1, "cheb": 2}
MODE = {"auto": 0, "fused": 1, "split": 2}
STATUS = {0: "RSFT_OK", 1: "RSFT_E_ARG", 2: "RSFT_E_SHAPE", 3: "RSFT_E_SIGMA", 4: "RSFT_E_UNSUPPORTED",
          5: "RSFT_E_WORKSPACE", 6: "RSFT_E_CUDA", 7: "RSFT_E_STATE"}


class RsftError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)} {what}".strip())


class RsftParams(ctypes.Structure):
    _fields_ = [("ndim", c_int32), ("n", c_int64 * 3), ("b", c_int64 * 3), ("support", c_int64 * 3),
                ("loops", c_int32), ("prewin", c_int32), ("prewin_param", c_double),
                ("flat_atten_db", c_double), ("p_fa", c_double), ("noise_var", c_double),
                ("gamma_override", c_double), ("mu", c_int32), ("random_tau", c_int32),
                ("seed", c_uint64), ("max_batch", c_int64), ("mode", c_int32)]


class RsftInfo(ctypes.Structure):
    _fields_ = [("ntot", c_int64), ("btot", c_int64), ("bitmap_words", c_int64),
                ("detect_words", c_int64), ("mode", c_int32), ("lpad", c_int32),
                ("workspace_bytes", c_size_t)]


_LIB = None


class RsftDesignParams(ctypes.Structure):
    _fields_ = [("K", c_int32), ("p_d", c_double), ("p_fa", c_double), ("eta_m", c_double), ("eta_p", c_double),
                ("omega", c_double * 3), ("loops", c_int32)]


class RsftDesignResult(ctypes.Structure):
    _fields_ = [("mu", c_int32), ("snr_min", c_double), ("snr_min_db", c_double), ("pd_bar", c_double),
                ("pfa_bar", c_double), ("gamma", c_double), ("alpha_bar", c_double), ("beta_bar", c_double),
                ("eta_m", c_double), ("F", c_double)]


def lib():
    """Load librsft.so (raises if it has not been built: no fallback path exists)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} not built; run `python -m paper_1610_01050_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    P = POINTER
    sig = {
        "rsft_default_params": (None, [P(RsftParams)]),
        "rsft_plan_create": (c_int32, [P(RsftParams), P(c_void_p)]),
        "rsft_plan_destroy": (None, [c_void_p]),
        "rsft_plan": (c_int32, [P(RsftParams), c_int32, P(c_void_p)]),
        "rsft_destroy": (None, [c_void_p]),
        "rsft_set_schedule": (c_int32, [c_void_p, P(c_int64), P(c_int64)]),
        "rsft_get_schedule": (c_int32, [c_void_p, P(c_int64), P(c_int64), P(c_int64)]),
        "rsft_get_thresholds": (c_int32, [c_void_p, P(c_double), P(c_double)]),
        "rsft_get_window": (c_int32, [c_void_p, c_int32, c_int32, P(c_double)]),
        "rsft_get_info": (c_int32, [c_void_p, P(RsftInfo)]),
        "rsft_workspace_bytes": (c_size_t, [c_void_p]),
        "rsft_bind": (c_int32, [c_void_p, c_void_p, c_size_t, c_void_p]),
        "rsft_execute": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
        "rsft_execute_segments": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
        "rsft_bucketize_partial": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
        "rsft_finalize": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
        "rsft_detect": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
        "rsft_compact": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p]),
        "rsft_detect_compact": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p,
                                          c_void_p]),
        "rsft_run": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                               c_void_p]),
        "rsft_host_scratch_bytes": (c_size_t, [c_void_p, c_int64, c_int64]),
        "rsft_run_host": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_int64, P(c_int64), c_void_p,
                                    c_size_t, c_void_p]),
        "rsft_last_launch_count": (c_int32, [c_void_p]),
        "rsft_default_design_params": (None, [P(RsftDesignParams)]),
        "rsft_bartlett": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_double, c_void_p,
                                    c_void_p]),
        "rsft_bartlett_threshold": (c_int32, [c_void_p, c_int32, c_double, P(c_double)]),
        "rsft_synthesize": (c_int32, [P(c_int64), c_int32, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_double,
                                      c_uint64, c_void_p, c_void_p]),
        "rsft_design_thresholds": (c_int32, [c_void_p, P(RsftDesignParams), P(RsftDesignResult)]),
        "rsft_status_string": (ctypes.c_char_p, [c_int32]),
        "rsft_last_error": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


EXPORTED = ["rsft_default_params", "rsft_plan_create", "rsft_plan_destroy", "rsft_plan", "rsft_destroy",
            "rsft_set_schedule",
            "rsft_get_schedule", "rsft_get_thresholds", "rsft_get_window", "rsft_get_info",
            "rsft_workspace_bytes", "rsft_bind", "rsft_execute", "rsft_execute_segments", "rsft_bucketize_partial",
            "rsft_finalize",
            "rsft_detect", "rsft_compact",
            "rsft_detect_compact", "rsft_run",
            "rsft_host_scratch_bytes", "rsft_run_host", "rsft_last_launch_count", "rsft_status_string",
            "rsft_default_design_params", "rsft_design_thresholds", "rsft_synthesize",
            "rsft_bartlett", "rsft_bartlett_threshold",
            "rsft_last_error"]


def _check(st):
    if st != 0:
        raise RsftError(st, lib().rsft_last_error().decode())


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(POINTER(c_int64))


def _stream_handle(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return c_void_p(stream.cuda_stream)


class Plan:
    """An RSFT plan (rsft_plan_create) plus, after bind(), its device workspace."""

    def __init__(self, n, b, loops, support=(), prewin="hann", prewin_param=60.0, flat_atten_db=60.0,
                 p_fa=1e-6, noise_var=1.0, gamma_override=0.0, mu=0, seed=0, random_tau=False,
                 max_batch=1, mode="auto"):
        L = lib()
        if not 1 <= len(n) <= 3 or len(b) != len(n):
            raise RsftError(4 if len(n) > 3 else 1, "ndim must be 1..3 with len(b) == len(n)")
        p = RsftParams()
        L.rsft_default_params(ctypes.byref(p))
        p.ndim = len(n)
        for d in range(len(n)):
            p.n[d] = int(n[d])
            p.b[d] = int(b[d])
            p.support[d] = int(support[d]) if support else 0
        p.loops = int(loops)
        p.prewin = WIN[prewin]
        p.prewin_param = float(prewin_param)
        p.flat_atten_db = float(flat_atten_db)
        p.p_fa = float(p_fa)
        p.noise_var = float(noise_var)
        p.gamma_override = float(gamma_override)
        p.mu = int(mu)
        p.random_tau = int(bool(random_tau))
        p.seed = int(seed) & ((1 << 64) - 1)
        p.max_batch = int(max_batch)
        p.mode = MODE[mode]
        self.params = p
        self.n, self.b, self.loops = tuple(int(v) for v in n), tuple(int(v) for v in b), int(loops)
        self.ndim = len(n)
        self.max_batch = int(max_batch)
        h = c_void_p()
        _check(L.rsft_plan_create(ctypes.byref(p), ctypes.byref(h)))
        self._h = h
        self.workspace = None
        info = RsftInfo()
        _check(L.rsft_get_info(self._h, ctypes.byref(info)))
        self.ntot, self.btot = info.ntot, info.btot
        self.bitmap_words, self.detect_words = info.bitmap_words, info.detect_words
        self.mode, self.lpad, self.workspace_bytes = info.mode, info.lpad, info.workspace_bytes

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _LIB is not None:
            _LIB.rsft_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # ---------------------------------------------------------------- host queries
    def schedule(self):
        k = self.loops * self.ndim
        s, si, t = (np.zeros(k, np.int64) for _ in range(3))
        _check(lib().rsft_get_schedule(self._h, s.ctypes.data_as(POINTER(c_int64)),
                                       si.ctypes.data_as(POINTER(c_int64)), t.ctypes.data_as(POINTER(c_int64))))
        sh = (self.loops, self.ndim)
        return s.reshape(sh), si.reshape(sh), t.reshape(sh)

    def set_schedule(self, sigma, tau=None):
        s, sp = _i64(np.asarray(sigma).reshape(-1))
        if tau is None:
            _check(lib().rsft_set_schedule(self._h, sp, None))
        else:
            t, tp = _i64(np.asarray(tau).reshape(-1))
            _check(lib().rsft_set_schedule(self._h, sp, tp))
        self.workspace = None

    def thresholds(self):
        be = np.zeros(self.loops)
        ga = np.zeros(self.loops)
        _check(lib().rsft_get_thresholds(self._h, be.ctypes.data_as(POINTER(c_double)),
                                         ga.ctypes.data_as(POINTER(c_double))))
        return be, ga

    def window(self, d, which):
        size = self.n[d] * (self.loops if which == 2 else 1)
        out = np.zeros(size)
        _check(lib().rsft_get_window(self._h, d, which, out.ctypes.data_as(POINTER(c_double))))
        return out.reshape(self.loops, self.n[d]) if which == 2 else out

    # ---------------------------------------------------------------- device
    def bind(self, device=None, stream=None):
        import torch
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        with torch.cuda.device(dev):
            self.workspace = torch.empty(max(int(self.workspace_bytes), 256), dtype=torch.uint8, device=dev)
            _check(lib().rsft_bind(self._h, c_void_p(self.workspace.data_ptr()), self.workspace.numel(),
                                   _stream_handle(stream)))
        return self

    def _need_bind(self):
        if self.workspace is None:
            raise RsftError(7, "plan not bound")

    def new_bitmaps(self, batch, nloops=None):
        import torch
        nl = self.loops if nloops is None else nloops
        return torch.empty((batch, nl, self.bitmap_words), dtype=torch.int32, device=self.device)

    def execute(self, x, loop_begin=0, loop_end=None, bitmaps=None, spectra=None, stream=None):
        """First stage (Alg. 1 l.5-10) on complex64 device tensor x [batch, *n]."""
        import torch
        self._need_bind()
        loop_end = self.loops if loop_end is None else loop_end
        batch = x.shape[0]
        assert x.dtype == torch.complex64 and x.is_cuda and x.is_contiguous()
        assert tuple(x.shape[1:]) == self.n
        if bitmaps is None:
            bitmaps = self.new_bitmaps(batch, loop_end - loop_begin)
        sp = c_void_p(spectra.data_ptr()) if spectra is not None else None
        _check(lib().rsft_execute(self._h, c_void_p(x.data_ptr()), batch, loop_begin, loop_end,
                                  c_void_p(bitmaps.data_ptr()), sp, _stream_handle(stream)))
        return bitmaps

    def execute_segments(self, x, bitmaps=None, spectra=None, stream=None):
        """Segment mode: x [batch, L, *n] complex64; loop l folds segment l.  Returns
        bitmaps [batch, L, words] (the input of detect / detect_compact)."""
        import torch
        self._need_bind()
        batch = x.shape[0]
        assert x.dtype == torch.complex64 and x.is_cuda and x.is_contiguous()
        assert x.shape[1] == self.loops and tuple(x.shape[2:]) == self.n
        if bitmaps is None:
            bitmaps = self.new_bitmaps(batch)
        sp = c_void_p(spectra.data_ptr()) if spectra is not None else None
        _check(lib().rsft_execute_segments(self._h, c_void_p(x.data_ptr()), batch, c_void_p(bitmaps.data_ptr()), sp,
                                           _stream_handle(stream)))
        return bitmaps

    def bucketize_partial(self, x_slab, dim0_offset, partial=None, stream=None):
        """Folded spectrum [L, B_tot] (layout [l][k_last][outer class]) of the dim-0 slab
        x_slab = rows [dim0_offset, dim0_offset + len) of one frame (variant B, linear in x)."""
        import torch
        self._need_bind()
        assert x_slab.dtype == torch.complex64 and x_slab.is_cuda and x_slab.is_contiguous()
        assert tuple(x_slab.shape[1:]) == self.n[1:]
        if partial is None:
            partial = torch.empty((self.loops, self.btot), dtype=torch.complex64, device=self.device)
        _check(lib().rsft_bucketize_partial(self._h, c_void_p(x_slab.data_ptr()), dim0_offset, x_slab.shape[0],
                                            c_void_p(partial.data_ptr()), _stream_handle(stream)))
        return partial

    def finalize(self, folded, loop_begin=0, loop_end=None, bitmaps=None, spectra=None, stream=None):
        """Bitmaps [loop_end - loop_begin, words] from summed folded spectra
        [loop_end - loop_begin, B_tot] (those loops' rows of the partial layout)."""
        import torch
        self._need_bind()
        loop_end = self.loops if loop_end is None else loop_end
        assert folded.dtype == torch.complex64 and folded.is_cuda and folded.is_contiguous()
        assert folded.shape[0] == loop_end - loop_begin
        if bitmaps is None:
            bitmaps = torch.empty((loop_end - loop_begin, self.bitmap_words), dtype=torch.int32, device=self.device)
        sp = c_void_p(spectra.data_ptr()) if spectra is not None else None
        _check(lib().rsft_finalize(self._h, c_void_p(folded.data_ptr()), loop_begin, loop_end,
                                   c_void_p(bitmaps.data_ptr()), sp, _stream_handle(stream)))
        return bitmaps

    def detect(self, bitmaps, dim0=None, detect=None, counts=None, stream=None):
        """Reverse map + accumulation + second stage (Alg. 1 l.11-14)."""
        import torch
        self._need_bind()
        batch = bitmaps.shape[0]
        d0b, d0e = (0, self.n[0]) if dim0 is None else dim0
        locs = (d0e - d0b) * (self.ntot // self.n[0])
        if detect is None:
            detect = torch.empty((batch, (locs + 31) // 32), dtype=torch.int32, device=self.device)
        cp = c_void_p(counts.data_ptr()) if counts is not None else None
        _check(lib().rsft_detect(self._h, c_void_p(bitmaps.data_ptr()), batch, d0b, d0e,
                                 c_void_p(detect.data_ptr()), cp, _stream_handle(stream)))
        return detect

    def compact(self, detect, capacity, idx=None, count=None, stream=None):
        import torch
        self._need_bind()
        batch = detect.shape[0]
        if idx is None:
            idx = torch.empty(max(capacity, 1), dtype=torch.int64, device=self.device)
        if count is None:
            count = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(lib().rsft_compact(self._h, c_void_p(detect.data_ptr()), batch, c_void_p(idx.data_ptr()),
                                  capacity, c_void_p(count.data_ptr()), _stream_handle(stream)))
        return idx, count

    def detect_compact(self, bitmaps, capacity, detect=None, idx=None, count=None, stream=None):
        """Second stage + compaction in one call (full range): (detect, idx, count)."""
        import torch
        self._need_bind()
        batch = bitmaps.shape[0]
        if detect is None:
            detect = torch.empty((batch, self.detect_words), dtype=torch.int32, device=self.device)
        if idx is None:
            idx = torch.empty(max(capacity, 1), dtype=torch.int64, device=self.device)
        if count is None:
            count = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(lib().rsft_detect_compact(self._h, c_void_p(bitmaps.data_ptr()), batch, c_void_p(detect.data_ptr()),
                                         c_void_p(idx.data_ptr()), capacity, c_void_p(count.data_ptr()),
                                         _stream_handle(stream)))
        return detect, idx, count

    def run(self, x, capacity, bitmaps=None, detect=None, idx=None, count=None, stream=None):
        """Whole hot path (execute all loops + detect + compact): (bitmaps, detect, idx, count)."""
        import torch
        self._need_bind()
        batch = x.shape[0]
        assert x.dtype == torch.complex64 and x.is_cuda and x.is_contiguous()
        assert tuple(x.shape[1:]) == self.n
        if bitmaps is None:
            bitmaps = self.new_bitmaps(batch)
        if detect is None:
            detect = torch.empty((batch, self.detect_words), dtype=torch.int32, device=self.device)
        if idx is None:
            idx = torch.empty(max(capacity, 1), dtype=torch.int64, device=self.device)
        if count is None:
            count = torch.empty(1, dtype=torch.int64, device=self.device)
        _check(lib().rsft_run(self._h, c_void_p(x.data_ptr()), batch, c_void_p(bitmaps.data_ptr()),
                              c_void_p(detect.data_ptr()), c_void_p(idx.data_ptr()), capacity,
                              c_void_p(count.data_ptr()), _stream_handle(stream)))
        return bitmaps, detect, idx, count

    def host_scratch_bytes(self, batch, capacity):
        return lib().rsft_host_scratch_bytes(self._h, batch, capacity)

    def run_host(self, h_x, capacity, scratch, stream=None):
        """End-to-end on a host (pinned) complex64 tensor: returns (indices ndarray, count)."""
        import torch
        self._need_bind()
        batch = h_x.shape[0]
        h_idx = torch.empty(max(capacity, 1), dtype=torch.int64, pin_memory=True)
        cnt = c_int64(0)
        _check(lib().rsft_run_host(self._h, c_void_p(h_x.data_ptr()), batch, c_void_p(h_idx.data_ptr()),
                                   capacity, ctypes.byref(cnt), c_void_p(scratch.data_ptr()),
                                   scratch.numel(), _stream_handle(stream)))
        n = min(cnt.value, capacity)
        return h_idx[:n].numpy().copy(), cnt.value

    def design_thresholds(self, K, p_d=0.9, p_fa=1e-6, eta_m=0.0, eta_p=1.0, omega=None, loops=0):
        """Optimal thresholds (Eq. opt) for this plan's windows: dict with mu,
        snr_min(_db), pd_bar, pfa_bar, gamma, alpha_bar, beta_bar, eta_m, F.  eta_p = 0 is
        the upper bound of Remark 3 (co-existing sinusoids detected with rate 1)."""
        d = RsftDesignParams()
        lib().rsft_default_design_params(ctypes.byref(d))
        d.K, d.p_d, d.p_fa, d.eta_m, d.eta_p, d.loops = K, p_d, p_fa, eta_m, eta_p, loops
        if omega is not None:
            for i, v in enumerate(omega):
                d.omega[i] = v
        r = RsftDesignResult()
        _check(lib().rsft_design_thresholds(self._h, ctypes.byref(d), ctypes.byref(r)))
        return {f: getattr(r, f) for f, _ in RsftDesignResult._fields_}

    def bartlett(self, x, gamma=None, p_fa=None, power=None, detect=None, scratch=None, stream=None):
        """Bartlett baseline (Alg. 2): x [batch, segments, *n] (or [segments, *n]) complex64 ->
        (power x [batch, *n], detect bitmap [batch, words])."""
        import torch
        self._need_bind()
        single = x.dim() == len(self.n) + 1
        xb = x.unsqueeze(0) if single else x
        batch, T = xb.shape[0], xb.shape[1]
        assert xb.dtype == torch.complex64 and xb.is_cuda and xb.is_contiguous() and tuple(xb.shape[2:]) == self.n
        if gamma is None:
            gamma = self.bartlett_threshold(T, p_fa if p_fa is not None else 1e-6)
        if power is None:
            power = torch.empty((batch,) + self.n, dtype=torch.float32, device=self.device)
        if detect is None:
            detect = torch.empty((batch, self.detect_words), dtype=torch.int32, device=self.device)
        if scratch is None and self.ntot > 8192:       # two-pass frames: [batch][T][N_tot]
            scratch = torch.empty((batch, T) + self.n, dtype=torch.complex64, device=self.device)
        _check(lib().rsft_bartlett(self._h, c_void_p(xb.data_ptr()), batch, T,
                                   c_void_p(scratch.data_ptr()) if scratch is not None else None,
                                   c_void_p(power.data_ptr()), float(gamma), c_void_p(detect.data_ptr()),
                                   _stream_handle(stream)))
        if single:
            return power[0], detect[0]
        return power, detect

    def bartlett_threshold(self, segments, p_fa):
        g = c_double(0.0)
        _check(lib().rsft_bartlett_threshold(self._h, segments, p_fa, ctypes.byref(g)))
        return g.value

    def last_launch_count(self):
        return int(lib().rsft_last_launch_count(self._h))


def synthesize(n, batch, segments, omega, sigma_b, sigma_n, seed, out=None, stream=None):
    """GPU scene generator (rsft_synthesize): complex64 [batch, segments, *n] per Eq. sig_model
    with per-segment Swerling amplitudes.  omega: [batch, K, D] bins, sigma_b: [batch, K]
    (torch fp64 CUDA tensors or None when K = 0)."""
    import torch
    n = tuple(int(v) for v in n)
    K = 0 if omega is None else int(omega.shape[1])
    if out is None:
        out = torch.empty((batch, segments) + n, dtype=torch.complex64, device="cuda")
    nn = (c_int64 * len(n))(*n)
    op = c_void_p(omega.data_ptr()) if K else None
    sp = c_void_p(sigma_b.data_ptr()) if K else None
    _check(lib().rsft_synthesize(nn, len(n), batch, segments, K, op, sp, float(sigma_n), int(seed),
                                 c_void_p(out.data_ptr()), _stream_handle(stream)))
    return out


def bitmap_to_bool(words, nbits):
    """uint32 bitmap words (any int32 array) -> bool array of nbits (host helper)."""
    w = np.ascontiguousarray(np.asarray(words).astype(np.uint32))
    bits = np.unpackbits(w.view(np.uint8), bitorder="little")
    return bits[:nbits].astype(bool)
