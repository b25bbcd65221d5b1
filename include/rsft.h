/*
 * rsft.h — C ABI of the B200-native (sm_100a) Realistic Sparse Fourier Transform hot path.
 *
 * Method: Wang, Patel, Petropulu, arXiv 1610.01050, Algorithm 1.
 * Citations "P:<line>" refer to /root/reference/PAPER.md; "Lnn" to the readings in DESIGN.md.
 *
 * Pipeline per frame x in C^{N_0 x ... x N_{D-1}} (row-major, last dim contiguous), per loop l:
 *   y = W x            pre-permutation window            (Alg. 1 l.5,  P:220)
 *   p = P_{sigma,tau} y  per-dimension permutation       (Def. 1; l.6 P:221)
 *   z = Wbar p         flat window                        (l.7 P:222)
 *   f = Aliasing(z)    fold into B_0 x ... buckets        (Def. 2; l.8 P:223)
 *   fhat = NDFFT_B(f)  forward, unnormalised              (l.9 P:224; L7)
 *   c_l = |fhat|^2 > gamma_l                              (l.10 P:225; Eq. tpd; L8)
 *   abar = sum_l Reverse(c_l)                             (l.11-12 P:226-227; Def. 4; Eq. a_i)
 *   o = {i : abar_i >= mu}                                (l.14 P:229; L10)
 *
 * Conventions (all entry points):
 *  - Every call returns rsft_status; RSFT_OK == 0.  No exceptions, no abort().
 *  - The plan is host memory owned by the library (rsft_plan_destroy frees it).
 *  - EVERY device buffer is caller-owned (input, outputs, workspace).  The library never
 *    allocates device memory.  It never synchronises, except in the one-time rsft_bind
 *    and in rsft_run_host (both documented below).
 *  - Device work is issued only on the `stream` argument (a cudaStream_t passed as void*;
 *    NULL = the legacy default stream).  Results are valid after the caller syncs it.
 *  - Argument / shape errors are returned before any launch.  Launch failures return
 *    RSFT_E_CUDA; the CUDA error string is kept in rsft_last_error().
 *  - One host thread per plan at a time; distinct plans are independent.
 *  - Data types: input frames are complex64 (interleaved float32 re, im).  Bitmaps are
 *    uint32 words, bit k of word w <-> flat index 32 w + k (row-major flattening).
 */
#ifndef RSFT_H
#define RSFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rsft_plan_s* rsft_plan_t;

typedef enum {
  RSFT_OK = 0,
  RSFT_E_ARG = 1,          /* null pointer, bad range, mu/loops/p_fa out of range     */
  RSFT_E_SHAPE = 2,        /* N_d or B_d not a power of two, B_d > N_d, support rule (L2)      */
  RSFT_E_SIGMA = 3,        /* even sigma in rsft_set_schedule (Eq. mod_inv)     */
  RSFT_E_UNSUPPORTED = 4,  /* D > 3, B_d > 64, L > 63, N_last < 32, or tables beyond smem     */
  RSFT_E_WORKSPACE = 5,    /* workspace missing, too small or misaligned (256 B)              */
  RSFT_E_CUDA = 6,         /* a CUDA runtime call or launch failed (see rsft_last_error)      */
  RSFT_E_STATE = 7         /* plan not bound (rsft_bind) before a device call                 */
} rsft_status;

typedef enum {
  RSFT_WIN_RECT = 0,       /* w = 1                                                           */
  RSFT_WIN_HANN = 1,       /* periodic Hann w[n] = sin^2(pi n / N)  (BASELINE; L3)            */
  RSFT_WIN_CHEB = 2        /* periodic Dolph-Chebyshev, prewin_param dB        */
} rsft_win;

typedef enum {
  RSFT_MODE_AUTO = 0,      /* library picks                                                   */
  RSFT_MODE_FUSED = 1,     /* one CTA per frame: fold + FFT + threshold fused (D <= 2)        */
  RSFT_MODE_SPLIT = 2      /* CTA per (frame, outer residue class) + outer-FFT kernel (D >= 2) */
} rsft_mode;

typedef struct {
  int32_t ndim;            /* D in 1..3 ("any fixed dimension")                          */
  int64_t n[3];            /* N_d, powers of two                                       */
  int64_t b[3];            /* B_d, powers of two, 1 <= B_d <= min(N_d, 64) (Def. 2)       */
  int64_t support[3];      /* flat-window support W_d; 0 => N_d; need 2 B_d | W_d <= N_d */
  int32_t loops;           /* L (the paper's T iterations, Alg. 1 l.4 P:219), 1..63 (> 32: one
                              pass over x per 32 loops; rsft_bucketize_partial: <= 32)        */
  int32_t prewin;          /* rsft_win of the pre-permutation window               */
  double prewin_param;     /* Chebyshev attenuation dB when prewin == RSFT_WIN_CHEB           */
  double flat_atten_db;    /* Dolph-Chebyshev taper of the flat window, default 60 (L2)       */
  double p_fa;             /* first-stage per-bucket false-alarm probability, (0,1) (L8)      */
  double noise_var;        /* sigma_n^2 > 0 (L11)                                      */
  double gamma_override;   /* > 0: gamma_l = gamma_override for every loop       */
  int32_t mu;              /* second-stage vote threshold 1..L (L9)                    */
  int32_t random_tau;      /* 0: tau = 0; 1: seeded tau (L4)                          */
  uint64_t seed;           /* sigma/tau schedule seed (L5)                                    */
  int64_t max_batch;       /* largest batch passed to execute/detect (sizes the workspace)    */
  int32_t mode;            /* rsft_mode                                                       */
} rsft_params;

/* Fill defaults: D=1, loops=1, Hann, 60 dB flat taper, p_fa=1e-6, noise_var=1, mu=loops,
 * tau=0, max_batch=1, mode auto. */
void rsft_default_params(rsft_params* p);

/* Validate params and build the host plan (windows, sigma/sigma^{-1}/tau schedule, per-loop
 * weight tables, beta_l, gamma_l).  Host only: no CUDA call.  Errors: E_ARG, E_SHAPE,
 * E_UNSUPPORTED.  *out is set to NULL on error. */
rsft_status rsft_plan_create(const rsft_params* params, rsft_plan_t* out);
void rsft_plan_destroy(rsft_plan_t plan);

/* SURVEY §8(b) spelling of the same two calls: rsft_plan(params, device, out) creates the plan
 * (host only, like rsft_plan_create) and records `device` (>= 0) as the CUDA device rsft_bind
 * must be called on (rsft_bind returns E_STATE on another current device; -1 = any);
 * rsft_destroy == rsft_plan_destroy. */
rsft_status rsft_plan(const rsft_params* params, int32_t device, rsft_plan_t* out);
void rsft_destroy(rsft_plan_t plan);

/* Replace the seeded schedule.  sigma: [L][D] odd values in [N_d] (Def. 1: sigma invertible
 * mod N_d); tau: [L][D] in [N_d] or NULL (=> 0).  Recomputes tables, beta, gamma and
 * marks the plan unbound.  Errors: E_SIGMA (even sigma), E_ARG. */
rsft_status rsft_set_schedule(rsft_plan_t plan, const int64_t* sigma, const int64_t* tau);

/* Read back the schedule ([L][D] each; any pointer may be NULL). */
rsft_status rsft_get_schedule(rsft_plan_t plan, int64_t* sigma, int64_t* sigma_inv, int64_t* tau);

/* beta_l = ||Wbar P_sigma_l w||^2 (Eq. alpha_beta) and gamma_l (Eq. tpd),
 * fp64, [L] each; either pointer may be NULL. */
rsft_status rsft_get_thresholds(rsft_plan_t plan, double* beta, double* gamma);

/* Plan-time windows for dimension d, fp64 [N_d]: which = 0 -> pre-window w_d;
 * which = 1 -> real flat prototype g_d (gbar_d = g_d e^{-j pi t/B_d}, L1-L2);
 * which = 2 -> fp32 per-loop weight table h_{l,d}[s] widened to fp64, [L][N_d] (I3). */
rsft_status rsft_get_window(rsft_plan_t plan, int32_t d, int32_t which, double* out);

/* Derived sizes. */
typedef struct {
  int64_t ntot, btot;          /* prod N_d, prod B_d                                        */
  int64_t bitmap_words;        /* words per loop per frame = ceil(B_tot / 32)                */
  int64_t detect_words;        /* words per frame of the detection bitmap = ceil(N_tot / 32) */
  int32_t mode;                /* resolved rsft_mode for batch = max_batch                   */
  int32_t lpad;                /* compile-time loop count used by the fold kernels          */
  size_t workspace_bytes;
} rsft_info;
rsft_status rsft_get_info(rsft_plan_t plan, rsft_info* info);
/* Workspace size.  The plan is host-only (no CUDA call), so the split-mode folded-spectra
 * buffer is sized for a 148-SM device (B200); on a device with more SMs the launcher keeps
 * fewer dim-0 chunks per class (memory-safe, slightly less parallel). */
size_t rsft_workspace_bytes(rsft_plan_t plan);

/* Upload the plan tables into the caller-owned device workspace (>= rsft_workspace_bytes,
 * 256-byte aligned) on `stream`, on the current CUDA device, and synchronise `stream`.  The workspace must stay alive
 * and untouched while the plan is used.  Errors: E_WORKSPACE, E_CUDA. */
rsft_status rsft_bind(rsft_plan_t plan, void* d_workspace, size_t bytes, void* stream);

/* First stage for loops [loop_begin, loop_end) of `batch` frames (Alg. 1 l.5-10):
 *   d_x        device, complex64 [batch][N_0]...[N_{D-1}], 16-byte aligned, read once.
 *   d_bitmaps  device, uint32 [batch][loop_end-loop_begin][bitmap_words]: bit k set iff
 *              |fhat_l[k]|^2 > gamma_l (flat bucket index k, row-major over B_d).
 *   d_spectra  NULL, or device complex64 [batch][loop_end-loop_begin][B_tot]: fhat (parity).
 * Errors: E_ARG (range, batch > max_batch, null), E_STATE, E_CUDA. */
rsft_status rsft_execute(rsft_plan_t plan, const void* d_x, int64_t batch, int32_t loop_begin,
                         int32_t loop_end, uint32_t* d_bitmaps, void* d_spectra, void* stream);

/* Segment mode ("iterations ... on different segments"; Eq. sig_model):
 * loop l runs the first stage on segment l of each frame.
 *   d_x        device complex64 [batch][L][N_0]...[N_{D-1}] (segment l of frame f at (f L + l) N_tot).
 *   d_bitmaps  device uint32 [batch][L][bitmap_words]: the input of rsft_detect, unchanged.
 *   d_spectra  NULL or device complex64 [batch][L][B_tot].
 * Fused mode: one strided launch per loop; split mode: one launch per (frame, segment).
 * Errors: as rsft_execute. */
rsft_status rsft_execute_segments(rsft_plan_t plan, const void* d_x, int64_t batch, uint32_t* d_bitmaps,
                                  void* d_spectra, void* stream);

/* Slab sharding of ONE frame (SURVEY §8(e) variant B).  Pre-window, permutation, flat
 * window and aliasing (Alg. 1 l.5-8) are linear in x (Eqs. z, l: P:272-279), so
 * dim-0 slabs produce partial folded spectra that add up (in any order, up to fp32 rounding)
 * to the whole frame's.  Split mode (D >= 2) only.
 *   d_x_slab   device complex64 [dim0_len][N_1]...[N_{D-1}]: rows [dim0_offset,
 *              dim0_offset + dim0_len) of one frame, 16-byte aligned.
 *   dim0_offset, dim0_len: multiples of B_0, dim0_len > 0, offset + len <= N_0.
 *   d_partial  device complex64 [L][B_last][B_tot / B_last] (all loops of the plan): the
 *              slab's folded spectrum after the last-dim DFT (the last-dim relabelling and
 *              half-bucket twiddle applied), indexed [l][k_last][outer residue class];
 *              overwritten.  Sum the partials of all slabs, then call rsft_finalize.
 * Errors: E_ARG (range, alignment, null), E_UNSUPPORTED (fused-mode plan), E_STATE, E_CUDA. */
rsft_status rsft_bucketize_partial(rsft_plan_t plan, const void* d_x_slab, int64_t dim0_offset, int64_t dim0_len,
                                   void* d_partial, void* stream);

/* Finish the first stage of loops [loop_begin, loop_end) from summed folded spectra
 * (Alg. 1 l.9-10): outer relabelling + half-bucket twiddles, outer-dims FFT, |.|^2 > gamma_l.
 *   d_folded   device complex64 [loop_end-loop_begin][B_last][B_tot / B_last]: rows
 *              loop_begin.. of the rsft_bucketize_partial layout, summed over slabs (e.g. this
 *              rank's block after a reduce-scatter over loops).
 *   d_bitmaps  device uint32 [loop_end-loop_begin][bitmap_words] (overwritten).
 *   d_spectra  NULL or device complex64 [loop_end-loop_begin][B_tot].
 * Errors: E_ARG, E_UNSUPPORTED (fused-mode plan), E_STATE, E_CUDA. */
rsft_status rsft_finalize(rsft_plan_t plan, const void* d_folded, int32_t loop_begin, int32_t loop_end,
                          uint32_t* d_bitmaps, void* d_spectra, void* stream);

/* Reverse mapping + accumulation + second-stage test (Alg. 1 l.11-14) for locations whose
 * dim-0 index lies in [dim0_begin, dim0_end) (sharded voting; full range = [0, N_0)):
 *   d_bitmaps  device uint32 [batch][L][bitmap_words] — ALL loops of the plan.
 *   d_detect   device uint32 [batch][ceil((dim0_end-dim0_begin) * N_tot/N_0 / 32)]:
 *              bit i set iff abar_i >= mu (location index relative to the slab start).
 *   d_counts   NULL, or device uint8 [batch][(dim0_end-dim0_begin) * N_tot/N_0]: abar.
 * D == 1 requires the full range.  The slab size times N_tot/N_0 must be a multiple of 32.
 * Errors: E_ARG, E_STATE, E_CUDA. */
rsft_status rsft_detect(rsft_plan_t plan, const uint32_t* d_bitmaps, int64_t batch,
                        int64_t dim0_begin, int64_t dim0_end, uint32_t* d_detect,
                        uint8_t* d_counts, void* stream);

/* Detection bitmap (full range, [batch][detect_words]) -> ascending flat indices
 * frame * N_tot + i of the set bits, written to d_idx[0 .. min(count, capacity)).
 * *d_count (device int64) receives the true count; count > capacity means truncated
 * (no sync is performed, so overflow is reported in *d_count, not in the return value).
 * Uses the workspace's compaction scratch.  Errors: E_ARG, E_STATE, E_CUDA. */
rsft_status rsft_compact(rsft_plan_t plan, const uint32_t* d_detect, int64_t batch,
                         int64_t* d_idx, int64_t capacity, int64_t* d_count, void* stream);

/* Second stage + compaction (full dim-0 range): the same detection bitmap as rsft_detect and
 * the same index list / count as rsft_compact.  Runs the vote kernel for the frame shape
 * (D = 1: a warp per frame; D = 2 with N_0 <= 256: a CTA per frame; D = 3 with small planes: a
 * warp per dim-0 plane; else a CTA per vote region), which also writes per-region detection
 * counts and region-local sorted index lists into the workspace; then, for up to 8192 vote
 * regions, ONE launch in which every CTA sums the counts of the preceding regions itself and
 * copies its regions' lists to their offsets (total -> *d_count); for more regions a two-pass
 * parallel scan of the region counts and a separate writer.  A region whose list overflowed is
 * re-read from its detection words.  Both forms give the same list (integer work).
 * Errors: E_ARG, E_STATE, E_WORKSPACE, E_CUDA. */
rsft_status rsft_detect_compact(rsft_plan_t plan, const uint32_t* d_bitmaps, int64_t batch,
                                uint32_t* d_detect, int64_t* d_idx, int64_t capacity,
                                int64_t* d_count, void* stream);

/* Whole hot path on device buffers (Alg. 1 l.5-14), with the outputs of rsft_execute
 * (all loops) + rsft_detect_compact (d_bitmaps [batch][L][bitmap_words], d_detect
 * [batch][detect_words], sorted indices, *d_count).  Fused-mode plans run first and second stage
 * in ONE warp-specialised kernel: D = 1 with a flat-window support <= 1024 (k_gather1d with vote
 * warps) and D = 2 with L <= 8, B_0 <= 32, B_1 in {8, 16, 32}, N_1 in {128, 256}, N_0 <= 1024
 * (k_fused2v: fold warps stream the frame while epilogue warps FFT, threshold and vote the
 * previous one); then the region scan + index writer of rsft_detect_compact.  Other plans issue
 * rsft_execute + rsft_detect_compact back to back on `stream` (programmatic dependent launches).
 * Bucket values come from a different FFT order than rsft_execute's (equal to fp32 rounding).
 * Errors: as rsft_execute and rsft_detect_compact. */
rsft_status rsft_run(rsft_plan_t plan, const void* d_x, int64_t batch, uint32_t* d_bitmaps, uint32_t* d_detect,
                     int64_t* d_idx, int64_t capacity, int64_t* d_count, void* stream);

/* End-to-end convenience call on HOST buffers (blocking: synchronises `stream`):
 * copies h_x (complex64 [batch][N...], pinned recommended) into d_scratch, runs rsft_run,
 * and copies the count and min(count, capacity) indices back.
 * d_scratch: device buffer of >= rsft_host_scratch_bytes(plan, batch, capacity) bytes.
 * Returns the true count in *h_count.  Errors: as above. */
size_t rsft_host_scratch_bytes(rsft_plan_t plan, int64_t batch, int64_t capacity);
rsft_status rsft_run_host(rsft_plan_t plan, const void* h_x, int64_t batch, int64_t* h_idx,
                          int64_t capacity, int64_t* h_count, void* d_scratch,
                          size_t scratch_bytes, void* stream);

/* Optimal thresholds (Eq. opt; host, fp64): minimise the worst-case per-sample
 * SNR_min for the final targets p_d / p_fa of Problem 1, using the
 * first-stage laws of Eq. bpd and the asymptotic Normal laws of the votes of
 * Claims 2-3; alpha_bar / beta_bar are the permutation averages of Eq.
 * alpha_beta for this plan's windows (alpha at the Claim 1 peak bucket of the
 * weakest sinusoid at omega, every odd sigma, tau = 0), separable over dimensions. */
typedef struct {
  int32_t K;               /* sparsity budget K                                        */
  double p_d, p_fa;        /* final per-location detection / false-alarm targets       */
  double eta_m;            /* 6-dB bandwidth of the pre-window in bins (product over dims);
                              <= 0: measured from the plan's windows                           */
  double eta_p;            /* Claim 3 calibration (>= 1, 1 = lower bound, Remark 3); 0: upper
                              bound (co-existing sinusoids detected with rate 1)              */
  double omega[3];         /* weakest sinusoid frequency per dim, in DFT bins (e.g. 64.5)      */
  int32_t loops;           /* T; 0 => the plan's L                                             */
} rsft_design_params;

typedef struct {
  int32_t mu;              /* optimal second-stage threshold mu* in [T]                        */
  double snr_min, snr_min_db;   /* SNR_min* (linear, dB)                                       */
  double pd_bar, pfa_bar;  /* first-stage rates at the optimum                                 */
  double gamma;            /* gamma* = sigma_n^2 beta_bar ln(1 / pfa_bar) (Eq. bpd)            */
  double alpha_bar, beta_bar, eta_m, F;   /* inputs as used; F = T K eta_m / B (Claim 3)       */
} rsft_design_result;

/* Defaults: K = 1, p_d = 0.9, p_fa = 1e-6, eta_m measured, eta_p = 1, omega = 0.5 bins, T = L. */
void rsft_default_design_params(rsft_design_params* d);
/* Errors: E_ARG (ranges; infeasible design, e.g. K eta_m >= B per Remark 2 P:517). Host only. */
rsft_status rsft_design_thresholds(rsft_plan_t plan, const rsft_design_params* d, rsft_design_result* out);

/* Scene generator for Monte Carlo runs (harness utility, not part of the method): writes
 * complex64 d_x [batch][segments][N...] following Eq. sig_model / sinusoid,
 * separable over dims: x = sum_k b_{f,k,s} prod_d e^{j 2 pi omega_{f,k,d} n_d / N_d} + nu, with
 * b_{f,k,s} ~ CN(0, sigma_b[f][k]^2) redrawn per segment and nu ~ CN(0, sigma_n^2);
 * counter-based random numbers (SplitMix64 + Box-Muller; synth.counter_normals mirrors them).
 *   n[ndim]: N_d;  d_omega: device fp64 [batch][K][ndim] in DFT bins;  d_sigma_b: device fp64
 *   [batch][K].  Errors: E_ARG, E_CUDA. */
rsft_status rsft_synthesize(const int64_t* n, int32_t ndim, int64_t batch, int32_t segments, int32_t K,
                            const double* d_omega, const double* d_sigma_b, double sigma_n, uint64_t seed,
                            void* d_x, void* stream);

/* Bartlett baseline (Algorithm 2, App. A): for each frame
 * and each of its `segments` segments u = W r_s (the plan's separable pre-window), N-D FFT
 * (hand-written, N_d <= 4096), x += |u_hat|^2; then bit i of d_detect = (x_i / segments > gamma).
 * Frames of <= 8192 samples run in one pass (power kept on chip); larger frames (D >= 2, with
 * N_tot / N_0 <= 8192) in two passes through d_scratch (inner dims, then dim 0 + |.|^2).
 *   d_x      device complex64 [batch][segments][N...];
 *   d_scratch device complex64 [batch][segments][N_tot] when N_tot > 8192, else unused (may be NULL);
 *   d_power  device fp32 [batch][N_tot] (x, overwritten);  d_detect NULL or uint32
 *            [batch][detect_words].  Errors: E_ARG, E_STATE, E_UNSUPPORTED (N_d > 4096, no
 *            scratch, inner block > 8192), E_CUDA. */
rsft_status rsft_bartlett(rsft_plan_t plan, const void* d_x, int64_t batch, int32_t segments, void* d_scratch,
                          float* d_power, double gamma, uint32_t* d_detect, void* stream);
/* gamma of Eq. bartlettROC for a per-bin false-alarm target: the H'0 statistic is
 * N(sigma_n^2 beta', sigma_n^4 beta'^2 / T), beta' = ||w||^2; gamma = sigma_n^2 beta'
 * (1 + Phi^{-1}(1 - p_fa) / sqrt(T)).  Host only. */
rsft_status rsft_bartlett_threshold(rsft_plan_t plan, int32_t segments, double p_fa, double* gamma);

/* Number of kernels the last execute/detect/compact/run_host call launched. */
int32_t rsft_last_launch_count(rsft_plan_t plan);

const char* rsft_status_string(rsft_status s);
const char* rsft_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RSFT_H */
