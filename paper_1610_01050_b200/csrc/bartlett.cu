// Bartlett baseline: Algorithm 2 of the paper's Appendix A
// (P:926-943): for every segment s, u = W r_s (the plan's separable pre-window), u_hat =
// N-D FFT(u) (forward, unnormalised), x += |u_hat|^2; then l = x / T > gamma (NP test,
// Eq. bartlettROC).  The dense comparison workload for the RSFT's complexity claim
// (Tables I-II).  Hand-written FFTs (no cuFFT), radix-2 DIT in shared memory.
// Data movement is the design point (the FFT is cheap next to HBM at these sizes):
//  * frames of <= 8192 samples (c1: 4096): ONE pass -- a CTA keeps the frame's power in shared
//    memory while it streams the T segments (window on load, N-D FFT, |.|^2), then writes the
//    power and the detection words once: HBM = T N 8 B read + N 4 B written.
//  * larger frames (D >= 2, dim-0 rows of <= 8192 samples; c2, c3, c4): TWO passes -- pass 1
//    transforms the contiguous inner block (all dims but 0) of a tile of dim-0 rows, window
//    fused into the load, into the scratch (T N 8 B read + T N 8 B written, coalesced); pass 2
//    transforms dim 0 for a tile of adjacent inner columns and accumulates |.|^2 over the T
//    segments in registers, writing power and detection bits once (T N 8 B read + N 4 B).
//    3x the input bytes, the minimum for a 2-D FFT whose frame exceeds one SM's shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "rsft_internal.h"

namespace rsft {

constexpr int kBartTile = 8192;            // complex elements per CTA tile (64 KiB smem)
constexpr int kBartThreads = 512;

// In-place radix-2 DIT along one axis of a shared-memory tile (bit-reversed input, natural
// output): 2^lg points `ps` apart; line r of nlines starts at (r >> sh) * hs + (r & (2^sh - 1)) * ls.
// tw[k] = e^{-j 2 pi k / 4096} for k < 2048 (shared copy); one barrier per stage.
__device__ __forceinline__ void bart_fft_axis(float2* sv, int lg, int ps, int nlines, int sh, int hs, int ls,
                                              const float2* __restrict__ tw) {
  if (lg == 0) return;
  const int nbf = nlines << (lg - 1);
  const int lm = (1 << sh) - 1;
  for (int s = 1; s <= lg; ++s) {
    const int half = 1 << (s - 1);
    for (int bf = threadIdx.x; bf < nbf; bf += blockDim.x) {
      const int r = bf >> (lg - 1), q = bf & ((1 << (lg - 1)) - 1);
      const int j = q & (half - 1), g = q >> (s - 1);
      float2* e0 = sv + (r >> sh) * hs + (r & lm) * ls + ((g << s) + j) * ps;
      float2* e1 = e0 + half * ps;
      const float2 t = tw[j << (12 - s)];
      const float2 b = *e1;
      const float2 tb = make_float2(t.x * b.x - t.y * b.y, t.x * b.y + t.y * b.x);
      const float2 a = *e0;
      *e0 = make_float2(a.x + tb.x, a.y + tb.y);
      *e1 = make_float2(a.x - tb.x, a.y - tb.y);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int bart_brev(int v, int lg) { return lg ? (int)(__brev((unsigned)v) >> (32 - lg)) : 0; }

struct BartGeo {                           // dims right-aligned: (n0, n1, n2), D = 1..3
  int n0, n1, n2, lg0, lg1, lg2;
  const float* w0; const float* w1; const float* w2;
};

// Pass 1 / single pass.  Tile = `rows` consecutive dim-0 rows (all of dims 1, 2), contiguous in
// memory.  single: the tile is the whole frame; the CTA loops over the T segments keeping the
// power in shared memory, then writes power + detection.  Otherwise: one (frame, segment, row
// tile) per CTA iteration, written to the scratch (natural order).
__global__ void __launch_bounds__(kBartThreads) k_bart_inner(PlanDev pd, BartGeo g, const float2* __restrict__ x,
                                                             int64_t batch, int T, int rows, int single,
                                                             float2* __restrict__ scratch, float* __restrict__ power,
                                                             float scale, float gamma, uint32_t* __restrict__ det) {
  extern __shared__ __align__(16) float2 bsm[];
  float2* tw = bsm;                                  // [2048]
  float2* sv = tw + 2048;                            // [rows * n1 * n2]
  float* pw = reinterpret_cast<float*>(sv + kBartTile);   // single: [n0 n1 n2]
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) tw[i] = pd.btw[i];
  const int inner = g.n1 * g.n2, elems = rows * inner;
  const int lgi = g.lg1 + g.lg2;
  const int64_t ntot = (int64_t)g.n0 * inner;
  const int64_t tiles_per_seg = g.n0 / rows;
  const int64_t units = single ? batch : batch * T * tiles_per_seg;
  const bool fft0 = single && g.n0 > 1;              // single pass also transforms dim 0
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t frame = single ? u : u / (T * tiles_per_seg);
    const int seg0 = single ? 0 : (int)((u / tiles_per_seg) % T);
    const int tile = single ? 0 : (int)(u % tiles_per_seg);
    if (single)
      for (int e = threadIdx.x; e < elems; e += blockDim.x) pw[e] = 0.f;
    for (int s = seg0; s < (single ? T : seg0 + 1); ++s) {
      __syncthreads();                               // tw ready / previous tile's readers done
      const float2* src = x + ((size_t)frame * T + s) * ntot + (size_t)tile * elems;
      for (int e = threadIdx.x; e < elems; e += blockDim.x) {
        const int i2 = e & (g.n2 - 1), i1 = (e >> g.lg2) & (g.n1 - 1), r = e >> lgi;
        const float w = g.w0[tile * rows + r] * g.w1[i1] * g.w2[i2];
        float2 v = src[e];
        v.x *= w; v.y *= w;
        const int pr = fft0 ? bart_brev(r, g.lg0) : r;
        sv[(pr << lgi) + (bart_brev(i1, g.lg1) << g.lg2) + bart_brev(i2, g.lg2)] = v;
      }
      __syncthreads();
      bart_fft_axis(sv, g.lg2, 1, rows * g.n1, 0, g.n2, 0, tw);                 // dim 2 (contiguous)
      bart_fft_axis(sv, g.lg1, g.n2, rows * g.n2, g.lg2, g.n1 * g.n2, 1, tw);   // dim 1
      if (fft0) bart_fft_axis(sv, g.lg0, inner, inner, lgi, 0, 1, tw);          // dim 0 (single)
      if (single) {
        for (int e = threadIdx.x; e < elems; e += blockDim.x) {
          const float2 v = sv[e];
          pw[e] += v.x * v.x + v.y * v.y;
        }
      } else {
        float2* dst = scratch + ((size_t)frame * T + s) * ntot + (size_t)tile * elems;
        for (int e = threadIdx.x; e < elems; e += blockDim.x) dst[e] = sv[e];
      }
    }
    if (single) {
      __syncthreads();
      float* pdst = power + (size_t)frame * ntot;
      const int64_t words = (ntot + 31) >> 5;
      for (int e0 = threadIdx.x & ~31; e0 < ((elems + 31) & ~31); e0 += blockDim.x) {
        const int e = e0 + (threadIdx.x & 31);
        const float p = e < elems ? pw[e] : 0.f;
        if (e < elems) pdst[e] = p;
        const unsigned word = __ballot_sync(0xffffffffu, e < elems && p * scale > gamma);
        if (det && (threadIdx.x & 31) == 0) det[(size_t)frame * words + (e0 >> 5)] = word;
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// Warp-level FFT of n = 32 M points held in registers (no barrier): lane l holds
// v[k] = x[l + 32 k]; an in-lane M-point DIF over k, the twiddles W_n^{l q1}, then a 32-point
// DIF across the lanes (xor shuffles).  On return lane p holds v[r] = X[brev_M(r) + M brev5(p)].
// t = half-circle table e^{-j 2 pi k / 4096}, k < 2048, in shared memory.
// ---------------------------------------------------------------------------------------
__constant__ float2 c_btw[2048];                       // e^{-j 2 pi k / 4096}, k < 2048 (set at bind)

// compile-time twiddle indices: the constant bank (folds into the FFMA operands)
__device__ __forceinline__ float2 bart_twc(int j, int lgn) {
  const int i = (j << (12 - lgn)) & 4095;
  const float2 w = c_btw[i & 2047];
  return i < 2048 ? w : make_float2(-w.x, -w.y);
}
__device__ __forceinline__ float2 bart_twn(const float2* t, int j, int lgn) {
  const int i = (j << (12 - lgn)) & 4095;
  const float2 w = t[i & 2047];
  return i < 2048 ? w : make_float2(-w.x, -w.y);
}
__device__ __forceinline__ float2 bart_cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
constexpr int bart_lg(int m) { return m <= 1 ? 0 : 1 + bart_lg(m / 2); }
__device__ __forceinline__ int bart_brev_c(int v, int lg) { return lg ? (int)(__brev((unsigned)v) >> (32 - lg)) : 0; }

// in-lane M-point DIF (natural in, bit-reversed out); twiddles W_{2 span}^j from the constant
// bank, indexed as W_n^{j n / (2 span)} with n = 32 M (lgn = log2 n)
template <int M>
__device__ __forceinline__ void bart_lane_dif(float2 (&v)[M], int lgn) {
  constexpr int LM = bart_lg(M);
#pragma unroll
  for (int s = 0; s < LM; ++s) {
#pragma unroll
    for (int e = 0; e < M / 2; ++e) {
      const int span = M >> (s + 1);
      const int j = e & (span - 1), blk = (e / span) * 2 * span;
      const float2 a = v[blk + j], b = v[blk + j + span];
      v[blk + j] = make_float2(a.x + b.x, a.y + b.y);
      const float2 d = make_float2(a.x - b.x, a.y - b.y);
      v[blk + j + span] = j == 0 ? d : bart_cmul(d, bart_twc(j * (16 * M / span), lgn));
    }
  }
}

// 1024-point FFT of a warp's line with a shared-memory transpose instead of cross-lane shuffles:
// in-lane 32-point DIF over k, twiddles W_1024^{l q1}, transpose through the warp's 32 x 33
// scratch xs (lane q1 then holds Y_l[q1] for all l), in-lane 32-point DIF over l.
// On return lane q1 holds v[r] = X[q1 + 32 brev5(r)].
__device__ __forceinline__ void bart_warp_fft1024(float2 (&v)[32], int lane, const float2* __restrict__ t,
                                                  float2* __restrict__ xs) {
  bart_lane_dif<32>(v, 10);
  const float2 w1 = bart_twn(t, lane, 10);
  float2 cur = w1;
#pragma unroll
  for (int q1 = 1; q1 < 32; ++q1) {
    const int r = bart_brev_c(q1, 5);
    v[r] = bart_cmul(v[r], cur);
    cur = bart_cmul(cur, w1);
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) xs[bart_brev_c(r, 5) * 33 + lane] = v[r];
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; ++l) v[l] = xs[lane * 33 + l];
  __syncwarp();
  bart_lane_dif<32>(v, 10);
}

template <int M>
__device__ __forceinline__ void bart_warp_fft(float2 (&v)[M], int lane, int lgn, const float2* __restrict__ t,
                                              const float2 (&stw)[5]) {
  constexpr int LM = bart_lg(M);
#pragma unroll
  for (int s = 0; s < LM; ++s) {                      // in-lane DIF over k (span M / 2^{s+1})
#pragma unroll
    for (int e = 0; e < M / 2; ++e) {
      const int span = M >> (s + 1);
      const int j = e & (span - 1), blk = (e / span) * 2 * span;
      const float2 a = v[blk + j], b = v[blk + j + span];
      v[blk + j] = make_float2(a.x + b.x, a.y + b.y);
      const float2 d = make_float2(a.x - b.x, a.y - b.y);
      v[blk + j + span] = j == 0 ? d : bart_cmul(d, bart_twc(j * (16 * M / span), lgn));
    }
  }
  if (M > 1) {                                        // W_n^{lane q1}, q1 = brev(r), by recurrence
    const float2 w1 = bart_twn(t, lane, lgn);
    float2 cur = w1;
#pragma unroll
    for (int q1 = 1; q1 < M; ++q1) {
      const int r = bart_brev_c(q1, LM);
      v[r] = bart_cmul(v[r], cur);
      cur = bart_cmul(cur, w1);
    }
  }
#pragma unroll
  for (int r = 0; r < M; ++r) {                       // 32-point DIF across lanes
    float2 x = v[r];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int h = 16 >> q;
      const float2 p = make_float2(__shfl_xor_sync(0xffffffffu, x.x, h), __shfl_xor_sync(0xffffffffu, x.y, h));
      x = (lane & h) ? bart_cmul(make_float2(p.x - x.x, p.y - x.y), stw[q]) : make_float2(x.x + p.x, x.y + p.y);
    }
    v[r] = x;
  }
}

__device__ __forceinline__ void bart_stw(float2 (&stw)[5], int lane, const float2* t) {
#pragma unroll
  for (int q = 0; q < 5; ++q) {                       // W_{2h}^{lane mod h}, h = 16 >> q
    const int h = 16 >> q;
    stw[q] = bart_twn(t, (lane & (h - 1)) * (16 / h), 5);
  }
}

// natural-order position of v[r] held by lane p after bart_warp_fft
template <int M>
__device__ __forceinline__ int bart_pos(int r, int lane) {
  return bart_brev_c(r, bart_lg(M)) + M * (int)(__brev((unsigned)lane) >> 27);
}

// RW = 32 / M lines of n = 32 M points per warp, no cross-lane shuffle stages (the four-step FFT
// through a transpose): lane l holds a[j M + k] = x_j[l + 32 k] (k < M) on entry.  In-lane M-point
// DIF over k, twiddles W_n^{l q1} (q1 = brev_M(r); w1 = W_n^l), a transpose through the warp's
// [32][33] scratch xs so that lane L = j M + q1 holds a[l] = Y_j[l][q1] for l < 32, and an in-lane
// 32-point DIF over l.  On return lane L = j M + q1 holds a[r2] = X_j[q1 + M brev5(r2)].
// (X[q1 + M q2] = sum_l W_n^{l q1} W_32^{l q2} sum_k x[l + 32 k] W_M^{k q1}.)
template <int M>
__device__ __forceinline__ void bart_warp_fft_t(float2 (&a)[32], int lane, float2 w1, float2* __restrict__ xs) {
  constexpr int RW = 32 / M, LM = bart_lg(M);
#pragma unroll
  for (int j = 0; j < RW; ++j) {
    float2 (&v)[M] = *reinterpret_cast<float2 (*)[M]>(&a[j * M]);
    bart_lane_dif<M>(v, 5 + LM);
    float2 cur = w1;
#pragma unroll
    for (int q1 = 1; q1 < M; ++q1) {
      const int r = bart_brev_c(q1, LM);
      v[r] = bart_cmul(v[r], cur);
      cur = bart_cmul(cur, w1);
    }
#pragma unroll
    for (int r = 0; r < M; ++r) xs[(j * M + bart_brev_c(r, LM)) * 33 + lane] = v[r];
  }
  __syncwarp();
#pragma unroll
  for (int l = 0; l < 32; ++l) a[l] = xs[lane * 33 + l];
  __syncwarp();
  bart_lane_dif<32>(a, 10);
}

// Pass 1, D == 2: a warp takes RW = 32 / M rows (frame, segment, row) at a time: window on load,
// row FFTs (n1 = 32 M) through the transpose form (bart_warp_fft_t), stores to the scratch in
// natural order (lane (j, q1) writes elements q1 + M q2: M-element runs per row).
template <int M>
__global__ void __launch_bounds__(256) k_bart_rows(PlanDev pd, const float2* __restrict__ x, int64_t nrows, int n0,
                                                   int lgn1, const float* __restrict__ w0, const float* __restrict__ w1,
                                                   float2* __restrict__ scratch) {
  extern __shared__ __align__(16) float2 br[];
  constexpr int RW = 32 / M, n1 = 32 * M;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2* xs = br + warp * (32 * 33);
  const float2 tw1 = bart_twn(pd.btw, lane, lgn1);     // W_n1^lane
  float wc[M];
#pragma unroll
  for (int k = 0; k < M; ++k) wc[k] = w1[lane + 32 * k];
  const int L = lane / M, q1 = lane % M;               // output line / column phase of this lane
  const int64_t groups = nrows / RW;                   // nrows = batch T n0, n0 % RW == 0
  for (int64_t g = (int64_t)blockIdx.x * 8 + warp; g < groups; g += (int64_t)gridDim.x * 8) {
    const int64_t row0 = g * RW;
    const float2* src = x + (size_t)row0 * n1;
    float2 a[32];
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      const float wr = w0[(int)((row0 + j) % n0)];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const float2 v = src[(size_t)j * n1 + lane + 32 * k];
        const float w = wr * wc[k];
        a[j * M + k] = make_float2(v.x * w, v.y * w);
      }
    }
    bart_warp_fft_t<M>(a, lane, tw1, xs);
    float2* dst = scratch + (size_t)(row0 + L) * n1 + q1;
#pragma unroll
    for (int r2 = 0; r2 < 32; ++r2) dst[M * bart_brev_c(r2, 5)] = a[r2];
  }
}

// Pass 1, D == 3: one CTA per (frame, segment, dim-0 plane of n1 x n2 <= 8192): window on
// load into shared memory, dim-2 lines (warp per line), dim-1 lines (warp per column, padded
// rows), coalesced store of the plane to the scratch.
template <int M2, int M1>
__global__ void __launch_bounds__(256) k_bart_planes(PlanDev pd, const float2* __restrict__ x, int64_t nplanes,
                                                     int n0, int lgn1, int lgn2, const float* __restrict__ w0,
                                                     const float* __restrict__ w1, const float* __restrict__ w2,
                                                     float2* __restrict__ scratch) {
  extern __shared__ __align__(16) float2 bp[];
  float2* t = bp;                                      // [2048]
  float2* pl = t + 2048;                               // [n1][n2 + 1]
  constexpr int n1 = 32 * M1, n2 = 32 * M2, st = n2 + 1;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) t[i] = pd.btw[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float2 stw[5];
  bart_stw(stw, lane, t);
  for (int64_t pi = blockIdx.x; pi < nplanes; pi += gridDim.x) {
    const float2* src = x + (size_t)pi * n1 * n2;
    const float wr = w0[(int)(pi % n0)];
    __syncthreads();                                   // previous plane's readers done
    for (int e = threadIdx.x; e < n1 * n2; e += blockDim.x) {
      const int i1 = e / n2, i2 = e - i1 * n2;
      const float2 a = src[e];
      const float w = wr * w1[i1] * w2[i2];
      pl[i1 * st + i2] = make_float2(a.x * w, a.y * w);
    }
    __syncthreads();
    for (int i1 = warp; i1 < n1; i1 += nw) {           // dim 2
      float2 v[M2];
#pragma unroll
      for (int k = 0; k < M2; ++k) v[k] = pl[i1 * st + lane + 32 * k];
      bart_warp_fft<M2>(v, lane, lgn2, t, stw);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < M2; ++r) pl[i1 * st + bart_pos<M2>(r, lane)] = v[r];
    }
    __syncthreads();
    for (int i2 = warp; i2 < n2; i2 += nw) {           // dim 1
      float2 v[M1];
#pragma unroll
      for (int k = 0; k < M1; ++k) v[k] = pl[(lane + 32 * k) * st + i2];
      bart_warp_fft<M1>(v, lane, lgn1, t, stw);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < M1; ++r) pl[bart_pos<M1>(r, lane) * st + i2] = v[r];
    }
    __syncthreads();
    float2* dst = scratch + (size_t)pi * n1 * n2;
    for (int e = threadIdx.x; e < n1 * n2; e += blockDim.x) {
      const int i1 = e / n2, i2 = e - i1 * n2;
      dst[e] = pl[i1 * st + i2];
    }
  }
}

// Pass 2 (D >= 2): one CTA of CW warps per (frame, tile of C = CW RW adjacent inner columns), RW =
// 32 / M0 columns per warp; per segment the [n0][C] tile is staged in shared memory (padded rows),
// the NEXT segment's tile loads are issued before this one's FFTs (registers), each warp transforms
// its RW columns along dim 0 (bart_warp_fft_t) and accumulates |.|^2 in registers over the T
// segments; power (natural order) and the detection bits are written once.
// CW warps per CTA: 8 for 1024-point columns (c4: one CTA per SM, 3.14 vs 3.68 ms per step with
// 4), 4 below (two CTAs per SM; c2: 0.94 vs 1.02 ms with 8).
template <int M0> struct BartColCfg { static constexpr int CW = M0 == 32 ? 8 : 4; };
template <int M0, int CW = BartColCfg<M0>::CW>
__global__ void __launch_bounds__(32 * CW, 8 / CW) k_bart_cols(PlanDev pd, const float2* __restrict__ scratch,
                                                                     int64_t batch, int T, int64_t inner, int lgn0,
                                                                     float* __restrict__ power, float scale,
                                                                     float gamma, uint32_t* __restrict__ det) {
  extern __shared__ __align__(16) float2 bc[];
  constexpr int n0 = 32 * M0, RW = 32 / M0, C = RW * CW, st = C + 1;
  constexpr int NT = 32 * CW;
  constexpr int NQ = n0 * C / 2 / NT;                   // 16-B chunks per thread per segment
  float2* tile = bc;                                   // [n0][C + 1]
  float2* xs = tile + n0 * st + (threadIdx.x >> 5) * (32 * 33);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float2 tw1 = bart_twn(pd.btw, lane, lgn0);     // W_n0^lane
  const int64_t ctiles = inner / C, ntot = (int64_t)n0 * inner, words = (ntot + 31) >> 5;
  float* ptile = reinterpret_cast<float*>(tile);       // reused for the power transpose: [n0][C]
  const int L = lane / M0, q1 = lane % M0;             // output column (of the warp's RW) / phase
  for (int64_t u = blockIdx.x; u < batch * ctiles; u += gridDim.x) {
    const int64_t frame = u / ctiles;
    const int64_t c0 = (u - frame * ctiles) * C;
    float acc[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) acc[r] = 0.f;
    const float2* base = scratch + (size_t)frame * T * ntot + c0;
    float4 q[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {                      // segment 0's tile
      const int qi = threadIdx.x + NT * j, r = qi / (C / 2), c2 = (qi % (C / 2)) * 2;
      q[j] = __ldcs(reinterpret_cast<const float4*>(base + (size_t)r * inner + c2));
    }
    for (int s = 0; s < T; ++s) {
      __syncthreads();                                 // previous tile's readers done
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const int qi = threadIdx.x + NT * j, r = qi / (C / 2), c2 = (qi % (C / 2)) * 2;
        tile[r * st + c2] = make_float2(q[j].x, q[j].y);
        tile[r * st + c2 + 1] = make_float2(q[j].z, q[j].w);
      }
      __syncthreads();
      if (s + 1 < T) {                                 // next segment's loads in flight during the FFTs
        const float2* src = base + (size_t)(s + 1) * ntot;
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          const int qi = threadIdx.x + NT * j, r = qi / (C / 2), c2 = (qi % (C / 2)) * 2;
          q[j] = __ldcs(reinterpret_cast<const float4*>(src + (size_t)r * inner + c2));
        }
      }
      float2 a[32];
#pragma unroll
      for (int j = 0; j < RW; ++j)
#pragma unroll
        for (int k = 0; k < M0; ++k) a[j * M0 + k] = tile[(lane + 32 * k) * st + warp * RW + j];
      bart_warp_fft_t<M0>(a, lane, tw1, xs);
#pragma unroll
      for (int r = 0; r < 32; ++r) acc[r] += a[r].x * a[r].x + a[r].y * a[r].y;
    }
    __syncthreads();
#pragma unroll
    for (int r2 = 0; r2 < 32; ++r2) ptile[(q1 + M0 * bart_brev_c(r2, 5)) * C + warp * RW + L] = acc[r2];
    __syncthreads();
    float* pdst = power + (size_t)frame * ntot + c0;
    for (int e = threadIdx.x; e < n0 * C; e += blockDim.x) {
      const int r = e / C, c = e % C;
      const float p = ptile[e];
      pdst[(size_t)r * inner + c] = p;
      if (det && p * scale > gamma) {
        const int64_t loc = (int64_t)r * inner + c0 + c;
        atomicOr(det + (size_t)frame * words + (loc >> 5), 1u << (loc & 31));
      }
    }
  }
}

// Single pass for 1-D frames of N = R C samples, 1024 <= N <= 4096 (c1): the four-step FFT with
// warp-register FFTs.  n = C r + c; R-point DFTs down the columns (warp per column), twiddles
// W_N^{c k1}, C-point DFTs along the rows (warp per row): X[k1 + R k2].  One CTA per frame streams
// the T segments (window on load) and keeps |X|^2 in shared memory; power and detection words
// are written once (T N 8 B read, N 4 B written).  Padded rows keep the column accesses
// conflict-free.
template <int MR, int MC>
__global__ void __launch_bounds__(256) k_bart_1d(PlanDev pd, const float2* __restrict__ x, int64_t batch, int T,
                                                 const float* __restrict__ w0, float* __restrict__ power, float scale,
                                                 float gamma, uint32_t* __restrict__ det) {
  extern __shared__ __align__(16) float2 b1[];
  constexpr int R = 32 * MR, C = 32 * MC, N = R * C, st = C + 1;
  constexpr int lgR = bart_lg(R), lgC = bart_lg(C), lgN = lgR + lgC;
  float2* t = b1;                                      // [2048]
  float2* tile = t + 2048;                             // [R][C + 1]
  float* pw = reinterpret_cast<float*>(tile + R * st); // [R][C + 1]
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) t[i] = pd.btw[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float2 stw[5];
  bart_stw(stw, lane, t);
  for (int64_t frame = blockIdx.x; frame < batch; frame += gridDim.x) {
    for (int e = threadIdx.x; e < R * st; e += blockDim.x) pw[e] = 0.f;
    for (int s = 0; s < T; ++s) {
      __syncthreads();
      const float2* src = x + ((size_t)frame * T + s) * N;
      for (int n = threadIdx.x; n < N; n += blockDim.x) {
        const float2 a = src[n];
        const float w = w0[n];
        tile[(n >> lgC) * st + (n & (C - 1))] = make_float2(a.x * w, a.y * w);
      }
      __syncthreads();
      for (int c = warp; c < C; c += nw) {             // R-point DFTs down the columns
        float2 v[MR];
#pragma unroll
        for (int j = 0; j < MR; ++j) v[j] = tile[(lane + 32 * j) * st + c];
        bart_warp_fft<MR>(v, lane, lgR, t, stw);
#pragma unroll
        for (int r = 0; r < MR; ++r) {
          const int k1 = bart_pos<MR>(r, lane);
          tile[k1 * st + c] = bart_cmul(v[r], bart_twn(t, (c * k1) & (N - 1), lgN));
        }
      }
      __syncthreads();
      for (int k1 = warp; k1 < R; k1 += nw) {          // C-point DFTs along the rows
        float2 v[MC];
#pragma unroll
        for (int j = 0; j < MC; ++j) v[j] = tile[k1 * st + lane + 32 * j];
        bart_warp_fft<MC>(v, lane, lgC, t, stw);
#pragma unroll
        for (int r = 0; r < MC; ++r) pw[k1 * st + bart_pos<MC>(r, lane)] += v[r].x * v[r].x + v[r].y * v[r].y;
      }
    }
    __syncthreads();
    float* pdst = power + (size_t)frame * N;
    uint32_t* ddst = det ? det + (size_t)frame * (N >> 5) : nullptr;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {        // X[k1 + R k2] -> natural order
      const float p = pw[(k & (R - 1)) * st + (k >> lgR)];
      pdst[k] = p;
      const unsigned word = __ballot_sync(0xffffffffu, p * scale > gamma);
      if (ddst && lane == 0) ddst[k >> 5] = word;
    }
    __syncthreads();
  }
}

// Single pass for 1-D frames of N = 4096 = 64 x 64 samples (c1) with the transpose-form warp FFTs
// (no shuffle stages, bart_warp_fft_t): n = 64 r + c; warp w owns columns c = 16 w .. 16 w + 15 and,
// after the barrier, rows k1 = 16 w .. 16 w + 15.  Per segment: the warp loads its 16 columns
// straight from global memory (lane l: rows l and l + 32, 16 contiguous samples each; window on
// load), runs the 64-point DFTs down them, applies W_N^{c k1} and stores the tile [k1][c]; then
// the 64-point DFTs along its 16 rows, |X|^2 accumulated in registers over the T segments.
// X[k1 + 64 k2] = sum_c W_64^{c k2} W_N^{c k1} sum_r x[64 r + c] W_64^{r k1}.  Power and detection
// words are written once per frame (natural order through the tile).
__global__ void __launch_bounds__(128) k_bart_1d4096(PlanDev pd, const float2* __restrict__ x, int64_t batch, int T,
                                                     const float* __restrict__ w0, float* __restrict__ power,
                                                     float scale, float gamma, uint32_t* __restrict__ det) {
  extern __shared__ __align__(16) float2 b4[];
  constexpr int N = 4096, R = 64, C = 64, st = C + 1;
  float2* tile = b4;                                   // [R][C + 1]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2* xs = tile + R * st + warp * (32 * 33);
  const float2 tw1 = bart_twn(pd.btw, lane, 6);        // W_64^lane
  const int c0 = 16 * warp;
  const int L = lane >> 1, q1 = lane & 1;              // output line (of 16) / phase after the transpose
  float wcol[2][16];                                   // window of this lane's samples (registers: 4.8 M
#pragma unroll                                         // frames/s against 2.8 M with L1 loads, 3 CTAs/SM)
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int j = 0; j < 16; ++j) wcol[k][j] = w0[C * (lane + 32 * k) + c0 + j];
  for (int64_t frame = blockIdx.x; frame < batch; frame += gridDim.x) {
    float acc[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) acc[r] = 0.f;
    for (int s = 0; s < T; ++s) {
      const float2* src = x + ((size_t)frame * T + s) * N + c0;
      float2 a[32];                                    // a[j M + k] = col_j[lane + 32 k], M = 2
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float4* p4 = reinterpret_cast<const float4*>(src + C * (lane + 32 * k));
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {
          const float4 v = __ldcs(p4 + j2);
          const float wa = wcol[k][2 * j2], wb = wcol[k][2 * j2 + 1];
          a[(2 * j2) * 2 + k] = make_float2(v.x * wa, v.y * wa);
          a[(2 * j2 + 1) * 2 + k] = make_float2(v.z * wb, v.w * wb);
        }
      }
      bart_warp_fft_t<2>(a, lane, tw1, xs);            // lane (L, q1): col c0 + L, k1 = q1 + 2 brev5(r2)
      __syncthreads();                                 // previous segment's row readers done
      {
        const int c = c0 + L;
#pragma unroll
        for (int r2 = 0; r2 < 32; ++r2) {
          const int k1 = q1 + 2 * bart_brev_c(r2, 5);
          tile[k1 * st + c] = bart_cmul(a[r2], bart_twn(pd.btw, (c * k1) & (N - 1), 12));
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j)                     // rows k1 = c0 + j: a[j M + k] = row[lane + 32 k]
#pragma unroll
        for (int k = 0; k < 2; ++k) a[j * 2 + k] = tile[(c0 + j) * st + lane + 32 * k];
      bart_warp_fft_t<2>(a, lane, tw1, xs);            // lane (L, q1): k1 = c0 + L, k2 = q1 + 2 brev5(r2)
#pragma unroll
      for (int r2 = 0; r2 < 32; ++r2) acc[r2] += a[r2].x * a[r2].x + a[r2].y * a[r2].y;
    }
    __syncthreads();
    float* pt = reinterpret_cast<float*>(tile);        // power in natural order k = k1 + 64 k2
#pragma unroll
    for (int r2 = 0; r2 < 32; ++r2) pt[(c0 + L) + R * (q1 + 2 * bart_brev_c(r2, 5))] = acc[r2];
    __syncthreads();
    float* pdst = power + (size_t)frame * N;
    uint32_t* ddst = det ? det + (size_t)frame * (N >> 5) : nullptr;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      const float p = pt[k];
      pdst[k] = p;
      const unsigned word = __ballot_sync(0xffffffffu, p * scale > gamma);
      if (ddst && lane == 0) ddst[k >> 5] = word;
    }
    __syncthreads();
  }
}

rsft_status upload_bartlett_twiddles(cudaStream_t st) {
  float2 tw[2048];
  for (int k = 0; k < 2048; ++k)
    tw[k] = make_float2((float)std::cos(-2.0 * M_PI * k / 4096.0), (float)std::sin(-2.0 * M_PI * k / 4096.0));
  return cudaMemcpyToSymbolAsync(c_btw, tw, sizeof(tw), 0, cudaMemcpyHostToDevice, st) == cudaSuccess ? RSFT_OK
                                                                                                   : RSFT_E_CUDA;
}

}  // namespace rsft

using namespace rsft;

extern "C" {

rsft_status rsft_bartlett(rsft_plan_t p, const void* d_x, int64_t batch, int32_t segments, void* d_scratch,
                          float* d_power, double gamma, uint32_t* d_detect, void* stream) {
  if (!p || !d_x || !d_power || segments < 1 || batch < 1) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  for (int d = 0; d < p->D; ++d)
    if (p->n[d] > 4096) return RSFT_E_UNSUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  p->last_launches = 0;
  BartGeo g{};
  int nn[3] = {1, 1, 1};
  const float* w[3] = {p->dev.bwin[0], p->dev.bwin[1], p->dev.bwin[2]};
  const float* wr[3];
  for (int d = 0; d < 3; ++d) {                     // right-align the dims in (n0, n1, n2)
    const int dd = d - (3 - p->D);
    nn[d] = dd >= 0 ? (int)p->n[dd] : 1;
    wr[d] = dd >= 0 ? w[dd] : p->dev.bone;
  }
  // D = 1: the single dim is dim 0 (n0); right-aligned it sits in n2 -- move it to n0
  if (p->D == 1) { nn[0] = nn[2]; nn[2] = 1; wr[0] = wr[2]; wr[2] = p->dev.bone; }
  if (p->D == 2) { nn[0] = nn[1]; nn[1] = nn[2]; nn[2] = 1; wr[0] = wr[1]; wr[1] = wr[2]; wr[2] = p->dev.bone; }
  g.n0 = nn[0]; g.n1 = nn[1]; g.n2 = nn[2];
  g.lg0 = __builtin_ctz(nn[0]); g.lg1 = __builtin_ctz(nn[1]); g.lg2 = __builtin_ctz(nn[2]);
  g.w0 = wr[0]; g.w1 = wr[1]; g.w2 = wr[2];
  const int64_t ntot = p->ntot, inner = (int64_t)nn[1] * nn[2];
  const float scale = (float)(1.0 / segments), gam = (float)gamma;
  const bool single = ntot <= kBartTile;
  if (!single && (inner > kBartTile || !d_scratch)) return RSFT_E_UNSUPPORTED;
  const size_t tw_bytes = 2048 * 8;
  const char* e1 = getenv("RSFT_BART_1D_SHFL");       // 1: the shuffle-form four-step kernel for N = 4096
  if (p->D == 1 && ntot == 4096 && !(e1 && e1[0] == '1')) {   // transpose-form four-step, one pass
    const size_t smem = ((size_t)64 * 65 + 4 * 32 * 33) * 8;
    if (cudaFuncSetAttribute(k_bart_1d4096, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return RSFT_E_CUDA;
    int nb = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_bart_1d4096, 128, smem);
    const int64_t grid = std::min<int64_t>(batch, (int64_t)std::max(nb, 1) * p->num_sms);
    k_bart_1d4096<<<(unsigned)grid, 128, smem, st>>>(p->dev, reinterpret_cast<const float2*>(d_x), batch, segments,
                                                     wr[0], d_power, scale, gam, d_detect);
    p->last_launches = 1;
  } else if (p->D == 1 && ntot >= 1024 && ntot <= 4096) {   // four-step warp FFTs, one pass
    const int lg = __builtin_ctzll(ntot), lr = lg / 2, lc = lg - lr;
    void (*k)(PlanDev, const float2*, int64_t, int, const float*, float*, float, float, uint32_t*) = nullptr;
    if (lr == 5 && lc == 5) k = k_bart_1d<1, 1>;
    if (lr == 5 && lc == 6) k = k_bart_1d<1, 2>;
    if (lr == 6 && lc == 6) k = k_bart_1d<2, 2>;
    if (!k) return RSFT_E_UNSUPPORTED;
    const int R = 1 << lr, C = 1 << lc;
    const size_t smem = 2048 * 8 + (size_t)R * (C + 1) * 12;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return RSFT_E_CUDA;
    int nb = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 256, smem);
    const int64_t grid = std::min<int64_t>(batch, (int64_t)std::max(nb, 1) * p->num_sms);
    k<<<(unsigned)grid, 256, smem, st>>>(p->dev, reinterpret_cast<const float2*>(d_x), batch, segments, wr[0], d_power,
                                          scale, gam, d_detect);
    p->last_launches = 1;
  } else if (single) {
    const size_t smem = tw_bytes + (size_t)kBartTile * 8 + (size_t)ntot * 4;
    if (cudaFuncSetAttribute(k_bart_inner, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return RSFT_E_CUDA;
    int nb = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_bart_inner, kBartThreads, smem);
    const int64_t grid = std::min<int64_t>(batch, (int64_t)std::max(nb, 1) * p->num_sms);
    k_bart_inner<<<(unsigned)grid, kBartThreads, smem, st>>>(p->dev, g, reinterpret_cast<const float2*>(d_x), batch,
                                                             segments, (int)nn[0], 1, nullptr, d_power, scale, gam,
                                                             d_detect);
    p->last_launches = 1;
  } else {
    // pass 1: inner dims (D = 2: rows, warp per row; D = 3: planes, CTA per plane)
    const int64_t nlines = batch * segments * nn[0];
    const float2* xin = reinterpret_cast<const float2*>(d_x);
    float2* scr = reinterpret_cast<float2*>(d_scratch);
    auto mof = [](int n) { return n / 32; };
    if (p->D == 2) {
      const int m = mof(nn[1]);
      void (*k1)(PlanDev, const float2*, int64_t, int, int, const float*, const float*, float2*) =
          m == 1 ? k_bart_rows<1> : m == 2 ? k_bart_rows<2> : m == 4 ? k_bart_rows<4> : m == 8 ? k_bart_rows<8>
        : m == 16 ? k_bart_rows<16> : m == 32 ? k_bart_rows<32> : nullptr;
      if (!k1) return RSFT_E_UNSUPPORTED;
      if (nn[0] % (32 / m)) return RSFT_E_UNSUPPORTED;   // whole row groups per warp
      const size_t smem = (size_t)8 * 32 * 33 * 8;     // per-warp transpose scratch
      if (cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return RSFT_E_CUDA;
      const int64_t grid = std::min<int64_t>((nlines / (32 / m) + 7) / 8, 6 * (int64_t)p->num_sms);
      k1<<<(unsigned)grid, 256, smem, st>>>(p->dev, xin, nlines, nn[0], g.lg1, wr[0], wr[1], scr);
    } else {
      const int m2 = mof(nn[2]), m1 = mof(nn[1]);
      void (*k1)(PlanDev, const float2*, int64_t, int, int, int, const float*, const float*, const float*, float2*) = nullptr;
#define RSFT_BP(A, B_) if (m2 == A && m1 == B_) k1 = k_bart_planes<A, B_>;
      RSFT_BP(1, 1) RSFT_BP(1, 2) RSFT_BP(1, 4) RSFT_BP(1, 8) RSFT_BP(2, 1) RSFT_BP(2, 2) RSFT_BP(2, 4)
      RSFT_BP(4, 1) RSFT_BP(4, 2) RSFT_BP(8, 1)
#undef RSFT_BP
      if (!k1) return RSFT_E_UNSUPPORTED;
      const size_t smem = (2048 + (size_t)nn[1] * (nn[2] + 1)) * 8;
      if (cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return RSFT_E_CUDA;
      const int64_t grid = std::min<int64_t>(nlines, 4 * (int64_t)p->num_sms);
      k1<<<(unsigned)grid, 256, smem, st>>>(p->dev, xin, nlines, nn[0], g.lg1, g.lg2, wr[0], wr[1], wr[2], scr);
    }
    if (d_detect && cudaMemsetAsync(d_detect, 0, (size_t)batch * ((ntot + 31) / 32) * 4, st) != cudaSuccess)
      return RSFT_E_CUDA;
    // pass 2: dim 0 + |.|^2 over the segments + detection
    const int m0 = mof(nn[0]);
    void (*k2)(PlanDev, const float2*, int64_t, int, int64_t, int, float*, float, float, uint32_t*) =
        m0 == 1 ? k_bart_cols<1> : m0 == 2 ? k_bart_cols<2> : m0 == 4 ? k_bart_cols<4> : m0 == 8 ? k_bart_cols<8>
      : m0 == 16 ? k_bart_cols<16> : m0 == 32 ? k_bart_cols<32> : nullptr;
    const int cw = m0 == 32 ? BartColCfg<32>::CW : BartColCfg<1>::CW;
    const int64_t ccols = (int64_t)cw * (32 / std::max(m0, 1));   // columns per CTA
    if (!k2 || inner % ccols) return RSFT_E_UNSUPPORTED;
    const size_t smem2 = ((size_t)nn[0] * (ccols + 1) + (size_t)cw * 32 * 33) * 8;
    if (cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2) != cudaSuccess)
      return RSFT_E_CUDA;
    int nb = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k2, 32 * cw, smem2);
    const int64_t units2 = batch * (inner / ccols);
    const int64_t grid2 = std::min<int64_t>(units2, (int64_t)std::max(nb, 1) * p->num_sms);
    k2<<<(unsigned)grid2, 32 * cw, smem2, st>>>(p->dev, scr, batch, segments, inner, g.lg0, d_power, scale, gam, d_detect);
    p->last_launches = 2;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { set_error(std::string("bartlett: ") + cudaGetErrorString(e)); return RSFT_E_CUDA; }
  return RSFT_OK;
}

// gamma of Eq. bartlettROC for a target per-bin P_fa: under H'0 the statistic l is
// N(sigma_n^2 beta', sigma_n^4 beta'^2 / T) with beta' = ||w||^2 (the compound window).
rsft_status rsft_bartlett_threshold(rsft_plan_t p, int32_t segments, double p_fa, double* gamma) {
  if (!p || !gamma || segments < 1 || !(p_fa > 0.0 && p_fa < 1.0)) return RSFT_E_ARG;
  double beta = 1.0;
  for (int d = 0; d < p->D; ++d) {
    double s = 0.0;
    for (double v : p->prewin[d]) s += v * v;
    beta *= s;
  }
  // Phi^{-1}(1 - p_fa) by bisection on the Normal tail
  double lo = -40.0, hi = 40.0;
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (0.5 * std::erfc(mid / std::sqrt(2.0)) > p_fa) lo = mid; else hi = mid;
  }
  const double z = 0.5 * (lo + hi);
  *gamma = p->P.noise_var * beta * (1.0 + z / std::sqrt((double)segments));
  return RSFT_OK;
}

}  // extern "C"
