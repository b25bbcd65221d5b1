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

// Pass 2 (D >= 2): dim-0 FFT of C adjacent inner columns for every segment, |.|^2 summed over
// the T segments in registers, then power + detection bits (atomicOr: a word spans 32 / C tiles).
template <int PT>
__global__ void __launch_bounds__(kBartThreads) k_bart_outer(PlanDev pd, BartGeo g, const float2* __restrict__ scratch,
                                                             int64_t batch, int T, int C, float* __restrict__ power,
                                                             float scale, float gamma, uint32_t* __restrict__ det) {
  extern __shared__ __align__(16) float2 bsm[];
  float2* tw = bsm;
  float2* sv = tw + 2048;                            // [n0][C]
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) tw[i] = pd.btw[i];
  const int inner = g.n1 * g.n2, lgc = __ffs(C) - 1;
  const int elems = g.n0 * C;
  const int64_t ntot = (int64_t)g.n0 * inner;
  const int64_t ctiles = inner / C;
  const int64_t units = batch * ctiles;
  const int64_t words = (ntot + 31) >> 5;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t frame = u / ctiles;
    const int c0 = (int)(u % ctiles) * C;
    float acc[PT];
#pragma unroll
    for (int k = 0; k < PT; ++k) acc[k] = 0.f;
    for (int s = 0; s < T; ++s) {
      __syncthreads();
      const float2* src = scratch + ((size_t)frame * T + s) * ntot + c0;
      for (int e = threadIdx.x; e < elems; e += blockDim.x) {
        const int r = e >> lgc, c = e & (C - 1);
        sv[(bart_brev(r, g.lg0) << lgc) + c] = src[(size_t)r * inner + c];
      }
      __syncthreads();
      bart_fft_axis(sv, g.lg0, C, C, lgc, 0, 1, tw);
#pragma unroll
      for (int k = 0; k < PT; ++k) {
        const int e = threadIdx.x + k * blockDim.x;
        if (e < elems) { const float2 v = sv[e]; acc[k] += v.x * v.x + v.y * v.y; }
      }
    }
    float* pdst = power + (size_t)frame * ntot + c0;
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int e = threadIdx.x + k * blockDim.x;
      if (e < elems) {
        const int r = e >> lgc, c = e & (C - 1);
        pdst[(size_t)r * inner + c] = acc[k];
        if (det && acc[k] * scale > gamma) {
          const int64_t loc = (int64_t)r * inner + c0 + c;
          atomicOr(det + (size_t)frame * words + (loc >> 5), 1u << (loc & 31));
        }
      }
    }
  }
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
  if (single) {
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
    const int rows = (int)std::min<int64_t>(nn[0], kBartTile / inner);
    const size_t smem1 = tw_bytes + (size_t)kBartTile * 8;
    if (cudaFuncSetAttribute(k_bart_inner, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1) != cudaSuccess)
      return RSFT_E_CUDA;
    int nb = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_bart_inner, kBartThreads, smem1);
    const int64_t units1 = batch * segments * (nn[0] / rows);
    const int64_t grid1 = std::min<int64_t>(units1, (int64_t)std::max(nb, 1) * p->num_sms);
    k_bart_inner<<<(unsigned)grid1, kBartThreads, smem1, st>>>(p->dev, g, reinterpret_cast<const float2*>(d_x), batch,
                                                               segments, rows, 0, reinterpret_cast<float2*>(d_scratch),
                                                               nullptr, scale, gam, nullptr);
    if (d_detect && cudaMemsetAsync(d_detect, 0, (size_t)batch * ((ntot + 31) / 32) * 4, st) != cudaSuccess)
      return RSFT_E_CUDA;
    const int C = (int)std::min<int64_t>(inner, kBartTile / nn[0]);
    const int pt = (nn[0] * C + kBartThreads - 1) / kBartThreads;
    auto kern = pt <= 4 ? k_bart_outer<4> : pt <= 8 ? k_bart_outer<8> : k_bart_outer<16>;
    if (pt > 16) return RSFT_E_UNSUPPORTED;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1) != cudaSuccess)
      return RSFT_E_CUDA;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kBartThreads, smem1);
    const int64_t units2 = batch * (inner / C);
    const int64_t grid2 = std::min<int64_t>(units2, (int64_t)std::max(nb, 1) * p->num_sms);
    kern<<<(unsigned)grid2, kBartThreads, smem1, st>>>(p->dev, g, reinterpret_cast<const float2*>(d_scratch), batch,
                                                       segments, C, d_power, scale, gam, d_detect);
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
