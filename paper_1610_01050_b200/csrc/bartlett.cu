// Bartlett baseline: Algorithm 2 of the paper's Appendix A
// (P:926-943): for every segment s, u = W r_s (the plan's separable pre-window), u_hat =
// N-D FFT(u) (forward, unnormalised), x += |u_hat|^2; then l = x / T > gamma (NP test,
// Eq. bartlettROC).  The dense comparison workload for the RSFT's complexity claim
// (Tables I-II).  Hand-written FFTs (no cuFFT): one kernel per axis, each CTA
// transforms C adjacent lines of that axis in shared memory (radix-2 DIT, stage-parallel);
// the first pass applies the window, the last pass accumulates |.|^2.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "rsft_internal.h"

namespace rsft {

constexpr int kBartTile = 8192;            // complex elements per CTA tile (64 KiB smem)

__global__ void __launch_bounds__(256) k_bart_axis(const float2* __restrict__ in, int64_t in_stride,
                                                   float2* __restrict__ out,
                                                   float* __restrict__ power, int D, int n0, int n1, int n2,
                                                   int axis, int window, int last,
                                                   const float* __restrict__ w0, const float* __restrict__ w1,
                                                   const float* __restrict__ w2, const float2* __restrict__ tw) {
  extern __shared__ float2 sv[];
  const int nn[3] = {n0, n1, n2};
  const int na = nn[axis];
  int64_t inner = 1;
  for (int d = axis + 1; d < 3; ++d) inner *= nn[d];
  const int lg = __ffs(na) - 1;
  const int C = (int)(inner < (int64_t)(kBartTile / na) ? inner : (int64_t)(kBartTile / na));
  const int64_t iblocks = inner / C;
  const int64_t o = blockIdx.x / iblocks, ib = blockIdx.x - o * iblocks;
  const int64_t fr = blockIdx.y;                   // frame of the batch
  const int64_t ntot = (int64_t)n0 * n1 * n2;
  in += fr * in_stride;
  out += fr * ntot;
  power += fr * ntot;
  const int64_t base = o * na * inner + ib * C;
  const int tid = threadIdx.x;
  // load C lines (coalesced along the C adjacent inner indices), window, bit-reversed
  for (int e = tid; e < na * C; e += blockDim.x) {
    const int p = e / C, c = e - p * C;
    const int64_t idx = base + (int64_t)p * inner + c;
    float2 v = in[idx];
    if (window) {
      const int i2 = (int)(idx % n2), i1 = (int)((idx / n2) % n1), i0 = (int)(idx / ((int64_t)n1 * n2));
      const float w = w0[i0] * w1[i1] * w2[i2];
      v.x *= w; v.y *= w;
    }
    sv[c * na + (int)(__brev((unsigned)p) >> (32 - lg))] = v;
  }
  __syncthreads();
  const int tstep = 4096 / na;                    // tw[k] = e^{-j 2 pi k / 4096}
  for (int s = 1; s <= lg; ++s) {
    const int half = 1 << (s - 1);
    for (int bf = tid; bf < (na >> 1) * C; bf += blockDim.x) {
      const int c = bf >> (lg - 1), r = bf & ((na >> 1) - 1);
      const int j = r & (half - 1), g = r >> (s - 1);
      float2* e0 = sv + c * na + (g << s) + j;
      float2* e1 = e0 + half;
      const float2 t = tw[(j << (lg - s)) * tstep];
      const float2 b = *e1;
      const float2 tb = make_float2(t.x * b.x - t.y * b.y, t.x * b.y + t.y * b.x);
      const float2 a = *e0;
      *e0 = make_float2(a.x + tb.x, a.y + tb.y);
      *e1 = make_float2(a.x - tb.x, a.y - tb.y);
    }
    __syncthreads();
  }
  for (int e = tid; e < na * C; e += blockDim.x) {
    const int p = e / C, c = e - p * C;
    const int64_t idx = base + (int64_t)p * inner + c;
    const float2 v = sv[c * na + p];
    if (last) power[idx] += v.x * v.x + v.y * v.y;
    else out[idx] = v;
  }
}

// l = x / T > gamma -> detection bitmap words (one ballot per 32 locations)
__global__ void k_bart_detect(const float* __restrict__ power, int64_t ntot, int64_t batch, float scale, float gamma,
                              uint32_t* __restrict__ det) {
  const int64_t per = (ntot + 31) & ~int64_t(31), words = per >> 5;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < batch * per;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i / per, k = i - f * per;
    const bool bit = k < ntot && power[f * ntot + k] * scale > gamma;
    const unsigned word = __ballot_sync(0xffffffffu, bit);
    if ((threadIdx.x & 31) == 0) det[f * words + (k >> 5)] = word;
  }
}

}  // namespace rsft

using namespace rsft;

extern "C" {

rsft_status rsft_bartlett(rsft_plan_t p, const void* d_x, int64_t batch, int32_t segments, void* d_scratch,
                          float* d_power, double gamma, uint32_t* d_detect, void* stream) {
  if (!p || !d_x || !d_scratch || !d_power || segments < 1 || batch < 1) return RSFT_E_ARG;
  if (!p->bound) return RSFT_E_STATE;
  for (int d = 0; d < p->D; ++d)
    if (p->n[d] > 4096) return RSFT_E_UNSUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  p->last_launches = 0;
  int nn[3] = {1, 1, 1};
  const float* w[3] = {p->dev.bwin[0], p->dev.bwin[1], p->dev.bwin[2]};
  const float* wr[3];
  for (int d = 0; d < 3; ++d) {                   // right-align the dims in (n0, n1, n2)
    const int dd = d - (3 - p->D);
    nn[d] = dd >= 0 ? (int)p->n[dd] : 1;
    wr[d] = dd >= 0 ? w[dd] : p->dev.bone;
  }
  const int64_t ntot = p->ntot;
  if (cudaMemsetAsync(d_power, 0, (size_t)batch * ntot * 4, st) != cudaSuccess) return RSFT_E_CUDA;
  cudaFuncSetAttribute(k_bart_axis, cudaFuncAttributeMaxDynamicSharedMemorySize, kBartTile * 8);
  for (int s = 0; s < segments; ++s) {
    const float2* src = reinterpret_cast<const float2*>(d_x) + (size_t)s * ntot;   // frame f: + f T N_tot
    bool first = true;
    for (int axis = 2; axis >= 3 - p->D; --axis) { // last dim first (contiguous), then outer dims
      const bool last = axis == 3 - p->D;
      int64_t inner = 1;
      for (int d = axis + 1; d < 3; ++d) inner *= nn[d];
      const int64_t C = std::min<int64_t>(inner, kBartTile / nn[axis]);
      const int64_t tiles = ntot / ((int64_t)nn[axis] * C);
      const size_t smem = (size_t)nn[axis] * C * 8;
      dim3 grid((unsigned)tiles, (unsigned)batch);
      k_bart_axis<<<grid, 256, smem, st>>>(first ? src : reinterpret_cast<const float2*>(d_scratch),
                                           first ? (int64_t)segments * ntot : ntot,
                                           reinterpret_cast<float2*>(d_scratch), d_power, 0, nn[0], nn[1], nn[2],
                                           axis, first ? 1 : 0, last ? 1 : 0, wr[0], wr[1], wr[2], p->dev.btw);
      p->last_launches += 1;
      first = false;
    }
  }
  if (d_detect) {
    k_bart_detect<<<1184, 256, 0, st>>>(d_power, ntot, batch, (float)(1.0 / segments), (float)gamma, d_detect);
    p->last_launches += 1;
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
