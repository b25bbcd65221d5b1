// Scene generator for Monte Carlo runs of the RSFT (harness utility, not the method): frames of
// T segments following the paper's signal model, Eq. sig_model / sinusoid, made
// separable over dimensions (§III-C):
//   x[f][s][n] = sum_k b_{f,k,s} prod_d exp(j 2 pi w_{f,k,d} n_d / N_d) + nu[f][s][n],
//   b_{f,k,s} ~ CN(0, sigma_{f,k}^2) drawn per segment (Swerling-like),
//   nu ~ CN(0, sigma_n^2) i.i.d.
// Random numbers come from a counter-based generator, SplitMix64 of (seed, stream, counter),
// turned into N(0, 1/2) pairs by Box-Muller; synth.counter_normals re-implements the same
// generator in NumPy (tests compare them).
#include <cuda_runtime.h>

#include <cmath>

#include "rsft_internal.h"

namespace rsft {

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// CN(0, 1) sample for (seed, stream, counter): u1, u2 from the two 32-bit halves of
// SplitMix64(seed ^ stream * C + counter), u1 in (0, 1]; Box-Muller with variance 1/2 per part.
__device__ __forceinline__ float2 cnormal(unsigned long long seed, unsigned long long stream,
                                          unsigned long long ctr) {
  const unsigned long long r = splitmix64(seed ^ (stream * 0xD1B54A32D192ED03ull) ^ splitmix64(ctr));
  const double u1 = ((double)(r >> 32) + 1.0) * (1.0 / 4294967296.0);
  const double u2 = (double)(r & 0xffffffffull) * (1.0 / 4294967296.0);
  const double rad = sqrt(-log(u1));              // |z|^2 ~ Exp(1): E|z|^2 = 1
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  return make_float2((float)(rad * cs), (float)(rad * sn));
}

__global__ void k_synth(float2* __restrict__ x, int64_t batch, int T, int D, int n0, int n1, int n2, int K,
                        const double* __restrict__ omega /* [batch][K][D] bins */,
                        const double* __restrict__ sigma_b /* [batch][K] */, double sigma_n,
                        unsigned long long seed) {
  const int64_t ntot = (int64_t)n0 * n1 * n2;
  const int64_t total = batch * T * ntot;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fs = i / ntot, n = i - fs * ntot;
    const int64_t f = fs / T;
    const int s = (int)(fs - f * T);
    const int i2 = (int)(n % n2), i1 = (int)((n / n2) % n1), i0 = (int)(n / ((int64_t)n1 * n2));
    const int idx[3] = {i0, i1, i2};
    const int nn[3] = {n0, n1, n2};
    double re = 0.0, im = 0.0;
    for (int k = 0; k < K; ++k) {
      const float2 b = cnormal(seed, 1, ((unsigned long long)f * K + k) * T + s);   // b_{f,k,s} / sigma
      double ph = 0.0;                             // phase / pi
      for (int d = 0; d < D; ++d) {
        const int dd = 3 - D + d;                  // dims are right-aligned in (n0, n1, n2)
        const double w = omega[((size_t)f * K + k) * D + d];
        const long long m = (long long)idx[dd];
        ph += 2.0 * fmod(w * (double)m, (double)nn[dd]) / (double)nn[dd];
      }
      double sn, cs;
      sincospi(ph, &sn, &cs);
      const double sb = sigma_b[(size_t)f * K + k];
      re += sb * (b.x * cs - b.y * sn);
      im += sb * (b.x * sn + b.y * cs);
    }
    const float2 v = cnormal(seed, 2, (unsigned long long)i);
    x[i] = make_float2((float)(re + sigma_n * v.x), (float)(im + sigma_n * v.y));
  }
}

}  // namespace rsft

extern "C" rsft_status rsft_synthesize(const int64_t* n, int32_t ndim, int64_t batch, int32_t segments, int32_t K,
                                       const double* d_omega, const double* d_sigma_b, double sigma_n,
                                       uint64_t seed, void* d_x, void* stream) {
  if (!n || ndim < 1 || ndim > 3 || batch < 0 || segments < 1 || K < 0 || !d_x || sigma_n < 0.0) return RSFT_E_ARG;
  if (K > 0 && (!d_omega || !d_sigma_b)) return RSFT_E_ARG;
  int nn[3] = {1, 1, 1};
  for (int d = 0; d < ndim; ++d) {
    if (n[d] < 1) return RSFT_E_ARG;
    nn[3 - ndim + d] = (int)n[d];
  }
  if (batch == 0) return RSFT_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  rsft::k_synth<<<1184, 256, 0, st>>>(reinterpret_cast<float2*>(d_x), batch, segments, ndim, nn[0], nn[1], nn[2], K,
                                      d_omega, d_sigma_b, sigma_n, seed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { rsft::set_error(std::string("k_synth launch: ") + cudaGetErrorString(e)); return RSFT_E_CUDA; }
  return RSFT_OK;
}
