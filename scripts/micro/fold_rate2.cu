// Microbenchmark: fold inner loop variants in shared memory (no global traffic), 8 warps/SM.
//  mode 0: single accumulator set, per-row weights [row][LP] (as the plain fold)
//  mode 1: two-level: inn += h1[row] x over 2 boxes of U rows, then acc += h0 * inn
//  mode 2: mode 1 with explicit weight/data prefetch one row ahead
#include <cstdio>
#include <cuda_runtime.h>

template <int LP, int U, int MODE>
__global__ void __launch_bounds__(256, 1) fold(float* out, int iters) {
  extern __shared__ float4 sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* buf = sm + warp * (U * 32 + 64 * LP / 4);
  float* wt = reinterpret_cast<float*>(buf + U * 32);
  for (int i = lane; i < U * 32; i += 32) buf[i] = make_float4(lane * 1e-3f, 1.f, 0.5f, 0.25f);
  for (int i = lane; i < 64 * LP; i += 32) wt[i] = 1e-3f * i;
  __syncwarp();
  float2 acc[LP][2];
  for (int l = 0; l < LP; ++l) acc[l][0] = acc[l][1] = make_float2(0.f, 0.f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float2 inn[LP][2];
    if (MODE >= 1)
      for (int l = 0; l < LP; ++l) inn[l][0] = inn[l][1] = make_float2(0.f, 0.f);
    for (int box = 0; box < 2; ++box) {
      const float* wb = wt + ((it * 2 + box) & 7) * U * LP;
      asm volatile("" ::: "memory");
      if (MODE == 2) {
        float4 v = buf[lane];
        float4 w[LP / 4];
#pragma unroll
        for (int l4 = 0; l4 < LP / 4; ++l4) w[l4] = reinterpret_cast<const float4*>(wb)[l4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float4 vn = v, wn[LP / 4];
          if (u + 1 < U) {
            vn = buf[(u + 1) * 32 + lane];
#pragma unroll
            for (int l4 = 0; l4 < LP / 4; ++l4) wn[l4] = reinterpret_cast<const float4*>(wb + (u + 1) * LP)[l4];
          }
#pragma unroll
          for (int l4 = 0; l4 < LP / 4; ++l4) {
            const float wv[4] = {w[l4].x, w[l4].y, w[l4].z, w[l4].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              inn[4 * l4 + i][0] = __ffma2_rn(make_float2(wv[i], wv[i]), make_float2(v.x, v.y), inn[4 * l4 + i][0]);
              inn[4 * l4 + i][1] = __ffma2_rn(make_float2(wv[i], wv[i]), make_float2(v.z, v.w), inn[4 * l4 + i][1]);
            }
          }
          if (u + 1 < U) {
            v = vn;
#pragma unroll
            for (int l4 = 0; l4 < LP / 4; ++l4) w[l4] = wn[l4];
          }
        }
      } else {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = buf[u * 32 + lane];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float4* wr = reinterpret_cast<const float4*>(wb + u * LP);
#pragma unroll
          for (int l4 = 0; l4 < LP / 4; ++l4) {
            float4 w = wr[l4];
            const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float2 (&tgt)[LP][2] = MODE == 0 ? acc : inn;
              tgt[4 * l4 + i][0] = __ffma2_rn(make_float2(wv[i], wv[i]), make_float2(v[u].x, v[u].y), tgt[4 * l4 + i][0]);
              tgt[4 * l4 + i][1] = __ffma2_rn(make_float2(wv[i], wv[i]), make_float2(v[u].z, v[u].w), tgt[4 * l4 + i][1]);
            }
          }
        }
      }
    }
    if (MODE >= 1) {
      const float2* h0 = reinterpret_cast<const float2*>(wt + (it & 31) * LP);
#pragma unroll
      for (int l2 = 0; l2 < LP / 2; ++l2) {
        const float2 w = h0[l2];
        for (int e = 0; e < 2; ++e) {
          acc[2 * l2][e] = __ffma2_rn(make_float2(w.x, w.x), inn[2 * l2][e], acc[2 * l2][e]);
          acc[2 * l2 + 1][e] = __ffma2_rn(make_float2(w.y, w.y), inn[2 * l2 + 1][e], acc[2 * l2 + 1][e]);
        }
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int l = 0; l < LP; ++l) s += acc[l][0].x + acc[l][0].y + acc[l][1].x + acc[l][1].y;
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
}

template <int LP, int U, int MODE>
void run(int sms, float* out, int warps) {
  const int iters = 1024;
  size_t smem = (size_t)warps * (U * 32 + 64 * LP / 4) * 16;
  cudaFuncSetAttribute(fold<LP, U, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fold<LP, U, MODE><<<sms, warps * 32, smem>>>(out, iters);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  fold<LP, U, MODE><<<sms, warps * 32, smem>>>(out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float cyc; cudaMemcpy(&cyc, out + 1, 4, cudaMemcpyDeviceToHost);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ffma2 = (double)warps * iters * (2 * U * LP * 2 + (MODE ? LP * 2 : 0));
  printf("LP=%2d U=%d mode %d warps=%2d: %.3f FFMA2/clk/SM  %.1f us %s\n", LP, U, MODE, warps, ffma2 / cyc, ms * 1e3,
         cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  float* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8}) run<16, 8, 0>(sms, out, w);
  for (int w : {4, 8}) run<16, 8, 1>(sms, out, w);
  for (int w : {4, 8}) run<16, 8, 2>(sms, out, w);
  for (int w : {4, 8}) run<16, 4, 1>(sms, out, w);
  return 0;
}
