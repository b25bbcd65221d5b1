// Microbenchmark: compute throughput of the fold inner loop (rows of 32 float4 in shared
// memory, per-row broadcast weights [row][LP] in shared memory, LP complex x real FFMA2
// accumulators per lane), with no global memory traffic.  Reports FFMA2/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mac(float2& acc, float w, float vx, float vy) {
  asm("{\n\t.reg .b64 a, ww, v;\n\tmov.b64 a, {%0,%1};\n\tmov.b64 ww, {%2,%2};\n\t"
      "mov.b64 v, {%3,%4};\n\tfma.rn.f32x2 a, ww, v, a;\n\tmov.b64 {%0,%1}, a;\n\t}"
      : "+f"(acc.x), "+f"(acc.y) : "f"(w), "f"(vx), "f"(vy));
}

template <int LP, int U, int MODE>
__global__ void fold(float* out, int iters) {
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
    const float* wb = wt + (it & 7) * U * LP;
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = buf[((it & 1) * 0 + u) * 32 + lane];
    asm volatile("" ::: "memory");
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4* wr = reinterpret_cast<const float4*>(wb + u * LP);
#pragma unroll
      for (int l4 = 0; l4 < LP / 4; ++l4) {
        float4 w = wr[l4];
        if (MODE == 0) {
          mac(acc[4 * l4][0], w.x, v[u].x, v[u].y); mac(acc[4 * l4][1], w.x, v[u].z, v[u].w);
          mac(acc[4 * l4 + 1][0], w.y, v[u].x, v[u].y); mac(acc[4 * l4 + 1][1], w.y, v[u].z, v[u].w);
          mac(acc[4 * l4 + 2][0], w.z, v[u].x, v[u].y); mac(acc[4 * l4 + 2][1], w.z, v[u].z, v[u].w);
          mac(acc[4 * l4 + 3][0], w.w, v[u].x, v[u].y); mac(acc[4 * l4 + 3][1], w.w, v[u].z, v[u].w);
        } else if (MODE == 2) {   // __ffma2_rn builtin
          const float2 a = make_float2(v[u].x, v[u].y), b = make_float2(v[u].z, v[u].w);
          acc[4*l4][0] = __ffma2_rn(make_float2(w.x, w.x), a, acc[4*l4][0]); acc[4*l4][1] = __ffma2_rn(make_float2(w.x, w.x), b, acc[4*l4][1]);
          acc[4*l4+1][0] = __ffma2_rn(make_float2(w.y, w.y), a, acc[4*l4+1][0]); acc[4*l4+1][1] = __ffma2_rn(make_float2(w.y, w.y), b, acc[4*l4+1][1]);
          acc[4*l4+2][0] = __ffma2_rn(make_float2(w.z, w.z), a, acc[4*l4+2][0]); acc[4*l4+2][1] = __ffma2_rn(make_float2(w.z, w.z), b, acc[4*l4+2][1]);
          acc[4*l4+3][0] = __ffma2_rn(make_float2(w.w, w.w), a, acc[4*l4+3][0]); acc[4*l4+3][1] = __ffma2_rn(make_float2(w.w, w.w), b, acc[4*l4+3][1]);
        } else {   // scalar FFMA
          acc[4*l4][0].x = fmaf(w.x, v[u].x, acc[4*l4][0].x); acc[4*l4][0].y = fmaf(w.x, v[u].y, acc[4*l4][0].y);
          acc[4*l4][1].x = fmaf(w.x, v[u].z, acc[4*l4][1].x); acc[4*l4][1].y = fmaf(w.x, v[u].w, acc[4*l4][1].y);
          acc[4*l4+1][0].x = fmaf(w.y, v[u].x, acc[4*l4+1][0].x); acc[4*l4+1][0].y = fmaf(w.y, v[u].y, acc[4*l4+1][0].y);
          acc[4*l4+1][1].x = fmaf(w.y, v[u].z, acc[4*l4+1][1].x); acc[4*l4+1][1].y = fmaf(w.y, v[u].w, acc[4*l4+1][1].y);
          acc[4*l4+2][0].x = fmaf(w.z, v[u].x, acc[4*l4+2][0].x); acc[4*l4+2][0].y = fmaf(w.z, v[u].y, acc[4*l4+2][0].y);
          acc[4*l4+2][1].x = fmaf(w.z, v[u].z, acc[4*l4+2][1].x); acc[4*l4+2][1].y = fmaf(w.z, v[u].w, acc[4*l4+2][1].y);
          acc[4*l4+3][0].x = fmaf(w.w, v[u].x, acc[4*l4+3][0].x); acc[4*l4+3][0].y = fmaf(w.w, v[u].y, acc[4*l4+3][0].y);
          acc[4*l4+3][1].x = fmaf(w.w, v[u].z, acc[4*l4+3][1].x); acc[4*l4+3][1].y = fmaf(w.w, v[u].w, acc[4*l4+3][1].y);
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
void run(int sms, float* out, int warps, int ctas) {
  const int iters = 2048;
  size_t smem = (size_t)warps * (U * 32 + 64 * LP / 4) * 16;
  cudaFuncSetAttribute(fold<LP, U, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fold<LP, U, MODE><<<sms * ctas, warps * 32, smem>>>(out, iters);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  fold<LP, U, MODE><<<sms * ctas, warps * 32, smem>>>(out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float cyc; cudaMemcpy(&cyc, out + 1, 4, cudaMemcpyDeviceToHost);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ffma2 = (double)warps * ctas * iters * U * LP * 2;   // per SM
  printf("LP=%2d U=%d %s warps/CTA=%2d ctas/SM=%d: %.3f FFMA2/clk/SM (clock64)  %.1f us  %s\n", LP, U, MODE == 1 ? "FFMA " : (MODE == 2 ? "ffma2_rn" : "FFMA2asm"),
         warps, ctas, ffma2 / cyc, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  float* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 12}) run<16, 8, 0>(sms, out, w, 1);
  for (int w : {4, 8, 12}) run<16, 8, 2>(sms, out, w, 1);
  for (int w : {4, 8, 12}) run<16, 8, 1>(sms, out, w, 1);
  for (int w : {8, 16}) run<16, 4, 2>(sms, out, w, 1);
  return 0;
}
