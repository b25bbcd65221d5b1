// Microbenchmark: issue rate of packed fma.rn.f32x2 (SASS FFMA2) on sm_100a in the form the
// fold kernels use (scalar weight broadcast to both halves, R.F32 x R.F32x2 + R.F32x2),
// versus plain FFMA, for 1..16 warps per SM.  Reports FFMA2 per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int FORM>
__global__ void rate(float* out, int iters, float w0) {
  float2 acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  float w = w0 + threadIdx.x * 1e-7f;
  float2 v = make_float2(1.0001f, 0.9999f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (FORM == 0) {   // FFMA2 R, R.F32, R.F32x2, R.F32x2
        asm volatile("{\n\t.reg .b64 a, ww, x;\n\tmov.b64 a, {%0,%1};\n\tmov.b64 ww, {%2,%2};\n\tmov.b64 x, {%3,%4};\n\t"
                     "fma.rn.f32x2 a, ww, x, a;\n\tmov.b64 {%0,%1}, a;\n\t}"
                     : "+f"(acc[i].x), "+f"(acc[i].y) : "f"(w), "f"(v.x), "f"(v.y));
      } else {           // two scalar FFMA
        asm volatile("fma.rn.f32 %0, %2, %3, %0;\n\tfma.rn.f32 %1, %2, %4, %1;" : "+f"(acc[i].x), "+f"(acc[i].y) : "f"(w), "f"(v.x), "f"(v.y));
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += acc[i].x + acc[i].y;
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
}

int main() {
  float* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int form = 0; form < 2; ++form)
    for (int warps : {1, 2, 4, 8, 12, 16, 32}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      if (form == 0) rate<0><<<sms, warps * 32>>>(out, iters, 0.5f); else rate<1><<<sms, warps * 32>>>(out, iters, 0.5f);
      cudaEventRecord(a);
      if (form == 0) rate<0><<<sms, warps * 32>>>(out, iters, 0.5f); else rate<1><<<sms, warps * 32>>>(out, iters, 0.5f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float cyc; cudaMemcpy(&cyc, out + 1, 4, cudaMemcpyDeviceToHost);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double pairs = (double)warps * iters * 16;       // complex x real MACs per SM (warp-level)
      printf("%s warps/SM %2d: %.3f warp-MAC-pairs/clk/SM (clock64), %.2f TFLOP/s\n", form ? "2xFFMA" : "FFMA2 ",
             warps, pairs / cyc, 4.0 * 32 * pairs * sms / (ms / 1e3) / 1e12);
    }
  return 0;
}
