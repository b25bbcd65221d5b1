// Microbenchmark: HBM streaming read throughput on B200 with (a) LDG.128 (b) per-warp
// cp.async.bulk rings of various copy sizes.  Reads a large buffer, reduces to one value.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_sum(const float4* __restrict__ x, size_t n4, float* out) {
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(x + i); s += v.x + v.y + v.z + v.w;
  }
  if (s == 123.f) out[0] = s;
}

template <int STAGES>
__global__ void tma_sum(const char* __restrict__ x, size_t bytes, int chunk, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned char* ring = sm + (size_t)warp * STAGES * chunk;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)nw * STAGES * chunk) + warp * STAGES;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const size_t nchunks = bytes / chunk;
  const size_t gw = (size_t)gridDim.x * nw, wid = (size_t)blockIdx.x * nw + warp;
  const size_t mine = wid < nchunks ? (nchunks - 1 - wid) / gw + 1 : 0;
  auto issue = [&](size_t q) {
    int s = q % STAGES;
    const char* src = x + (wid + q * gw) * chunk;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bars + s)), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(su32(ring + (size_t)s * chunk)), "l"(src), "r"(chunk), "r"(su32(bars + s)) : "memory");
  };
  if (lane == 0) for (size_t q = 0; q < STAGES - 1 && q < mine; ++q) issue(q);
  float acc = 0.f;
  for (size_t q = 0; q < mine; ++q) {
    if (lane == 0 && q + STAGES - 1 < mine) issue(q + STAGES - 1);
    int s = q % STAGES; uint32_t par = (q / STAGES) & 1, ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(bars + s)), "r"(par) : "memory");
    const float4* b = reinterpret_cast<const float4*>(ring + (size_t)s * chunk);
    for (int i = lane; i < chunk / 16; i += 32) { float4 v = b[i]; acc += v.x + v.y + v.z + v.w; }
    __syncwarp();
  }
  if (acc == 123.f) out[0] = acc;
}

int main() {
  size_t bytes = (size_t)8 << 30;
  char* x; float* out;
  cudaMalloc(&x, bytes); cudaMalloc(&out, 4);
  cudaMemset(x, 0, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int bs : {256, 512, 1024}) for (int occ : {2, 4, 8}) {
    ldg_sum<<<sms * occ, bs>>>((const float4*)x, bytes / 16, out);
    cudaEventRecord(a); for (int r = 0; r < 3; ++r) ldg_sum<<<sms * occ, bs>>>((const float4*)x, bytes / 16, out); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("ldg  block %4d x %d/SM : %7.1f GB/s\n", bs, occ, 3.0 * bytes / (ms / 1e3) / 1e9);
  }
  for (int chunk : {512, 1024, 2048, 4096, 8192}) for (int warps : {4, 8, 16}) for (int ctas : {1, 2}) {
    const int ST = 4;
    size_t smem = (size_t)warps * ST * chunk + warps * ST * 8;
    if (smem * ctas > 220 * 1024) continue;
    cudaFuncSetAttribute(tma_sum<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tma_sum<ST><<<sms * ctas, warps * 32, smem>>>(x, bytes, chunk, out);
    cudaEventRecord(a); for (int r = 0; r < 3; ++r) tma_sum<ST><<<sms * ctas, warps * 32, smem>>>(x, bytes, chunk, out); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("tma  chunk %5d warps %2d ctas/SM %d stages %d (in flight/SM %6zu B): %7.1f GB/s %s\n", chunk, warps, ctas, ST,
           (size_t)ctas * warps * (ST - 1) * chunk, 3.0 * bytes / (ms / 1e3) / 1e9, cudaGetErrorString(e));
  }
  return 0;
}
