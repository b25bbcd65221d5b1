// Microbenchmark: streaming the c5 cube [2048][512][64] complex64 (512 MiB) with per-warp
// tensor-map TMA rings, box = [64 cols][b1 consecutive rows s1][b2 rows s1 stride 32][1 plane].
// Orders: 0 = class-major (a warp walks one residue class (r0, r1): a1 blocks, then a0),
//         1 = memory-major (consecutive warps take adjacent boxes of a plane).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void cube_sum(const __grid_constant__ CUtensorMap tm, int b1, int b2, int S, int order, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int box = 512 * b1 * b2;
  unsigned char* ring = sm + (size_t)warp * S * box;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)nw * S * box) + warp * S;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int n1 = 32 / b1, n2 = 16 / b2;             // box grid over (r1, a1) per plane
  const long nbox = 2048L * n1 * n2;
  const long gw = (long)gridDim.x * nw, wid = (long)blockIdx.x * nw + warp;
  const long per = nbox / gw, rem = nbox % gw;       // contiguous box ranges per warp
  const long mine = per + (wid < rem);
  const long start = wid * per + (wid < rem ? wid : rem);
  auto coords = [&](long q, int& c1, int& c2, int& c3) {
    long i = order == 0 ? start + q : wid + q * gw;
    if (order == 0) {              // i -> (r1g, r0, a0, a1g) with a1g fastest: class-major walk
      int a1g = (int)(i % n2); i /= n2;
      int a0 = (int)(i % 32); i /= 32;
      int r0 = (int)(i % 64); i /= 64;
      int r1g = (int)i;
      c1 = r1g * b1; c2 = a1g * b2; c3 = r0 + 64 * a0;
    } else {                       // i -> (plane, a1g, r1g) with r1g fastest: memory order
      int r1g = (int)(i % n1); i /= n1;
      int a1g = (int)(i % n2); i /= n2;
      c1 = r1g * b1; c2 = a1g * b2; c3 = (int)i;
    }
  };
  auto issue = [&](long q) {
    int s = q % S, c1, c2, c3;
    coords(q, c1, c2, c3);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bars + s)), "r"(box) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 :: "r"(su32(ring + (size_t)s * box)), "l"(&tm), "r"(0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(bars + s)) : "memory");
  };
  if (lane == 0) for (long q = 0; q < S - 1 && q < mine; ++q) issue(q);
  float acc = 0.f;
  for (long q = 0; q < mine; ++q) {
    if (lane == 0 && q + S - 1 < mine) issue(q + S - 1);
    int s = q % S; uint32_t par = (q / S) & 1, ok = 0;
    while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(bars + s)), "r"(par) : "memory");
    const float4* b = reinterpret_cast<const float4*>(ring + (size_t)s * box);
    for (int i = lane; i < box / 16; i += 32) { float4 v = b[i]; acc += v.x + v.w; }
    __syncwarp();
  }
  if (acc == 123.f) out[0] = acc;
}

int main() {
  size_t bytes = (size_t)512 << 20;
  char* x; float* out;
  cudaMalloc(&x, bytes); cudaMalloc(&out, 4);
  cudaMemset(x, 0, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fnp = nullptr; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct Cfg { int b1, b2, S, warps, ctas; };
  Cfg cfgs[] = {{1, 8, 3, 8, 1}, {1, 8, 2, 8, 2}, {1, 4, 4, 8, 2}, {1, 8, 4, 8, 1}, {1, 16, 2, 8, 1},
                {8, 1, 3, 8, 1}, {8, 1, 2, 8, 2}, {4, 1, 4, 8, 2}, {8, 2, 2, 8, 1}, {32, 1, 2, 8, 1},
                {4, 2, 3, 8, 1}, {2, 4, 3, 8, 1}, {16, 1, 3, 8, 1}};
  for (int order = 0; order < 2; ++order)
    for (Cfg c : cfgs) {
      CUtensorMap tm;
      cuuint64_t dims[4] = {64, 32, 16, 2048};
      cuuint64_t str[3] = {512, 16384, 262144};
      cuuint32_t boxd[4] = {64, (cuuint32_t)c.b1, (cuuint32_t)c.b2, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 4, x, dims, str, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) { printf("encode failed %d\n", (int)r); continue; }
      size_t box = 512 * c.b1 * c.b2;
      size_t smem = (size_t)c.warps * c.S * box + c.warps * c.S * 8;
      if (smem * c.ctas > 225 * 1024) { printf("skip b1=%d b2=%d S=%d\n", c.b1, c.b2, c.S); continue; }
      cudaFuncSetAttribute(cube_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int grid = sms * c.ctas;
      cube_sum<<<grid, c.warps * 32, smem>>>(tm, c.b1, c.b2, c.S, order, out);
      cudaEventRecord(a);
      for (int rep = 0; rep < 10; ++rep) cube_sum<<<grid, c.warps * 32, smem>>>(tm, c.b1, c.b2, c.S, order, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("order %d box [64][%2d r1][%2d a1] (%5zu B) S=%d warps=%d ctas/SM=%d inflight/SM=%6zu: %7.1f GB/s %s\n", order,
             c.b1, c.b2, box, c.S, c.warps, c.ctas, (size_t)c.ctas * c.warps * (c.S - 1) * box,
             10.0 * bytes / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
