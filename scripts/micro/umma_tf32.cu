// Microtest: tcgen05.mma kind::tf32 with an MN-major SWIZZLE_128B A operand (the layout a
// 128-byte-box TMA with CU_TENSOR_MAP_SWIZZLE_128B writes) and a K-major no-swizzle B
// operand; D = A(128 x 16) B(16 x 32) in TMEM, read back with tcgen05.ld 32x32b.x32.
// Checks (1) the descriptor layouts with exact small-integer data and (2) how the tensor
// core converts fp32 operands to tf32 (truncation vs rounding).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_tf32 umma_tf32.cu
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// A: element (m, k) of an M=128 x K=16 tile, MN-major, SW128: [blk = m/32][k][32 floats],
// 16-byte chunk index (m%32)/4 xor (k%8).  B: element (k, n), K-major no swizzle:
// [k/4][n/8][n%8][k%4].
__device__ __forceinline__ int a_off(int m, int k, int mode) {
  if (mode == 1) return (((k >> 2) * 16 + (m >> 3)) * 8 + (m & 7)) * 4 + (k & 3);   // K-major interleave
  if (mode == 2) return (((m >> 2) * 2 + (k >> 3)) * 8 + (k & 7)) * 4 + (m & 3);    // MN-major interleave
  const int blk = m >> 5, mm = m & 31;
  const int chunk = (mm >> 2) ^ (k & 7);
  return blk * (16 * 32) + k * 32 + chunk * 4 + (mm & 3);
}
__device__ __forceinline__ int b_off(int k, int n) { return (((k >> 2) * 4 + (n >> 3)) * 8 + (n & 7)) * 4 + (k & 3); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

__global__ void k_test(const float* A, const float* B, float* D, int mode) {
  __shared__ __align__(1024) float sa[128 * 16];
  __shared__ __align__(1024) float sb[16 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 16; i += blockDim.x) {
    const int m = i / 16, k = i % 16;
    sa[a_off(m, k, mode)] = A[m * 16 + k];
  }
  for (int i = t; i < 16 * 32; i += blockDim.x) {
    const int k = i / 32, n = i % 32;
    sb[b_off(k, n)] = B[k * 32 + n];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = taddr_s;
  if (mode == 3) {            // A -> TMEM columns [32, 48): lane m = row m, column 32 + k = A[m][k]
    uint32_t v[16];
    for (int k = 0; k < 16; ++k) v[k] = __float_as_uint(A[t * 16 + k]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(taddr + 32 + ((uint32_t)(warp * 32) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]),
                    "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
                    "r"(v[14]), "r"(v[15]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((mode == 1 || mode == 3 ? 0u : 1u) << 15) | ((32u >> 3) << 17) |
                         ((128u >> 4) << 24);
  if (t == 0) {
    for (int k0 = 0; k0 < 16; k0 += 8) {
      // mode 0: SW128 MN-major, LBO = MN-block stride, SBO = 8-row K-group stride
      // mode 1: K-major interleave, LBO = K core-matrix stride (16 x 128 B), SBO = 8-row M-group stride
      // mode 2: MN-major interleave: core matrix [4 m][8 k] 128 B; LBO = K-group stride, SBO = MN-group stride
      const uint64_t da = mode == 0 ? desc(smem_u32(sa) + (k0 / 8) * 1024, 16 * 128, 1024, 2)
                        : mode == 1 ? desc(smem_u32(sa) + (k0 / 4) * 2048, 2048, 128, 0)
                                    : desc(smem_u32(sa) + (k0 / 8) * 128, 128, 256, 0);
      const uint64_t db = desc(smem_u32(sb) + (k0 / 4) * 512, 512, 128, 0);
      const uint32_t acc = k0 > 0;
      if (mode == 3) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     :: "r"(taddr), "r"(taddr + 32 + k0), "l"(db), "r"(idesc), "r"(acc));
        continue;
      }
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                   :: "r"(taddr), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
  }
  // wait for the MMA
  asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}"
               :: "r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 32; ++j) D[t * 32 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(taddr));
}

int run(int mode) {
  printf("mode %d\n", mode);
  float hA[128 * 16], hB[16 * 32], hD[128 * 32];
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  // (1) layouts: small integers, exact
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 16; ++k) hA[m * 16 + k] = (float)(((m * 7 + k * 3) % 64) - 32);
  for (int k = 0; k < 16; ++k) for (int n = 0; n < 32; ++n) hB[k * 32 + n] = (float)(((k * 5 + n * 11) % 16) - 8);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  k_test<<<1, 128>>>(dA, dB, dD, mode);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 32; ++n) {
    double s = 0; for (int k = 0; k < 16; ++k) s += (double)hA[m * 16 + k] * hB[k * 32 + n];
    if (s != hD[m * 32 + n]) { if (bad < 8) printf("mismatch m=%d n=%d got %g want %g\n", m, n, hD[m * 32 + n], s); ++bad; }
  }
  printf("layout test: %d mismatches of %d\n", bad, 128 * 32);
  // (2) conversion: A[m][0] = 1 + c_m 2^-13 (c_m = 0..127 -> low 13 bits), B = e_00
  memset(hB, 0, sizeof hB); hB[0] = 1.f;
  for (int m = 0; m < 128; ++m) for (int k = 0; k < 16; ++k) {
    uint32_t bits = 0x3f800000u | (uint32_t)(m * 64);    // low 13 bits = m * 64 (m < 128)
    float v; memcpy(&v, &bits, 4); hA[m * 16 + k] = k == 0 ? v : 0.f;
  }
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  k_test<<<1, 128>>>(dA, dB, dD, mode);
  cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int trunc = 0, rn = 0, exact = 0;
  for (int m = 0; m < 128; ++m) {
    uint32_t in; memcpy(&in, &hA[m * 16], 4);
    uint32_t out; memcpy(&out, &hD[m * 32], 4);
    const uint32_t t = in & 0xffffe000u;
    const uint32_t low = in & 0x1fffu;
    const uint32_t r = low > 0x1000u || (low == 0x1000u && (t & 0x2000u)) ? t + 0x2000u : t;
    trunc += out == t; rn += out == r; exact += out == in;
  }
  printf("conversion: matches truncation %d, round-nearest-even %d, exact fp32 %d (of 128)\n", trunc, rn, exact);
  printf("D[1][0] = %08x from A %08x\n", *(uint32_t*)&hD[32], *(uint32_t*)&hA[16]);
  return 0;
}
int main() { for (int m = 0; m < 4; ++m) run(m); return 0; }
