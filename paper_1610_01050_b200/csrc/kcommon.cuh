// Device helpers shared by the CUDA translation units of librsft (kernels.cu: fold / FFT /
// threshold; vote.cu: reverse map / vote / compaction).  Header-only, everything inline.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "rsft_internal.h"

namespace rsft {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// Streaming 16-byte load of x (read exactly once: no L1 allocation).  Volatile so that a
// row group's U loads stay in program order; pin() below then forces all U loads to be
// issued before the first FMA consumes any of them (U x 512 B in flight per warp).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void pin(float4& a) {
  asm volatile("" : "+f"(a.x), "+f"(a.y), "+f"(a.z), "+f"(a.w));
}

__device__ __forceinline__ int brev(int v, int lg) { return lg ? (int)(__brev((unsigned)v) >> (32 - lg)) : 0; }

// acc += w * v for a complex pair v: one complex x real MAC as a single packed FMA
// (__ffma2_rn -> SASS FFMA2 R, R.F32, R.F32x2, R.F32x2 on sm_100a).
__device__ __forceinline__ void mac(float2& acc, float w, float vx, float vy) {
  acc = __ffma2_rn(make_float2(w, w), make_float2(vx, vy), acc);
}

// ------------------------------------------------------------------------------------
// Programmatic dependent launch: every hot-path kernel is launched with programmatic stream
// serialization and starts with griddepcontrol.wait (before any global access: the previous
// kernel's writes are visible after it) + launch_dependents, so the next kernel's CTAs are
// scheduled while this one drains instead of after a full launch round trip.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// Tensor-map TMA (cp.async.bulk.tensor; SASS UTMALDG): one instruction moves a whole box
// (U rows x 512 B of one residue class), zero-filling out-of-bounds rows.
__device__ __forceinline__ void tma_load_4d(void* dst, uint64_t tmap, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3, %4, %5}], [%6];"
               :: "r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, uint64_t tmap, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               :: "r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, uint64_t tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

// expect_tx + 4-D tensor-map load issued by lane 0 only, through predicates: every lane runs
// the producer cursor (warp-uniform values), so there is no divergent branch per box.
__device__ __forceinline__ void tma_load_4d_lane0(int lane, void* dst, uint64_t tmap, int c0, int c1, int c2, int c3,
                                                  uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %0, 0;\n\t"
               "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%7], %8;\n\t"
               "@p cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%1], [%2, {%3, %4, %5, %6}], [%7];\n\t}"
               :: "r"(lane), "r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)),
                  "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_5d_lane0(int lane, void* dst, uint64_t tmap, int c0, int c1, int c2, int c3,
                                                  int c4, uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %0, 0;\n\t"
               "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%8], %9;\n\t"
               "@p cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%1], [%2, {%3, %4, %5, %6, %7}], [%8];\n\t}"
               :: "r"(lane), "r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
                  "r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    // suspend-time hint (ns): the warp sleeps until the phase flips instead of spinning
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(a), "r"(parity), "r"(1000000u) : "memory");
  }
}

// mbar_wait for warps that usually wait long (nothing else to do meanwhile): test the phase, then
// sleep `ns` before the next test, so the waiting warp does not take issue slots from the warps
// doing the work (try_wait returns long before its suspend-time hint and its loop re-issues).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns) {
  const uint32_t a = smem_u32(bar);
  for (;;) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    __nanosleep(ns);
  }
}

constexpr int kStageIdx = 2048;          // indices staged per CTA for coalesced writes

// Block-wide exclusive scan of one int per thread; returns the prefix, *total = sum.
__device__ __forceinline__ int block_excl_scan(int c, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int wbase = 0, t = 0;
  for (int i = 0; i < nw; ++i) {
    if (i < warp) wbase += wsum[i];
    t += wsum[i];
  }
  *total = t;
  return wbase + incl - c;
}


}  // namespace rsft
