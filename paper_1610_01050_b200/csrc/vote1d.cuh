// The per-frame body of the D = 1 vote (identity I1, Props. 3-4 P:437-450; Alg. 1 l.11-14
// P:226-229), shared by the warp-per-frame vote kernel (vote.cu: k_vote1d) and the fused c1 path
// (kernels.cu: k_gather1d with vote warps).  Header-only.
#pragma once
#include <cstdint>

#include "rsft_internal.h"

namespace rsft {

// One frame of the D = 1 vote (k_vote1d; the fused c1 path in k_gather1d): masks mlo / mhi of
// the L loops in registers; dw = the warp's N/32 detection words in shared memory (zero on entry,
// zero on exit); ent (32 ints) and q (64 words) warp-private scratch.  Writes the frame's
// detection words, its count (rcount) and its ascending local index list (slots, if not null).
template <int LP>
__device__ __forceinline__ void vote1d_frame(const PlanDev& pd, const uint32_t (&mlo)[LP], const uint32_t (&mhi)[LP],
                                             const int (&sg)[LP], const int* __restrict__ sinv_s, int* ent,
                                             uint32_t* q, uint32_t* dw, int64_t frame, uint32_t* __restrict__ detect,
                                             unsigned long long* __restrict__ rcount, uint32_t* __restrict__ slots,
                                             int list_cap) {
  const int lane = threadIdx.x & 31;
  const int N = pd.n[0], L = pd.L, mu = pd.mu, lga = pd.lga[0];
  const int A = 1 << lga, nw = N >> 5;
  const uint32_t nm = (uint32_t)(N - 1), lt = (1u << lane) - 1u;
  const int ncl = L - mu + 1;                          // candidate loops needed
  // one vote: bit M_l(i) of loop l (Def. 3)
  auto vote = [&](int l, uint32_t i) -> uint32_t {
    const uint32_t k = (((uint32_t)sg[l] * i) & nm) >> lga;
    return ((k < 32 ? mlo[l] : mhi[l]) >> (k & 31)) & 1u;
  };
  // candidate loops: the ncl loops with the fewest set buckets (bit l of cmask); for
  // mu = L also a filter loop lf (fewest set buckets among the others)
  uint32_t cmask = 0u;
  int ncand = 0;
  int lf = -1;
  uint32_t flo = 0xffffffffu, fhi = 0xffffffffu, fsg = 0u;
  if (mu == L) {
    // one pass: the loop with the fewest set buckets gives the candidates, the runner-up filters
    // (best / runner-up kept in plain registers: compile-time indices only)
    int b1 = 1 << 30, b2 = 1 << 30, l1 = 0;
    uint32_t blo = 0u, bhi = 0u, bsg = 0u;
#pragma unroll
    for (int l = 0; l < LP; ++l) {
      const int pc = l < L ? __popc(mlo[l]) + __popc(mhi[l]) : (1 << 30);
      if (pc < b1) {
        if (b1 < (1 << 30)) { b2 = b1; lf = l1; flo = blo; fhi = bhi; fsg = bsg; }
        b1 = pc; l1 = l; blo = mlo[l]; bhi = mhi[l]; bsg = (uint32_t)sg[l];
      } else if (pc < b2) {
        b2 = pc; lf = l; flo = mlo[l]; fhi = mhi[l]; fsg = (uint32_t)sg[l];
      }
    }
    cmask = 1u << l1;
    ncand = b1;
    if (b2 >= (1 << 30)) lf = -1;
  } else {
    for (int t = 0; t < ncl; ++t) {
      int best = 1 << 30, bl = 0;
#pragma unroll
      for (int l = 0; l < LP; ++l) {
        const int pc = __popc(mlo[l]) + __popc(mhi[l]);
        if (l < L && !((cmask >> l) & 1u) && pc < best) { best = pc; bl = l; }
      }
      cmask |= 1u << bl;
      ncand += best;
    }
  }
  if (2 * ncand * A <= N) {                         // ---- candidate mode
    int base = 0;                                   // entries (loop, bucket), ascending loops
#pragma unroll
    for (int l = 0; l < LP; ++l) {
      if (!((cmask >> l) & 1u)) continue;
      const bool b0 = (mlo[l] >> lane) & 1u, b1 = (mhi[l] >> lane) & 1u;
      const uint32_t bl0 = __ballot_sync(0xffffffffu, b0), bl1 = __ballot_sync(0xffffffffu, b1);
      if (b0) ent[base + __popc(bl0 & lt)] = (l << 8) | lane;
      base += __popc(bl0);
      if (b1) ent[base + __popc(bl1 & lt)] = (l << 8) | (lane + 32);
      base += __popc(bl1);
    }
    __syncwarp();
    // full test of up to 32 queued locations (lane per location), all loops
    auto drain = [&](int n) {
      const uint32_t i = lane < n ? q[lane] : 0u;
      int cnt = 0;
#pragma unroll
      for (int l = 0; l < LP; ++l)
        if (l < L) cnt += (int)vote(l, i);
      if (lane < n && cnt >= mu) atomicOr(&dw[i >> 5], 1u << (i & 31));
    };
    int qn = 0;
    const int T = ncand * A;
    for (int c0 = 0; c0 < T; c0 += 32) {
      const int c = c0 + lane;
      const bool valid = c < T;
      const int e = ent[valid ? (c >> lga) : 0];
      const uint32_t u = ((uint32_t)(e & 255) << lga) | (uint32_t)(c & (A - 1));
      const uint32_t i = ((uint32_t)sinv_s[e >> 8] * u) & nm;          // Def. 4
      // mu = L: a location needs the filter loop's vote too (cheap pre-test, then queue)
      bool pass = valid;
      if (lf >= 0) {
        const uint32_t k = ((fsg * i) & nm) >> lga;
        pass = pass && (((k < 32 ? flo : fhi) >> (k & 31)) & 1u);
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, pass);
      if (pass) q[qn + __popc(bal & lt)] = i;
      qn += __popc(bal);
      __syncwarp();
      if (qn >= 32) {
        drain(32);
        __syncwarp();
        const uint32_t rest = lane + 32 < qn ? q[lane + 32] : 0u;
        __syncwarp();
        if (lane + 32 < qn) q[lane] = rest;
        qn -= 32;
        __syncwarp();
      }
    }
    if (qn > 0) drain(qn);
  } else {                                          // ---- dense mode
    for (int w = 0; w < nw; ++w) {
      const uint32_t i = (uint32_t)(w << 5) | (uint32_t)lane;
      int cnt = 0;
#pragma unroll
      for (int l = 0; l < LP; ++l)
        if (l < L) cnt += (int)vote(l, i);
      const uint32_t word = __ballot_sync(0xffffffffu, cnt >= mu);
      if (lane == 0) dw[w] = word;
    }
  }
  __syncwarp();
  // read-out: detection words (coalesced), count, ascending local index list
  uint32_t* det = detect + (size_t)frame * nw;
  uint32_t* sl = slots ? slots + (size_t)frame * list_cap : nullptr;
  int run = 0;
  for (int w0 = 0; w0 < nw; w0 += 32) {
    const int w = w0 + lane;
    uint32_t v = 0u;
    if (w < nw) { v = dw[w]; dw[w] = 0u; det[w] = v; }
    if (__ballot_sync(0xffffffffu, v != 0u) == 0u) continue;   // most words of a frame are empty
    const int c = __popc(v);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (sl) {
      int qq = run + incl - c;
      while (v) {
        const int bit = __ffs(v) - 1;
        v &= v - 1;
        if (qq < list_cap) sl[qq] = (uint32_t)((w << 5) + bit);
        ++qq;
      }
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (rcount && lane == 0) rcount[frame] = (unsigned long long)run;
}

}  // namespace rsft
