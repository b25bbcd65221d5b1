// K3/K4 of the RSFT hot path for sm_100a: reverse mapping + accumulation + second-stage test
// (Alg. 1 l.11-14; Def. 4; Eq. a_i; identity I1 from Props. 3-4,
// P:437-450) and the compaction of detections to sorted index lists.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "kcommon.cuh"
#include "hcommon.h"
#include "vote1d.cuh"

namespace rsft {

// Vote one region whose bitmap slice bm [L][lw] is in shared memory (see k_vote): builds
// E (shared, [L][B_rd][W] words), votes every item of the region, writes its detection words
// (detect, if not null) and abar (counts, MODE 2, if not null).  Returns this thread's
// detection popcount.  Contains __syncthreads: every thread of the CTA calls it.
// LIST: items are assigned kListIpt-contiguous per thread, kept in registers, and the
// region's detections are also written as ascending region-local location indices to
// slot[0 .. min(total, cap)) (the return value is then the region total, on every thread).
constexpr int kListIpt = 4;              // items per thread in LIST mode (<= 32 words)

template <int CW, int MODE, bool LIST = false>
__device__ int vote_region(const PlanDev& pd, const uint32_t* bm, int lw, uint32_t* E, const int* sig_rd,
                           const uint32_t* Xs, const uint32_t* NT, const int* kpre_s, const int* sig_ld,
                           int64_t frame, int64_t i0,
                           int64_t d0b, int64_t d0e, uint32_t* __restrict__ detect, uint8_t* __restrict__ counts,
                           bool ebuilt, int* wsum = nullptr, uint32_t* __restrict__ slot = nullptr) {
  const int D = pd.D, L = pd.L, wpl = pd.wpl;
  const int ld = D - 1;
  const int nld = pd.n[ld], lga_ld = pd.lga[ld];
  const int W = nld >> 5;
  const int lgW = __ffs(W) - 1;
  const int brd = D >= 2 ? pd.b[D - 2] : 1;
  const int blast = pd.blast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int rowbits = brd * blast;
  const int nrd = D >= 2 ? pd.n[D - 2] : 1;
  const int lga_rd = D >= 2 ? pd.lga[D - 2] : 0;
  const int chunks = W / CW;
  const int lg_chunks = __ffs(chunks) - 1;
  const int mu = pd.mu;
  const int64_t slab_locs = (d0e - d0b) * (pd.ntot / pd.n[0]);
  const int64_t slab_words = slab_locs >> 5;
  constexpr bool COUNT = true;
  int cnt = 0;
  (void)wpl;
    // E[l][krd][w] (all loops at once).  With nibble tables NT[l][g][n][w] = OR of the X masks
    // of the set bits of n in bucket group g (4 buckets), one entry costs B_last/4 lookups.
    // (ebuilt: the caller copied E from the precomputed table, k_etab.)
    if (ebuilt) {
    } else if (pd.xmask) {
      const int lg_rw = (brd > 1 ? __ffs(brd) - 1 : 0) + lgW;
      for (int j = tid; j < L * brd * W; j += blockDim.x) {
        const int l = j >> lg_rw, rem = j & ((1 << lg_rw) - 1);
        const int krd = rem >> lgW, w = rem & (W - 1);
        int base = 0;
        if (D == 3) base = lw < wpl ? (kpre_s[l] * rowbits) & 31 : kpre_s[l] * rowbits;
        const uint32_t* b = bm + (size_t)l * lw;
        const int f0 = base + krd * blast;
        uint32_t e = 0;
        if (NT) {
          const uint32_t* T = NT + (size_t)l * (blast >> 2) * 16 * W + w;
          if (blast <= 32) {
            uint32_t pat = (b[f0 >> 5] >> (f0 & 31)) & (blast == 32 ? 0xffffffffu : ((1u << blast) - 1u));
            for (int g = 0; g < (blast >> 2); ++g, pat >>= 4) e |= T[((g << 4) + (pat & 15)) * W];
          } else {
            uint32_t lo = b[f0 >> 5], hi = b[(f0 >> 5) + 1];
#pragma unroll
            for (int g = 0; g < 8; ++g, lo >>= 4) e |= T[((g << 4) + (lo & 15)) * W];
#pragma unroll
            for (int g = 8; g < 16; ++g, hi >>= 4) e |= T[((g << 4) + (hi & 15)) * W];
          }
        } else {
          const uint32_t* X = Xs + (size_t)l * blast * W;
          if (blast <= 32) {
            uint32_t pat = (b[f0 >> 5] >> (f0 & 31)) & (blast == 32 ? 0xffffffffu : ((1u << blast) - 1u));
            while (pat) {
              const int k = __ffs(pat) - 1;
              pat &= pat - 1;
              e |= X[k * W + w];
            }
          } else {                                   // blast == 64: two aligned words
            uint32_t lo = b[f0 >> 5], hi = b[(f0 >> 5) + 1];
            while (lo) { const int k = __ffs(lo) - 1; lo &= lo - 1; e |= X[k * W + w]; }
            while (hi) { const int k = __ffs(hi) + 31; hi &= hi - 1; e |= X[k * W + w]; }
          }
        }
        E[j] = e;
      }
    } else {                                         // no masks (too large): thread per E word
      const int lg_rw = (brd > 1 ? __ffs(brd) - 1 : 0) + lgW;
      for (int j = tid; j < L * brd * W; j += blockDim.x) {
        const int l = j >> lg_rw, rem = j & ((1 << lg_rw) - 1);
        const int krd = rem >> lgW, w = rem & (W - 1);
        int base = 0;
        if (D == 3) base = lw < wpl ? (kpre_s[l] * rowbits) & 31 : kpre_s[l] * rowbits;
        const uint32_t* b = bm + (size_t)l * lw;
        const uint32_t sg = (uint32_t)sig_ld[l];
        uint32_t m = (sg * (uint32_t)(w << 5)) & (uint32_t)(nld - 1);   // [sigma i]_N, i = 32 w
        const int f0 = base + krd * blast;
        uint32_t e = 0;
#pragma unroll 8
        for (int q = 0; q < 32; ++q) {                 // M_l(i) = floor(B [sigma i]_N / N) (Def. 3)
          const int flat = f0 + (int)(m >> lga_ld);
          e |= ((b[flat >> 5] >> (flat & 31)) & 1u) << q;
          m = (m + sg) & (uint32_t)(nld - 1);
        }
        E[j] = e;
      }
    }
    __syncthreads();
    int64_t rbeg, rend, out_base;
    if (D == 3) { rbeg = 0; rend = pd.n[1]; out_base = (i0 - d0b) * pd.n[1] * W; }
    else if (D == 2) { rbeg = d0b; rend = d0e; out_base = 0; }
    else { rbeg = 0; rend = 1; out_base = 0; }
    const int64_t nitems = (rend - rbeg) * chunks;

    // one item = CW consecutive detection words of one row
    auto vote_item = [&](int64_t it, uint32_t (&acc)[CW]) {
      const int64_t ri = it >> lg_chunks;
      const int w0 = (int)(it - ri * chunks) * CW;
      const int64_t row = rbeg + ri;
      uint32_t pl[CW][6];
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        acc[c] = MODE == 0 ? 0xffffffffu : 0u;
#pragma unroll
        for (int b = 0; b < 6; ++b) pl[c][b] = 0u;
      }
      // shared-window byte addresses (32-bit arithmetic; E row of loop l, bucket k_rd at
      // e_l + k_rd W 4; k_rd from the low bits of sigma * row mod N_rd (power of two: the
      // 32-bit product is exact mod 2^32)
      const uint32_t e_w0 = smem_u32(E) + (uint32_t)w0 * 4u;
      const uint32_t rowu = (uint32_t)row, nrdm = (uint32_t)(nrd - 1);
      const uint32_t sig_base = smem_u32(sig_rd);
      for (int l = 0; l < L; ++l) {
        uint32_t sg;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(sg) : "r"(sig_base + 4u * (uint32_t)l));
        const uint32_t krd = D >= 2 ? ((sg * rowu) & nrdm) >> lga_rd : 0u;
        const uint32_t ea = e_w0 + (((uint32_t)l * (uint32_t)brd + krd) * (uint32_t)W) * 4u;
        uint32_t m[CW];
        if (CW % 4 == 0) {
#pragma unroll
          for (int q = 0; q < CW; q += 4) {
            uint4 v;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ea + 4u * (uint32_t)q));
            m[q] = v.x; m[(q + 1) % CW] = v.y; m[(q + 2) % CW] = v.z; m[(q + 3) % CW] = v.w;
          }
        } else if (CW == 2) {
          const uint32_t* e = E + ((size_t)l * brd + krd) * W + w0;
          const uint2 v = *reinterpret_cast<const uint2*>(e);
          m[0] = v.x; m[CW > 1 ? 1 : 0] = v.y;
        } else {
          m[0] = E[((size_t)l * brd + krd) * W + w0];
        }
        uint32_t any = 0;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          if (MODE == 0) { acc[c] &= m[c]; any |= acc[c]; }
          else if (MODE == 1) acc[c] |= m[c];
          else {
            uint32_t carry = m[c];
#pragma unroll
            for (int b = 0; b < 6; ++b) {
              const uint32_t t = pl[c][b] & carry;
              pl[c][b] ^= carry;
              carry = t;
            }
          }
        }
        if (MODE == 0 && any == 0) break;              // unanimity already impossible
      }
      if (MODE == 2) {                                 // bit-sliced compare: count >= mu
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          uint32_t gt = 0u, eq = 0xffffffffu;
#pragma unroll
          for (int b = 5; b >= 0; --b) {
            if ((mu >> b) & 1) eq &= pl[c][b];
            else { gt |= eq & pl[c][b]; eq &= ~pl[c][b]; }
          }
          acc[c] = gt | eq;
        }
      }
      const int64_t widx = out_base + ri * W + w0;
      if (detect) {
        uint32_t* dst = detect + frame * slab_words + widx;
        if (CW % 4 == 0) {
#pragma unroll
          for (int q = 0; q < CW; q += 4)
            *reinterpret_cast<uint4*>(dst + q) = make_uint4(acc[q], acc[(q + 1) % CW], acc[(q + 2) % CW], acc[(q + 3) % CW]);
        } else if (CW == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(acc[0], acc[CW > 1 ? 1 : 0]);
        else dst[0] = acc[0];
      }
      if (MODE == 2 && counts) {
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          uint8_t* cdst = counts + frame * slab_locs + (widx + c) * 32;
          for (int j = 0; j < 32; ++j) {
            int v = 0;
#pragma unroll
            for (int b = 0; b < 6; ++b) v |= ((pl[c][b] >> j) & 1u) << b;
            cdst[j] = (uint8_t)v;
          }
        }
      }
    };

    if constexpr (LIST) {
      // items it = tid + k * blockDim (coalesced detection-word stores); word order is
      // k-major, so the position of item (k, tid) is sum_{k' < k} T_k' + prefix_k(tid)
      uint32_t words[kListIpt][CW];
      int ck[kListIpt];
#pragma unroll
      for (int k = 0; k < kListIpt; ++k) {
        const int64_t it = tid + (int64_t)k * blockDim.x;
        ck[k] = 0;
#pragma unroll
        for (int c = 0; c < CW; ++c) words[k][c] = 0u;
        if (it < nitems) {
          vote_item(it, words[k]);
#pragma unroll
          for (int c = 0; c < CW; ++c) ck[k] += __popc(words[k][c]);
        }
      }
      int incl[kListIpt];
#pragma unroll
      for (int k = 0; k < kListIpt; ++k) {
        incl[k] = ck[k];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl[k], off);
          if (lane >= off) incl[k] += v;
        }
        if (lane == 31) wsum[k * nwarps + warp] = incl[k];
      }
      __syncthreads();
      int pos[kListIpt], total = 0;
#pragma unroll
      for (int k = 0; k < kListIpt; ++k) {
        int before = 0, tk = 0;
        for (int w2 = 0; w2 < nwarps; ++w2) {
          const int v = wsum[k * nwarps + w2];
          if (w2 < warp) before += v;
          tk += v;
        }
        pos[k] = total + before + incl[k] - ck[k];
        total += tk;
      }
      if (total <= pd.list_cap) {
#pragma unroll
        for (int k = 0; k < kListIpt; ++k) {
          if (__ballot_sync(0xffffffffu, ck[k] != 0) == 0u) continue;   // most rows hold no detection
          const int64_t it = tid + (int64_t)k * blockDim.x;
          int q = pos[k];
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            uint32_t v = words[k][c];
            while (v) {
              const int bit = __ffs(v) - 1;
              v &= v - 1;
              slot[q++] = (uint32_t)((it * CW + c) * 32 + bit);
            }
          }
        }
      }
      __syncthreads();                             // wsum reused by the next region
      return total;
    }
    if constexpr (!LIST) {
      for (int64_t it = tid; it < nitems; it += blockDim.x) {
        uint32_t acc[CW];
        vote_item(it, acc);
        if (COUNT) {
#pragma unroll
          for (int c = 0; c < CW; ++c) cnt += __popc(acc[c]);
        }
      }
    }
  return cnt;
}

// ------------------------------------------------------------------------------------
// D == 3 vote, E words for every dim-0 bucket (computed once per frame instead of once per
// region: N_0 regions share B_0 distinct k_pre): etab[frame][l][k0][k1][w] = OR over the set
// last-dim buckets k2 of bucket row (k0, k1) of loop l's bitmap of the plan-constant X masks
// X[l][k2][w] (bit j of X = location 32 w + j of the last dim hashes to k2; Def. 3 / I1).
__global__ void __launch_bounds__(kThreads) k_etab(PlanDev pd, const uint32_t* __restrict__ bitmaps, int64_t batch) {
  pdl_enter();
  const int L = pd.L, B0 = pd.b[0], B1 = pd.b[1], W = pd.n[2] >> 5, blast = pd.blast, wpl = pd.wpl;
  const int64_t rows = (int64_t)L * B0 * B1;       // bucket rows (l, k0, k1) per frame
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < batch * rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t frame = i / rows;
    const int r = (int)(i - frame * rows);
    const int l = r / (B0 * B1), k01 = r - l * B0 * B1;   // k01 = k0 B1 + k1
    const int flat = k01 * blast;
    const uint32_t* b = bitmaps + ((size_t)frame * L + l) * wpl;
    const uint32_t* X = pd.xmask + (size_t)l * blast * W;
    uint32_t* dst = pd.etab + (size_t)i * W;
    uint32_t lo, hi = 0;
    if (blast <= 32) lo = (__ldg(b + (flat >> 5)) >> (flat & 31)) & (blast == 32 ? 0xffffffffu : ((1u << blast) - 1u));
    else { lo = __ldg(b + (flat >> 5)); hi = __ldg(b + (flat >> 5) + 1); }
    for (int w0 = 0; w0 < W; w0 += 4) {            // W is a power of two (1, 2, 4, ...)
      const int nw = W - w0 < 4 ? W - w0 : 4;
      uint32_t e[4] = {0u, 0u, 0u, 0u};
      uint32_t pl = lo, ph = hi;
      while (pl) {
        const int k = __ffs(pl) - 1; pl &= pl - 1;
        for (int q = 0; q < nw; ++q) e[q] |= __ldg(X + (size_t)k * W + w0 + q);
      }
      while (ph) {
        const int k = __ffs(ph) + 31; ph &= ph - 1;
        for (int q = 0; q < nw; ++q) e[q] |= __ldg(X + (size_t)k * W + w0 + q);
      }
      for (int q = 0; q < nw; ++q) dst[w0 + q] = e[q];
    }
  }
}

// cp.async (LDGSTS) helpers of the software-pipelined E copies (k_vote, k_vote3d)
__device__ __forceinline__ void v3_cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void v3_cp4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void v3_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void v3_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// k_etab for B_last = 8 with the plan-constant nibble tables (c3, c5): one thread per first-stage
// bitmap word = 4 bucket rows (k0, k1) of 8 last-dim buckets each; every E word is two nibble
// lookups, NT[l][0][bits 0-3][w] | NT[l][1][bits 4-7][w], and the 4 W words of the thread's rows
// are contiguous in etab (row index = 4 x word index: B_tot = 32 wpl).  One coalesced load per
// thread, issued before the table staging, no per-bit loop.
template <int W>
__global__ void __launch_bounds__(256) k_etab8(PlanDev pd, const uint32_t* __restrict__ bitmaps, int64_t nwords) {
  pdl_enter();
  extern __shared__ __align__(16) uint32_t nts[];    // [L][2][16][W]
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t bw = i < nwords ? __ldg(bitmaps + i) : 0u;
  const int L = pd.L, wpl = pd.wpl;
  for (int j = threadIdx.x; j < L * 8 * W; j += blockDim.x)
    reinterpret_cast<uint4*>(nts)[j] = __ldg(reinterpret_cast<const uint4*>(pd.ntab) + j);
  __syncthreads();
  if (i >= nwords) return;
  const int l = (int)((i / wpl) % L);
  const uint32_t* NT = nts + l * 32 * W;
  uint32_t out[4 * W];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t lo = (bw >> (8 * q)) & 15u, hi = (bw >> (8 * q + 4)) & 15u;
#pragma unroll
    for (int w = 0; w < W; ++w) out[q * W + w] = NT[lo * W + w] | NT[(16 + hi) * W + w];
  }
  uint4* dst = reinterpret_cast<uint4*>(pd.etab + (size_t)i * 4 * W);
#pragma unroll
  for (int v = 0; v < W; ++v) dst[v] = make_uint4(out[4 * v], out[4 * v + 1], out[4 * v + 2], out[4 * v + 3]);
}

// E words of every dim-0 bucket for the batch (D == 3): k_etab8 where it applies, else k_etab.
static rsft_status launch_etab(rsft_plan_s* p, const uint32_t* bm, int64_t batch, cudaStream_t st) {
  const int W = (int)(p->n[2] / 32);
  const char* off = getenv("RSFT_NO_ETAB8");         // read per launch: tests select either kernel
  const bool e8 = !(off && off[0] && off[0] != '0') && p->b[2] == 8 && p->dev.ntab && (p->b[0] * p->b[1]) % 4 == 0 &&
                  (W == 1 || W == 2 || W == 4) && p->dev.wpl * 32 == p->b[0] * p->b[1] * p->b[2];
  if (e8) {
    const int64_t nw = batch * p->L * p->dev.wpl;
    const size_t smem = (size_t)p->L * 32 * W * 4;
    auto kern = W == 1 ? k_etab8<1> : W == 2 ? k_etab8<2> : k_etab8<4>;
    if (cudaError_t le_ = pdl_launch(kern, (unsigned)((nw + 255) / 256), 256, smem, st, p->dev, bm, nw); le_ != cudaSuccess)
      return check(le_, "k_etab8 launch");
  } else {
    const int64_t ne = batch * p->L * p->b[0] * p->b[1];
    const int64_t eg = (ne + kThreads - 1) / kThreads;
    if (cudaError_t le_ = pdl_launch(k_etab, (unsigned)(eg < 4 * p->num_sms ? eg : 4 * p->num_sms), kThreads, 0, st,
                                     p->dev, bm, batch); le_ != cudaSuccess)
      return check(le_, "k_etab launch");
  }
  p->last_launches += 1;
  return RSFT_OK;
}

template <int CW, int MODE, bool COUNT, bool LIST>
#ifndef RSFT_VOTE_CTAS
#define RSFT_VOTE_CTAS 4
#endif
__global__ void __launch_bounds__(kThreads, RSFT_VOTE_CTAS) k_vote(PlanDev pd, const uint32_t* __restrict__ bitmaps,
                                                   int64_t d0b, int64_t d0e, int lw, int64_t np, int64_t nregions,
                                                   uint32_t* __restrict__ detect, uint8_t* __restrict__ counts,
                                                   unsigned long long* __restrict__ rcount, int use_etab) {
  pdl_enter();
  extern __shared__ __align__(16) uint32_t vsm[];
  __shared__ int wsum[kListIpt * kThreads / 32];
  const int D = pd.D, L = pd.L, wpl = pd.wpl;
  const int W = pd.n[D - 1] >> 5;                    // words per row of locations
  const int brd = D >= 2 ? pd.b[D - 2] : 1;
  const int blast = pd.blast;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  uint32_t* bm = vsm;
  uint32_t* E = bm + (((size_t)L * lw + 3) & ~size_t(3));   // 16-B aligned for uint4 loads
  int* sig_rd = reinterpret_cast<int*>(E + (((size_t)L * brd * W + 3) & ~size_t(3)));
  uint32_t* Xs = reinterpret_cast<uint32_t*>(sig_rd + kMaxLoops);
  const size_t xw = pd.xmask ? (size_t)L * blast * W : 0;
  uint32_t* NT = (pd.xmask && blast >= 4 && 16 * xw <= kMaxNibbleBytes) ? Xs + ((xw + 3) & ~size_t(3)) : nullptr;
  __shared__ int kpre_s[kMaxLoops];
  __shared__ int sig_ld[kMaxLoops];                  // last-dim sigma per loop
  const int rowbits = brd * blast;                   // bits of one k_pre slab

  for (int l = tid; l < L; l += blockDim.x) {
    sig_rd[l] = D >= 2 ? pd.loops[l].sig[D - 2] : 0;
    sig_ld[l] = pd.loops[l].sig[D - 1];
  }
  if (pd.xmask) {                                    // plan-constant: once per CTA
    const int nx = L * blast * W;
    if ((nx & 3) == 0)
      for (int i = tid; i < (nx >> 2); i += blockDim.x)
        reinterpret_cast<uint4*>(Xs)[i] = __ldg(reinterpret_cast<const uint4*>(pd.xmask) + i);
    else
      for (int i = tid; i < nx; i += blockDim.x) Xs[i] = __ldg(pd.xmask + i);
  }

  if (NT && pd.ntab) {                               // plan-constant nibble tables (bind time)
    const int n4 = (L * (blast >> 2) * 16 * W) >> 2;
    for (int i = tid; i < n4; i += blockDim.x)
      reinterpret_cast<uint4*>(NT)[i] = __ldg(reinterpret_cast<const uint4*>(pd.ntab) + i);
  } else if (NT) {                                   // nibble tables from the X masks (once)
    __syncthreads();
    const int ng = blast >> 2;
    for (int i = tid; i < L * ng * 16 * W; i += blockDim.x) {
      const int w = i % W, n = (i / W) & 15, g = (i / (W * 16)) % ng, l = i / (W * 16 * ng);
      uint32_t e = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((n >> q) & 1) e |= Xs[((size_t)l * blast + 4 * g + q) * W + w];
      NT[i] = e;
    }
  }

  for (int64_t region = blockIdx.x; region < nregions; region += gridDim.x) {
    __syncthreads();                                 // previous region's E / bm readers done
    const int64_t frame = region / np, prefix = region - frame * np;
    const int64_t i0 = d0b + prefix;
    if (D == 3)
      for (int l = tid; l < L; l += blockDim.x)
        kpre_s[l] = (int)(((int64_t)pd.loops[l].sig[0] * i0) & (pd.n[0] - 1)) >> pd.lga[0];

    if (use_etab) {                                  // D == 3: E rows of this region's dim-0 buckets
      __syncthreads();
      const int rw = brd * W, lg_rw = __ffs(rw) - 1;
      const uint32_t* et = pd.etab + (size_t)frame * L * pd.b[0] * rw;
      if ((rw & 3) == 0) {                           // 16-B copies, one L2 round trip per thread
        const int rw4 = rw >> 2, lg4 = lg_rw - 2;
        for (int j = tid; j < L * rw4; j += blockDim.x) {
          const int l = j >> lg4, rem = j & (rw4 - 1);
          reinterpret_cast<uint4*>(E)[j] =
              __ldg(reinterpret_cast<const uint4*>(et + ((size_t)l * pd.b[0] + kpre_s[l]) * rw) + rem);
        }
      } else {
        for (int j = tid; j < L * rw; j += blockDim.x) {
          const int l = j >> lg_rw, rem = j & (rw - 1);
          E[j] = __ldg(et + ((size_t)l * pd.b[0] + kpre_s[l]) * rw + rem);
        }
      }
    }
    // this region's slice of every loop's first-stage bitmap
    const uint32_t* src = bitmaps + (size_t)frame * L * wpl;
    for (int i = use_etab ? L * lw : tid; i < L * lw; i += blockDim.x) {
      const int l = i / lw, w = i - l * lw;
      int start = 0;
      if (D == 3 && lw < wpl) {
        const int kpre = (int)(((int64_t)pd.loops[l].sig[0] * i0) & (pd.n[0] - 1)) >> pd.lga[0];
        start = (kpre * rowbits) >> 5;
      }
      bm[i] = __ldg(src + (size_t)l * wpl + start + w);
    }
    __syncthreads();
    if (LIST) {                                      // region-local index list + count
      const int t = vote_region<CW, MODE, true>(pd, bm, lw, E, sig_rd, Xs, NT, kpre_s, sig_ld, frame, i0, d0b, d0e,
                                                detect, counts, use_etab, wsum,
                                                pd.region_slots + (size_t)region * pd.list_cap);
      if (tid == 0) rcount[region] = (unsigned long long)t;
      continue;
    }
    int cnt = vote_region<CW, MODE>(pd, bm, lw, E, sig_rd, Xs, NT, kpre_s, sig_ld, frame, i0, d0b, d0e, detect,
                                    counts, use_etab);
    if (COUNT) {                                     // this region's detection count
#pragma unroll
      for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
      if (lane == 0) wsum[warp] = cnt;
      __syncthreads();
      if (tid == 0) {
        long long t = 0;
        for (int i = 0; i < nwarps; ++i) t += wsum[i];
        rcount[region] = (unsigned long long)t;
      }
    }
  }
}

// One CTA per region: each thread owns 32 consecutive detection words of a pass of
// 32 x blockDim words (8 x 16-B loads in flight), one block scan of the per-thread counts
// gives every thread its output position in word order; ascending indices are staged in
// shared memory and written at the region's offset (coalesced).
constexpr int kRwWords = 32;               // words per thread per pass

__global__ void __launch_bounds__(kThreads) k_region_write(const uint32_t* __restrict__ det, int64_t rwords,
                                                           const unsigned long long* __restrict__ offsets,
                                                           const long long* __restrict__ d_count, int64_t nregions,
                                                           const uint32_t* __restrict__ slots,
                                                           long long* __restrict__ idx, int64_t capacity,
                                                           int list_cap) {
  pdl_enter();
  __shared__ int wsum[kThreads / 32];
  __shared__ long long s_idx[kStageIdx];
  const int tid = threadIdx.x;
  const int64_t r = blockIdx.x;
  const uint32_t* src = det + r * rwords;
  long long run = (long long)offsets[r];
  if (slots) {                                       // the vote left a region-local index list
    const long long n = (r + 1 < nregions ? (long long)offsets[r + 1] : *d_count) - run;
    if (n <= list_cap) {
      const uint32_t* sl = slots + (size_t)r * list_cap;
      const long long g0 = r * rwords * 32;
      for (long long i = tid; i < n; i += blockDim.x)
        if (run + i < capacity) idx[run + i] = g0 + (long long)sl[i];
      return;
    }
  }
  const bool vec = (rwords & 3) == 0;
  const int64_t pass = (int64_t)kRwWords * blockDim.x;
  for (int64_t p0 = 0; p0 < rwords; p0 += pass) {
    const int64_t w0 = p0 + (int64_t)tid * kRwWords;
    uint32_t w[kRwWords];
#pragma unroll
    for (int q = 0; q < kRwWords; q += 4) {
      if (vec && w0 + q + 3 < rwords) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src + w0 + q));
        w[q] = v.x; w[q + 1] = v.y; w[q + 2] = v.z; w[q + 3] = v.w;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) w[q + c] = w0 + q + c < rwords ? src[w0 + q + c] : 0u;
      }
    }
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < kRwWords; ++q) cnt += __popc(w[q]);
    int total;
    int lp = block_excl_scan(cnt, wsum, &total);
    const bool staged = total <= kStageIdx;
#pragma unroll
    for (int q = 0; q < kRwWords; ++q) {
      uint32_t v = w[q];
      while (v) {
        const int bit = __ffs(v) - 1;
        v &= v - 1;
        const long long g = (r * rwords + w0 + q) * 32 + bit;
        if (staged) s_idx[lp] = g;
        else if (run + lp < capacity) idx[run + lp] = g;
        ++lp;
      }
    }
    __syncthreads();
    if (staged)
      for (int i = tid; i < total; i += blockDim.x)
        if (run + i < capacity) idx[run + i] = s_idx[i];
    run += total;
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------
// K3 for D == 1 (c1-like: many short frames): one WARP per frame, no CTA barrier.
// Reverse mapping + accumulation + second stage (Alg. 1 l.11-14) through the
// hash-lookup form (identity I1, Props. 3-4 P:437-450): abar[i] = sum_l c_l[M_l(i)],
// M_l(i) = floor(B [sigma_l i]_N / N) (Def. 3).  The L first-stage bitmaps of the frame
// (<= 64 buckets each) live in registers as 64-bit masks.
// Candidate mode: a location with abar >= mu has a vote in at least one of ANY L - mu + 1
// loops, so the candidates are the reverse maps R(k, sigma_l^{-1}) (Def. 4, A = N/B locations
// each) of the set buckets of the L - mu + 1 loops with the fewest set buckets; for mu = L a
// candidate must also vote in a filter loop (one cheap test), the survivors are compacted
// into a per-warp queue and tested against all loops 32 at a time, setting their bits in a
// per-warp shared bitmap.
// Used when the candidates are fewer than N/2; otherwise dense mode tests every location.
// Outputs: detection words, and (list mode) the frame's count + ascending local index list
// for k_region_write.
// ------------------------------------------------------------------------------------
constexpr int kVote1dWarps = 8;

template <int LP, int MINB = 1>
__global__ void __launch_bounds__(32 * kVote1dWarps, MINB) k_vote1d(PlanDev pd, const uint32_t* __restrict__ bitmaps,
                                                               int64_t batch, uint32_t* __restrict__ detect,
                                                               unsigned long long* __restrict__ rcount,
                                                               uint32_t* __restrict__ slots, int list_cap) {
  pdl_enter();
  extern __shared__ __align__(16) uint32_t v1s[];
  __shared__ int sig_s[LP], sinv_s[LP];
  __shared__ int ent_s[kVote1dWarps][32];
  __shared__ uint32_t q_s[kVote1dWarps][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int N = pd.n[0], L = pd.L, wpl = pd.wpl;
  const int nw = N >> 5;
  for (int l = threadIdx.x; l < LP; l += blockDim.x) {
    sig_s[l] = l < L ? pd.loops[l].sig[0] : 0;
    sinv_s[l] = l < L ? pd.loops[l].sinv[0] : 0;
  }
  uint32_t* dw = v1s + (size_t)warp * nw;            // this warp's detection words (kept zero)
  for (int w = lane; w < nw; w += 32) dw[w] = 0u;
  __syncthreads();
  int sg[LP];
#pragma unroll
  for (int l = 0; l < LP; ++l) sg[l] = sig_s[l];
  const bool vec = ((L * wpl) & 3) == 0;
  uint32_t* q = q_s[warp];

  const int64_t gw = (int64_t)blockIdx.x * kVote1dWarps + warp, TW = (int64_t)gridDim.x * kVote1dWarps;
  for (int64_t frame = gw; frame < batch; frame += TW) {
    // the frame's L masks (bit k <-> bucket k) in registers (same address on every lane)
    const uint32_t* src = bitmaps + (size_t)frame * L * wpl;
    uint32_t mlo[LP], mhi[LP];
    if (vec && wpl == 2) {
#pragma unroll
      for (int l = 0; l < LP; l += 2) {
        const uint4 v = l < L ? __ldg(reinterpret_cast<const uint4*>(src) + (l >> 1)) : make_uint4(0u, 0u, 0u, 0u);
        mlo[l] = v.x; mhi[l] = v.y;
        if (l + 1 < LP) { mlo[l + 1] = l + 1 < L ? v.z : 0u; mhi[l + 1] = l + 1 < L ? v.w : 0u; }
      }
    } else {
#pragma unroll
      for (int l = 0; l < LP; ++l) {
        mlo[l] = l < L ? __ldg(src + l * wpl) : 0u;
        mhi[l] = (l < L && wpl > 1) ? __ldg(src + l * wpl + 1) : 0u;
      }
    }
    vote1d_frame<LP>(pd, mlo, mhi, sg, sinv_s, ent_s[warp], q, dw, frame, detect, rcount, slots, list_cap);
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------
// K3 for D == 3 with small vote regions (c3: region = one dim-0 plane of N1 x N2 = 128 x 32
// locations): one WARP per region (frame, i0), no CTA barrier.  Identity I1 (Props. 3-4,
// P:437-450): abar[i] = sum_l c_l[M_l(i)]; with k_etab's expansions E[frame][l][k0][k1][w]
// (the last-dim masks of the set buckets of bucket row (k0, k1), OR-ed) the votes of the 32
// locations of detection word (i0, i1, w) in loop l are ONE word,
// E[frame][l][k0_l(i0)][k1_l(i1)][w], k_d = floor(B_d [sigma_{l,d} i_d]_{N_d} / N_d) (Def. 3).
// Lanes take consecutive words (coalesced detection stores); MODE 0 ANDs the L words
// (mu = L), 1 ORs them (mu = 1), 2 counts them in bit-sliced planes and tests >= mu
// (Alg. 1 l.11-14).  The L loads of a word are independent (all in flight).
// Outputs: detection words, and (list mode) the region count + ascending local index list.
// ------------------------------------------------------------------------------------

// Issue the copies of region r's E blocks (one dim-0 bucket per loop, rw words each) into the
// warp's shared buffer dst (cp.async: no registers held, completion by commit group).
__device__ __forceinline__ void v3_issue(const PlanDev& pd, const int* s0, int64_t r, int64_t slab, int64_t d0b,
                                         int L, int B0, int rw, int lgrw, uint32_t n0m, int lga0, int lane,
                                         uint32_t dst) {
  const int64_t frame = r / slab, i0 = d0b + (r - frame * slab);
  const uint32_t* et = pd.etab + (size_t)frame * L * B0 * rw;
  if ((rw & 3) == 0) {                               // 16-B pieces: one per lane at c3 (L rw = 128)
    const int lg4 = lgrw - 2;
    for (int j = lane; j < (L * rw) >> 2; j += 32) {
      const int l = j >> lg4, q = j & ((rw >> 2) - 1);
      const int k0 = (int)((((uint32_t)s0[l] * (uint32_t)i0) & n0m) >> lga0);
      v3_cp16(dst + 16u * j, et + ((size_t)l * B0 + k0) * rw + 4 * q);
    }
  } else {
    for (int j = lane; j < L * rw; j += 32) {
      const int l = j >> lgrw, q = j & (rw - 1);
      const int k0 = (int)((((uint32_t)s0[l] * (uint32_t)i0) & n0m) >> lga0);
      v3_cp4(dst + 4u * j, et + ((size_t)l * B0 + k0) * rw + q);
    }
  }
}

// IT > 0: the region's items fit IT passes of 32 (c3: 4 passes).  The word offset of every
// (pass, loop) lookup, l rw + k1_l(i1) W + w, does not depend on the region (sigma_{l,1} is per
// loop), so each lane computes its IT x LP byte offsets once per kernel and keeps them in
// registers: a lookup is then an add + a shared load, with no per-lookup branch (the index
// arithmetic was 53 % of the kernel's instructions, ncu `profiles/r02c_c3_k_vote3d_before.lines.txt`).
template <int LP, int MODE, int IT>
__global__ void __launch_bounds__(256) k_vote3d(PlanDev pd, int64_t batch, int64_t d0b, int64_t d0e,
                                                 uint32_t* __restrict__ detect, unsigned long long* __restrict__ rcount,
                                                 uint32_t* __restrict__ slots, int list_cap) {
  pdl_enter();
  __shared__ int s0[LP], s1[LP];
  extern __shared__ __align__(16) uint32_t v3s[];    // per warp: two buffers of the region's E rows [L][B1][W]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int L = pd.L, B0 = pd.b[0], B1 = pd.b[1], W = pd.n[2] >> 5, N1 = pd.n[1];
  const int rw = B1 * W, lgrw = __ffs(rw) - 1;       // words per (loop, k0) E block
  const int ew = L * rw;                             // words per buffer
  uint32_t* es0 = v3s + (size_t)warp * 2 * ew;
  const uint32_t sa0 = smem_u32(es0);
  const uint32_t n0m = (uint32_t)(pd.n[0] - 1), n1m = (uint32_t)(N1 - 1);
  const int lga0 = pd.lga[0], lga1 = pd.lga[1];
  for (int l = threadIdx.x; l < LP; l += blockDim.x) {
    s0[l] = l < L ? pd.loops[l].sig[0] : 0;
    s1[l] = l < L ? pd.loops[l].sig[1] : 0;
  }
  __syncthreads();
  int sg1[LP];
#pragma unroll
  for (int l = 0; l < LP; ++l) sg1[l] = s1[l];
  const int64_t slab = d0e - d0b;
  const int64_t nregions = batch * slab;
  const int items = N1 * W;                          // detection words per region
  const int lgW = __ffs(W) - 1;
  const int64_t slab_words = slab * items;
  const int mu = pd.mu;
  // byte offsets of the (pass, loop) lookups in the warp's E buffer, constant over regions;
  // loops l >= L read word 0 and are neutralised by pad masks (no per-lookup branch)
  uint32_t offs[IT > 0 ? IT : 1][LP];
  uint32_t pad[LP];
#pragma unroll
  for (int l = 0; l < LP; ++l) pad[l] = l < L ? 0u : 0xffffffffu;
  if constexpr (IT > 0) {
#pragma unroll
    for (int iq = 0; iq < IT; ++iq) {
      const uint32_t it = (uint32_t)(iq * 32 + lane), i1 = it >> lgW, w = it & (uint32_t)(W - 1);
#pragma unroll
      for (int l = 0; l < LP; ++l)
        offs[iq][l] = l < L ? 4u * ((uint32_t)(l * rw) + ((((uint32_t)sg1[l] * i1) & n1m) >> lga1) * W + w) : 0u;
    }
  }
  // the L words of detection word it (and the second stage on them)
  auto vote_word = [&](const uint32_t* es, const uint32_t (&e)[LP], bool padded) -> uint32_t {
    (void)es;
    uint32_t word = 0u;
    if (MODE == 0) {
      word = 0xffffffffu;
#pragma unroll
      for (int l = 0; l < LP; ++l) if (padded || l < L) word &= e[l];
    } else if (MODE == 1) {
#pragma unroll
      for (int l = 0; l < LP; ++l) word |= e[l];
    } else {
      uint32_t pl[6] = {0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
      for (int l = 0; l < LP; ++l) {
        uint32_t carry = e[l];
#pragma unroll
        for (int b = 0; b < 6; ++b) { const uint32_t t = pl[b] & carry; pl[b] ^= carry; carry = t; }
      }
      uint32_t gt = 0u, eq = 0xffffffffu;            // bit-sliced count >= mu
#pragma unroll
      for (int b = 5; b >= 0; --b) {
        const uint32_t mb = ((mu >> b) & 1) ? 0xffffffffu : 0u;
        gt |= eq & pl[b] & ~mb;
        eq &= ~(pl[b] ^ mb);
      }
      word = gt | eq;
    }
    return word;
  };
  // detection word store + region-local index list (ascending), run = detections so far
  auto emit = [&](int it, uint32_t word, uint32_t* det, uint32_t* sl, int& run) {
    if (it < items) det[it] = word;
    if (__ballot_sync(0xffffffffu, word != 0u) == 0u) return;   // no detection in these 32 words
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (sl) {
      int q = run + incl - c;
      uint32_t v = word;
      while (v) {
        const int bit = __ffs(v) - 1;
        v &= v - 1;
        if (q < list_cap) sl[q] = (uint32_t)((it << 5) + bit);
        ++q;
      }
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  };
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp, TW = (int64_t)gridDim.x * nwarps;
  // software pipeline: region r + TW's E blocks are in flight (cp.async) while region r votes
  if (gw < nregions) v3_issue(pd, s0, gw, slab, d0b, L, B0, rw, lgrw, n0m, lga0, lane, sa0);
  v3_commit();
  int buf = 0;
  for (int64_t r = gw; r < nregions; r += TW, buf ^= 1) {
    const int64_t frame = r / slab, i0 = d0b + (r - frame * slab);
    if (r + TW < nregions)
      v3_issue(pd, s0, r + TW, slab, d0b, L, B0, rw, lgrw, n0m, lga0, lane, sa0 + 4u * (uint32_t)((buf ^ 1) * ew));
    v3_commit();
    v3_wait1();                                      // this region's group has landed (own copies)
    __syncwarp();                                    // ... and every lane's
    const uint32_t* es = es0 + buf * ew;
    uint32_t* det = detect + (size_t)frame * slab_words + (size_t)(i0 - d0b) * items;
    uint32_t* sl = slots ? slots + (size_t)r * list_cap : nullptr;
    int run = 0;
    if constexpr (IT > 0) {
#pragma unroll
      for (int iq = 0; iq < IT; ++iq) {
        const int it = iq * 32 + lane;
        const uint32_t sb = sa0 + 4u * (uint32_t)(buf * ew);
        uint32_t e[LP];
#pragma unroll
        for (int l = 0; l < LP; ++l) {
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(e[l]) : "r"(sb + offs[iq][l]));
          e[l] = MODE == 0 ? (e[l] | pad[l]) : (e[l] & ~pad[l]);
        }
        const uint32_t word = it < items ? vote_word(es, e, true) : 0u;
        emit(it, word, det, sl, run);
      }
    } else {
      for (int it0 = 0; it0 < items; it0 += 32) {
        const int it = it0 + lane;
        uint32_t word = 0u;
        if (it < items) {
          const uint32_t i1 = (uint32_t)(it >> lgW), w = (uint32_t)(it & (W - 1));
          uint32_t e[LP];
#pragma unroll
          for (int l = 0; l < LP; ++l)
            e[l] = l < L ? es[l * rw + (int)(((((uint32_t)sg1[l] * i1) & n1m) >> lga1) * W + w)] : 0u;
          word = vote_word(es, e, false);
        }
        emit(it, word, det, sl, run);
      }
    }
    if (rcount && lane == 0) rcount[r] = (unsigned long long)run;
    __syncwarp();                                    // every lane done reading buf before it is refilled
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ------------------------------------------------------------------------------------
// K3 for D == 2 (c2/c4 frames): persistent CTAs, one frame per CTA iteration, rows of the
// frame split over the threads (R consecutive rows each).  Identity I1 (Props. 3-4)
// in word-parallel form: for loop l the 32 locations of detection word (i0, w) vote with ONE
// word E[l][k0_l(i0)][w], E[l][k0] = OR of the last-dim masks X[l][k1] of the set buckets
// (k0, k1) of loop l (built per frame from the plan-constant nibble tables: B1/4 lookups per
// word), k0_l(i0) = floor(B0 [sigma_{l,0} i0]_{N0} / N0) (Def. 3).  MODE 0 ANDs the L words
// (mu = L), 1 ORs them (mu = 1), 2 counts in bit-sliced planes and tests >= mu (Alg. 1
// l.11-14).  Each thread writes its rows' detection words (contiguous) and, after a
// block scan of the per-thread popcounts, the frame's ascending local index list; the frame
// count goes to rcount for the offset scan.  4 barriers per frame.
// ------------------------------------------------------------------------------------
template <int LP, int MODE, int R>
__global__ void __launch_bounds__(512) k_vote2d(PlanDev pd, const uint32_t* __restrict__ bitmaps, int64_t batch,
                                                 uint32_t* __restrict__ detect, unsigned long long* __restrict__ rcount,
                                                 uint32_t* __restrict__ slots, int list_cap) {
  pdl_enter();
  extern __shared__ __align__(16) uint32_t v2s[];
  __shared__ int wsum[16];
  __shared__ int s0[LP];
  const int tid = threadIdx.x;
  const int L = pd.L, N0 = pd.n[0], N1 = pd.n[1], B0 = pd.b[0], B1 = pd.b[1], wpl = pd.wpl;
  const int W = N1 >> 5, lgW = __ffs(W) - 1, ng = B1 >> 2, lga0 = pd.lga[0];
  const uint32_t n0m = (uint32_t)(N0 - 1);
  uint32_t* NT = v2s;                                // [L][ng][16][W]
  uint32_t* E = NT + (size_t)L * ng * 16 * W;        // [L][B0][W] (16-B aligned: W % 4 == 0)
  uint32_t* bm = E + (size_t)L * B0 * W;             // [L][wpl]
  {
    const int n4 = (L * ng * 16 * W) >> 2;
    for (int i = tid; i < n4; i += blockDim.x)
      reinterpret_cast<uint4*>(NT)[i] = __ldg(reinterpret_cast<const uint4*>(pd.ntab) + i);
    for (int l = tid; l < LP; l += blockDim.x) s0[l] = l < L ? pd.loops[l].sig[0] : 0;
  }
  __syncthreads();
  int sg0[LP];
#pragma unroll
  for (int l = 0; l < LP; ++l) sg0[l] = s0[l];
  const int lgbw = (__ffs(B0) - 1) + lgW;
  const int mu = pd.mu;
  const int64_t fwords = (int64_t)N0 * W;

  for (int64_t frame = blockIdx.x; frame < batch; frame += gridDim.x) {
    for (int i = tid; i < L * wpl; i += blockDim.x) bm[i] = __ldg(bitmaps + (size_t)frame * L * wpl + i);
    __syncthreads();
    for (int j = tid; j < L * B0 * W; j += blockDim.x) {       // E rows of every dim-0 bucket
      const int l = j >> lgbw, k0 = (j >> lgW) & (B0 - 1), w = j & (W - 1);
      const int flat = k0 * B1;
      const uint32_t* T = NT + (size_t)l * ng * 16 * W + w;
      uint32_t e = 0u;
      if (B1 <= 32) {
        uint32_t pat = (bm[l * wpl + (flat >> 5)] >> (flat & 31)) & (B1 == 32 ? 0xffffffffu : ((1u << B1) - 1u));
        for (int g = 0; g < ng; ++g, pat >>= 4) e |= T[((g << 4) + (pat & 15)) * W];
      } else {
        uint32_t lo = bm[l * wpl + (flat >> 5)], hi = bm[l * wpl + (flat >> 5) + 1];
#pragma unroll
        for (int g = 0; g < 8; ++g, lo >>= 4) e |= T[((g << 4) + (lo & 15)) * W];
#pragma unroll
        for (int g = 8; g < 16; ++g, hi >>= 4) e |= T[((g << 4) + (hi & 15)) * W];
      }
      E[j] = e;
    }
    __syncthreads();
    // vote rows i0 = tid R + r
    uint32_t acc[R][8];
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i0 = tid * R + r;
      uint32_t pl[MODE == 2 ? 8 : 1][MODE == 2 ? 6 : 1];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        acc[r][w] = MODE == 0 ? 0xffffffffu : 0u;
        if constexpr (MODE == 2) {
#pragma unroll
          for (int b = 0; b < 6; ++b) pl[w][b] = 0u;
        }
      }
      if (i0 < N0) {
#pragma unroll
        for (int l = 0; l < LP; ++l) {
          if (l >= L) break;
          const int k0 = (int)((((uint32_t)sg0[l] * (uint32_t)i0) & n0m) >> lga0);
          const uint32_t* er = E + ((size_t)l * B0 + k0) * W;
          uint32_t m[8];
#pragma unroll
          for (int w = 0; w < 8; w += 4) {
            if (w < W) {
              const uint4 v = *reinterpret_cast<const uint4*>(er + w);
              m[w] = v.x; m[w + 1] = v.y; m[w + 2] = v.z; m[w + 3] = v.w;
            } else {
              m[w] = m[w + 1] = m[w + 2] = m[w + 3] = 0u;
            }
          }
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            if (MODE == 0) acc[r][w] &= m[w];
            else if (MODE == 1) acc[r][w] |= m[w];
            else {
              uint32_t carry = m[w];
#pragma unroll
              for (int b = 0; b < 6; ++b) { const uint32_t t = pl[w][b] & carry; pl[w][b] ^= carry; carry = t; }
            }
          }
        }
        if constexpr (MODE == 2) {
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            uint32_t gt = 0u, eq = 0xffffffffu;
#pragma unroll
            for (int b = 5; b >= 0; --b) {
              const uint32_t mb = ((mu >> b) & 1) ? 0xffffffffu : 0u;
              gt |= eq & pl[w][b] & ~mb;
              eq &= ~(pl[w][b] ^ mb);
            }
            acc[r][w] = gt | eq;
          }
        }
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          if (w >= W) acc[r][w] = 0u;
          cnt += __popc(acc[r][w]);
        }
        uint32_t* dst = detect + (size_t)frame * fwords + (size_t)i0 * W;
#pragma unroll
        for (int w = 0; w < 8; w += 4)
          if (w < W) *reinterpret_cast<uint4*>(dst + w) = make_uint4(acc[r][w], acc[r][w + 1], acc[r][w + 2], acc[r][w + 3]);
      } else {
#pragma unroll
        for (int w = 0; w < 8; ++w) acc[r][w] = 0u;
      }
    }
    int total;
    int pos = block_excl_scan(cnt, wsum, &total);
    if (slots && total <= list_cap) {
      uint32_t* sl = slots + (size_t)frame * list_cap;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i0 = tid * R + r;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          uint32_t v = acc[r][w];
          while (v) {
            const int bit = __ffs(v) - 1;
            v &= v - 1;
            sl[pos++] = (uint32_t)(i0 * N1 + (w << 5) + bit);
          }
        }
      }
    }
    if (rcount && tid == 0) rcount[frame] = (unsigned long long)total;
    __syncthreads();                                 // wsum / bm / E reused by the next frame
  }
}

// Exclusive scan of the per-region detection counts in place, in two fully parallel passes
// over tiles of kScanTile counts: k_scan_tiles writes each tile's total; k_scan_apply sums the
// totals of the preceding tiles (block reduce), scans its own tile (coalesced, staged in
// shared memory) and writes the offsets; the last tile writes the grand total to *d_count.
constexpr int kScanTile = 4096;
__global__ void __launch_bounds__(1024) k_scan_tiles(const unsigned long long* __restrict__ counts, int64_t n,
                                                     long long* __restrict__ tile_sum) {
  pdl_enter();
  __shared__ long long red[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  long long s = 0;
#pragma unroll
  for (int j = 0; j < kScanTile / 1024; ++j) {
    const int64_t i = t0 + j * 1024 + t;
    if (i < n) s += (long long)__ldcg(counts + i);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[wid] = s;
  __syncthreads();
  if (wid == 0) {
    long long v = red[lane];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) tile_sum[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(1024) k_scan_apply(unsigned long long* __restrict__ counts, int64_t n,
                                                     const long long* __restrict__ tile_sum,
                                                     long long* __restrict__ d_count) {
  pdl_enter();
  __shared__ unsigned long long tile[kScanTile];
  __shared__ long long part[64];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  constexpr int PER = kScanTile / 1024;
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
#pragma unroll
  for (int j = 0; j < PER; ++j) {                    // coalesced load of the tile
    const int64_t i = t0 + j * 1024 + t;
    tile[j * 1024 + t] = i < n ? __ldcg(counts + i) : 0ull;
  }
  long long before = 0;                              // totals of the preceding tiles
  for (int64_t q = t; q < blockIdx.x; q += 1024) before += __ldcg(tile_sum + q);
#pragma unroll
  for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
  if (lane == 0) part[wid] = before;
  __syncthreads();
  long long carry = 0;
  for (int w = 0; w < 32; ++w) carry += part[w];
  long long v[PER], s = 0;                           // thread t scans tile[t PER .. + PER)
#pragma unroll
  for (int j = 0; j < PER; ++j) { v[j] = (long long)tile[t * PER + j]; s += v[j]; }
  long long incl = s;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const long long u = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += u;
  }
  __syncthreads();                                   // part[] reads of the carry are done
  if (lane == 31) part[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const long long w = part[lane];
    long long wi = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += u;
    }
    part[32 + lane] = wi - w;
    if (lane == 31 && blockIdx.x == gridDim.x - 1) *d_count = carry + wi;
  }
  __syncthreads();
  long long run = carry + part[32 + wid] + incl - s;
#pragma unroll
  for (int j = 0; j < PER; ++j) { tile[t * PER + j] = (unsigned long long)run; run += v[j]; }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int64_t i = t0 + j * 1024 + t;
    if (i < n) counts[i] = tile[j * 1024 + t];
  }
}

// Warp per region (regions of <= 32 x kRwWarpWords detection words): copies the vote's
// region-local index list, or -- when the list overflowed -- re-reads the region's detection
// words in order (warp prefix sums), writing flat indices at the region's offset.
__global__ void __launch_bounds__(256) k_region_write_warp(const uint32_t* __restrict__ det, int64_t rwords,
                                                            const unsigned long long* __restrict__ offsets,
                                                            const long long* __restrict__ d_count, int64_t nregions,
                                                            const uint32_t* __restrict__ slots,
                                                            long long* __restrict__ idx, int64_t capacity,
                                                            int list_cap) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nregions) return;
  const long long run0 = (long long)offsets[r];
  const long long n = (r + 1 < nregions ? (long long)offsets[r + 1] : *d_count) - run0;
  const long long g0 = r * rwords * 32;
  if (slots && n <= list_cap) {
    const uint32_t* sl = slots + (size_t)r * list_cap;
    for (long long i = lane; i < n; i += 32)
      if (run0 + i < capacity) idx[run0 + i] = g0 + (long long)sl[i];
    return;
  }
  const uint32_t* src = det + r * rwords;
  long long run = run0;
  for (int64_t w0 = 0; w0 < rwords; w0 += 32) {
    const int64_t w = w0 + lane;
    uint32_t v = w < rwords ? src[w] : 0u;
    const int c = __popc(v);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    long long q = run + incl - c;
    while (v) {
      const int bit = __ffs(v) - 1;
      v &= v - 1;
      if (q < capacity) idx[q] = g0 + (w << 5) + bit;
      ++q;
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// Few regions with region-local lists (c4 / c2: one region per frame, nregions <= kDirectRegions):
// the scan and the writer in ONE launch.  A CTA of 8 warps takes G = 8 / WPR consecutive regions
// (WPR warps per region: 4 for frames of >= 4096 detection words, 1 otherwise); it sums the raw
// counts of every preceding region itself (block reduce over <= 64 KiB that sit in L2; counts
// stay counts), each region's warps add the counts of the CTA's earlier regions and copy the
// region's list with 4 independent loads in flight per thread (or, after a list overflow, one
// warp re-reads the detection words in order); the last region writes *d_count.  Positions
// depend only on the counts: same output as the two-pass scan + writer (bit-identity test:
// RSFT_NO_SCANWRITE=1 selects that path).
constexpr int64_t kDirectRegions = 8192;
template <int WPR>
__global__ void __launch_bounds__(256) k_region_scan_write(const uint32_t* __restrict__ det, int64_t rwords,
                                                            const unsigned long long* __restrict__ counts,
                                                            long long* __restrict__ d_count, int64_t nregions,
                                                            const uint32_t* __restrict__ slots,
                                                            long long* __restrict__ idx, int64_t capacity,
                                                            int list_cap) {
  constexpr int G = 8 / WPR;                          // regions per CTA (even)
  pdl_enter();
  __shared__ long long red[8];
  __shared__ long long own[G];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * G;
  long long s = 0;
  const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(counts);     // r0 is even
  for (int64_t i = t; i < (r0 >> 1); i += 256) {
    const ulonglong2 v = __ldcg(c2 + i);
    s += (long long)v.x + (long long)v.y;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[wid] = s;
  if (t < G) own[t] = r0 + t < nregions ? (long long)__ldcg(counts + r0 + t) : 0ll;
  __syncthreads();
  const int q = wid / WPR, sub = (wid % WPR) * 32 + lane;
  long long run0 = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) run0 += red[i];
#pragma unroll
  for (int i = 0; i < G; ++i) run0 += i < q ? own[i] : 0ll;
  const int64_t r = r0 + q;
  if (r >= nregions) return;
  const long long n = own[q];
  if (r == nregions - 1 && sub == 0) *d_count = run0 + n;
  const long long g0 = r * rwords * 32;
  if (n <= list_cap) {
    constexpr int S = 32 * WPR;
    const uint32_t* sl = slots + (size_t)r * list_cap;
    for (long long i = sub; i < n; i += 4 * S) {
      uint32_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = i + u * S < n ? __ldcs(sl + i + u * S) : 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * S < n && run0 + i + u * S < capacity) idx[run0 + i + u * S] = g0 + (long long)v[u];
    }
    return;
  }
  if (wid % WPR) return;                             // list overflow: one warp re-reads the words
  const uint32_t* src = det + r * rwords;
  long long run = run0;
  for (int64_t w0 = 0; w0 < rwords; w0 += 32) {
    const int64_t w = w0 + lane;
    uint32_t v = w < rwords ? src[w] : 0u;
    const int c = __popc(v);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    long long qo = run + incl - c;
    while (v) {
      const int bit = __ffs(v) - 1;
      v &= v - 1;
      if (qo < capacity) idx[qo] = g0 + (w << 5) + bit;
      ++qo;
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ------------------------------------------------------------------------------------
// K4 compaction: detection bitmap -> ascending flat indices, single pass.  Chunks of
// kChunkWords words are taken in ticket order (atomic counter), so a chunk's predecessors
// are always resident or done; each chunk publishes its popcount (flag A) and, once its
// exclusive prefix is known from a decoupled look-back, its inclusive prefix (flag P).
// The result is deterministic (positions depend only on the bitmap).
// state[c]: bits 62-63 flag (0 none, 1 aggregate, 2 inclusive), bits 0-61 value.
// ------------------------------------------------------------------------------------
constexpr int kWordsPerThread = (int)(kChunkWords / kThreads);
constexpr unsigned long long kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kThreads) k_compact(const uint32_t* __restrict__ det, int64_t nwords,
                                                      int64_t nchunks, unsigned long long* state,
                                                      unsigned int* ticket, long long* __restrict__ idx,
                                                      int64_t capacity, long long* __restrict__ d_count) {
  pdl_enter();
  __shared__ int s_chunk;
  __shared__ long long s_prefix;
  __shared__ int wsum[kThreads / 32];
  __shared__ long long s_idx[kStageIdx];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_chunk = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t chunk = s_chunk;
  const int64_t base = chunk * kChunkWords + (int64_t)tid * kWordsPerThread;
  uint32_t w[kWordsPerThread];
  int c = 0;
  if (base + kWordsPerThread <= nwords && ((reinterpret_cast<uintptr_t>(det + base) & 15) == 0)) {
#pragma unroll
    for (int i = 0; i < kWordsPerThread; i += 4) {
      uint4 v = *reinterpret_cast<const uint4*>(det + base + i);
      w[i] = v.x; w[i + 1] = v.y; w[i + 2] = v.z; w[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kWordsPerThread; ++i) w[i] = base + i < nwords ? det[base + i] : 0u;
  }
#pragma unroll
  for (int i = 0; i < kWordsPerThread; ++i) c += __popc(w[i]);
  int incl = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int wbase = 0, total = 0;
  for (int i = 0; i < kThreads / 32; ++i) {
    if (i < warp) wbase += wsum[i];
    total += wsum[i];
  }
  if (warp == 0) {                                 // warp-parallel decoupled look-back
    volatile unsigned long long* vs = state;
    long long excl = 0;
    if (chunk == 0) {
      if (lane == 0) atomicExch(&state[0], kFlagP | (unsigned long long)total);
    } else {
      if (lane == 0) atomicExch(&state[chunk], kFlagA | (unsigned long long)total);
      int64_t top = chunk - 1;                       // window: predecessors top, top-1, ...
      while (true) {
        const int64_t j = top - lane;
        const unsigned long long v = j >= 0 ? vs[j] : (2ull << 62);
        const unsigned long long f = v & ~kValMask;
        const unsigned pmask = __ballot_sync(0xffffffffu, f == kFlagP);
        const unsigned zmask = __ballot_sync(0xffffffffu, f == 0);
        const int plane = pmask ? __ffs(pmask) - 1 : 31;
        const unsigned need = plane == 31 ? 0xffffffffu : ((2u << plane) - 1u);
        if (zmask & need) continue;                  // a predecessor has not published yet
        long long val = lane <= plane ? (long long)(v & kValMask) : 0;
#pragma unroll
        for (int off = 16; off; off >>= 1) val += __shfl_xor_sync(0xffffffffu, val, off);
        excl += val;
        if (pmask) break;
        top -= 32;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(&state[chunk], kFlagP | (unsigned long long)(excl + total));
      }
    }
    if (lane == 0) {
      s_prefix = excl;
      if (chunk == nchunks - 1) *d_count = excl + total;
    }
  }
  __syncthreads();
  // indices: staged in smem and written coalesced when the chunk's count fits
  const long long cbase = s_prefix;
  if (total <= kStageIdx) {
    int lp = wbase + incl - c;
#pragma unroll
    for (int i = 0; i < kWordsPerThread; ++i) {
      uint32_t v = w[i];
      while (v) {
        int bit = __ffs(v) - 1;
        v &= v - 1;
        s_idx[lp++] = (long long)(base + i) * 32 + bit;
      }
    }
    __syncthreads();
    for (int i = tid; i < total; i += blockDim.x)
      if (cbase + i < capacity) idx[cbase + i] = s_idx[i];
  } else {
    long long pos = cbase + wbase + incl - c;
#pragma unroll
    for (int i = 0; i < kWordsPerThread; ++i) {
      uint32_t v = w[i];
      while (v) {
        int bit = __ffs(v) - 1;
        v &= v - 1;
        if (pos < capacity) idx[pos] = (long long)(base + i) * 32 + bit;
        ++pos;
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// Host launchers
rsft_status launch_compact(rsft_plan_s* p, const uint32_t* det, int64_t batch, int64_t* idx,
                           int64_t capacity, int64_t* d_count, cudaStream_t st);

static int64_t vote_regions_per_frame(const rsft_plan_s* p, int64_t d0b, int64_t d0e) {
  return p->D == 3 ? d0e - d0b : 1;
}

// Shared memory of k_vote and the bitmap slice width lw (words per loop it loads).
static size_t vote_smem(const rsft_plan_s* p, int* lw_out) {
  const int D = p->D;
  const int64_t W = p->n[D - 1] / 32;
  const int64_t brd = D >= 2 ? p->b[D - 2] : 1;
  const int64_t wpl = p->dev.wpl;
  const int64_t rowbits = brd * p->b[D - 1];
  const int lw = (D == 3 && rowbits % 32 == 0) ? (int)(rowbits / 32) : (int)wpl;
  *lw_out = lw;
  const size_t xw = p->dev.xmask ? (size_t)p->L * p->b[D - 1] * W : 0;
  const size_t nt = (p->dev.xmask && p->b[D - 1] >= 4 && 16 * xw <= kMaxNibbleBytes) ? 4 * xw : 0;   // nibble tables
  return (((size_t)p->L * lw + 3) & ~size_t(3)) * 4 + (((size_t)p->L * brd * W + 3) & ~size_t(3)) * 4 +
         kMaxLoops * 4 + ((xw + 3) & ~size_t(3)) * 4 + nt * 4;
}

template <int CW, int MODE, bool COUNT, bool LIST>
static rsft_status launch_vote_t(rsft_plan_s* p, const uint32_t* bm, int64_t batch, int64_t d0b, int64_t d0e,
                                 uint32_t* det, uint8_t* counts, cudaStream_t st) {
  int lw = 0;
  // D == 3: E words of every dim-0 bucket once per frame (k_etab), copied per region (a
  // double-buffered cp.async copy of the next region's rows measured slower at c5: 20 vs 17 us)
  const int use_etab = p->D == 3 && p->dev.etab && p->dev.xmask && batch <= p->dev.etab_frames &&
                       (d0e - d0b) > p->b[0];
  const size_t smem = vote_smem(p, &lw);
  auto kern = k_vote<CW, MODE, COUNT, LIST>;
  rsft_status s = check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  if (s) return s;
  const int64_t np = vote_regions_per_frame(p, d0b, d0e);
  const int64_t nregions = np * batch;
  if (COUNT && nregions > p->dev.region_capacity) return RSFT_E_WORKSPACE;
  int nb = 0;
  s = check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads, smem), "occupancy");
  if (s) return s;
  if (nb < 1) { set_error("k_vote: zero occupancy"); return RSFT_E_UNSUPPORTED; }
  int64_t grid = (int64_t)nb * p->num_sms;
  if (grid > nregions) grid = nregions;
  if (use_etab)
    if ((s = launch_etab(p, bm, batch, st))) return s;
  if (cudaError_t le_ = pdl_launch(kern, (unsigned)grid, kThreads, smem, st, p->dev, bm, d0b, d0e, lw, np, nregions, det, counts,
                                               p->dev.region_state, use_etab); le_ != cudaSuccess)
    return check(le_, "kern launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_vote launch");
}

template <bool COUNT, bool LIST>
static rsft_status launch_vote_mode(rsft_plan_s* p, const uint32_t* bm, int64_t batch, int64_t d0b, int64_t d0e,
                                    uint32_t* det, uint8_t* counts, cudaStream_t st) {
  const int64_t W = p->n[p->D - 1] / 32;
  const int mode = (!counts && p->mu == p->L) ? 0 : (!counts && p->mu == 1) ? 1 : 2;
#define RSFT_VOTE_CASE(CWV, MV) \
  if (W % CWV == 0 && mode == MV) return launch_vote_t<CWV, MV, COUNT, LIST>(p, bm, batch, d0b, d0e, det, counts, st);
  RSFT_VOTE_CASE(8, 0) RSFT_VOTE_CASE(8, 1)
  RSFT_VOTE_CASE(4, 0) RSFT_VOTE_CASE(4, 1) RSFT_VOTE_CASE(4, 2)
  RSFT_VOTE_CASE(2, 0) RSFT_VOTE_CASE(2, 1) RSFT_VOTE_CASE(2, 2)
  RSFT_VOTE_CASE(1, 0) RSFT_VOTE_CASE(1, 1) RSFT_VOTE_CASE(1, 2)
#undef RSFT_VOTE_CASE
  return RSFT_E_UNSUPPORTED;
}

// D == 1 warp-per-frame vote (k_vote1d): full range, no abar output, frame words in smem.
bool vote1d_usable(const rsft_plan_s* p) {
  const char* off = getenv("RSFT_NO_VOTE1D");
  if (off && off[0] && off[0] != '0') return false;
  return p->D == 1 && p->n[0] >= 32 && p->n[0] <= 32768 && p->L <= 32 && p->b[0] <= 64;
}

static bool vote1d_ok(const rsft_plan_s* p, uint8_t* counts) {   // RSFT_NO_VOTE1D read per launch
  return !counts && vote1d_usable(p);             // the masks of one loop are 64-bit (B <= 64)
}

static rsft_status launch_vote1d(rsft_plan_s* p, const uint32_t* bm, int64_t batch, uint32_t* det,
                                 unsigned long long* rcount, uint32_t* slots, int list_cap, cudaStream_t st) {
  const size_t smem = (size_t)kVote1dWarps * (p->n[0] / 32) * 4;
  // L <= 8: the register-capped build (40 registers, 6 CTAs of 8 warps per SM): c1 step 0.978 vs
  // 1.001 ms with the uncapped one (89 registers, 2 CTAs/SM); RSFT_VOTE1D_OCC=1 selects the latter
  const char* oc = getenv("RSFT_VOTE1D_OCC");
  const bool cap = !(oc && oc[0] == '1') && p->L <= 8;
  auto kern = cap ? k_vote1d<8, 6> : p->L <= 8 ? k_vote1d<8> : p->L <= 16 ? k_vote1d<16> : k_vote1d<32>;
  rsft_status s = check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  if (s) return s;
  int nb = 0;
  s = check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * kVote1dWarps, smem), "occupancy");
  if (s) return s;
  if (nb < 1) { set_error("k_vote1d: zero occupancy"); return RSFT_E_UNSUPPORTED; }
  int64_t grid = (int64_t)nb * p->num_sms;
  const int64_t need = (batch + kVote1dWarps - 1) / kVote1dWarps;
  if (grid > need) grid = need;
  if (cudaError_t le_ = pdl_launch(kern, (unsigned)grid, 32 * kVote1dWarps, smem, st, p->dev, bm, batch, det, rcount, slots,
                                   list_cap); le_ != cudaSuccess)
    return check(le_, "k_vote1d launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_vote1d launch");
}

// D == 3 warp-per-region vote (k_vote3d) on the k_etab expansions: small regions, no abar.
static bool vote3d_ok(const rsft_plan_s* p, int64_t batch, int64_t d0b, int64_t d0e, uint8_t* counts) {
  const char* off = getenv("RSFT_NO_VOTE3D");        // read per launch: tests select either kernel
  if (off && off[0] && off[0] != '0') return false;
  const char* on = getenv("RSFT_VOTE3D");            // force for larger planes (measurement)
  const int64_t lim = on && on[0] == '1' ? (int64_t)1 << 20 : 256;
  return p->D == 3 && !counts && p->dev.etab && p->dev.xmask && batch <= p->dev.etab_frames &&
         (d0e - d0b) > p->b[0] && p->n[1] * (p->n[2] / 32) <= lim && p->L <= 32 &&
         16 * p->L * p->b[1] * (p->n[2] / 32) * 4 <= 192 * 1024;
}

static rsft_status launch_vote3d(rsft_plan_s* p, const uint32_t* bm, int64_t batch, int64_t d0b, int64_t d0e,
                                 uint32_t* det, unsigned long long* rcount, uint32_t* slots, int list_cap,
                                 cudaStream_t st) {
  if (rsft_status es = launch_etab(p, bm, batch, st)) return es;
  const int mode = p->mu == p->L ? 0 : p->mu == 1 ? 1 : 2;
  const int lp = p->L <= 8 ? 8 : p->L <= 16 ? 16 : 32;
  void (*kern)(PlanDev, int64_t, int64_t, int64_t, uint32_t*, unsigned long long*, uint32_t*, int) = nullptr;
  // precomputed-offset passes (IT) when a region's words fit IT passes of 32 (IT L <= 32 offsets
  // per lane); RSFT_VOTE3D_PK=0 (read per launch) keeps the per-lookup index arithmetic
  const int64_t items = p->n[1] * (p->n[2] / 32);
  const char* pke = getenv("RSFT_VOTE3D_PK");
  const bool pk = !(pke && pke[0] == '0') && (lp == 8 ? items <= 128 : lp == 16 && items <= 64);   // <= 32 offsets per lane
  const int it = !pk ? 0 : items <= 32 ? 1 : items <= 64 ? 2 : 4;
#define RSFT_V3(LPV, MV, ITV) if (lp == LPV && mode == MV && it == ITV) kern = k_vote3d<LPV, MV, ITV>;
  RSFT_V3(8, 0, 0) RSFT_V3(8, 1, 0) RSFT_V3(8, 2, 0) RSFT_V3(16, 0, 0) RSFT_V3(16, 1, 0) RSFT_V3(16, 2, 0)
  RSFT_V3(32, 0, 0) RSFT_V3(32, 1, 0) RSFT_V3(32, 2, 0)
  RSFT_V3(8, 0, 1) RSFT_V3(8, 1, 1) RSFT_V3(8, 2, 1) RSFT_V3(16, 0, 1) RSFT_V3(16, 1, 1) RSFT_V3(16, 2, 1)
  RSFT_V3(8, 0, 2) RSFT_V3(8, 1, 2) RSFT_V3(8, 2, 2) RSFT_V3(16, 0, 2) RSFT_V3(16, 1, 2) RSFT_V3(16, 2, 2)
  RSFT_V3(8, 0, 4) RSFT_V3(8, 1, 4) RSFT_V3(8, 2, 4)
#undef RSFT_V3
  const int64_t nregions = batch * (d0e - d0b);
  int64_t grid = (nregions + 7) / 8;
  if (grid > 16 * (int64_t)p->num_sms) grid = 16 * (int64_t)p->num_sms;
  const size_t smem = (size_t)8 * 2 * p->L * p->b[1] * (p->n[2] / 32) * 4;   // 8 warps x 2 buffers
  rsft_status s = check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  if (s) return s;
  if (cudaError_t le_ = pdl_launch(kern, (unsigned)grid, 256, smem, st, p->dev, batch, d0b, d0e, det, rcount, slots,
                                   list_cap); le_ != cudaSuccess)
    return check(le_, "k_vote3d launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_vote3d launch");
}

// D == 2 persistent CTA-per-frame vote (k_vote2d): full range, no abar, W = N1/32 in {4, 8},
// plan-constant nibble tables available, rows per thread <= 8.
static bool vote2d_ok(const rsft_plan_s* p, int64_t d0b, int64_t d0e, uint8_t* counts) {
  // default for short frames (N0 <= 256; c2: 0.98 vs 1.03 ms per step); at c4 (N0 = 1024) it
  // measured 184-189 us against 129 us for the CTA-per-region k_vote (shared-memory bank
  // conflicts on the random E rows, 2 CTAs/SM), so there it is opt-in.  RSFT_VOTE2D=1 / 0
  // (read per launch) forces it on / off.
  const char* on = getenv("RSFT_VOTE2D");
  if (on && on[0] == '0') return false;
  if (!(on && on[0]) && p->D == 2 && p->n[0] > 256) return false;
  const int64_t W = p->D == 2 ? p->n[1] / 32 : 0;
  return p->D == 2 && !counts && d0b == 0 && d0e == p->n[0] && (W == 4 || W == 8) && p->dev.ntab &&
         p->b[1] >= 4 && p->n[0] <= 4 * 512 && p->L <= 32;
}

static rsft_status launch_vote2d(rsft_plan_s* p, const uint32_t* bm, int64_t batch, uint32_t* det,
                                 unsigned long long* rcount, uint32_t* slots, int list_cap, cudaStream_t st) {
  const int64_t W = p->n[1] / 32, ng = p->b[1] / 4;
  const size_t smem = ((size_t)p->L * ng * 16 * W + (size_t)p->L * p->b[0] * W + (size_t)p->L * p->dev.wpl + 4) * 4;
  const int mode = p->mu == p->L ? 0 : p->mu == 1 ? 1 : 2;
  const int lp = p->L <= 8 ? 8 : p->L <= 16 ? 16 : 32;
  // 4 rows per thread: N0 / 4 threads (a warp at least)
  const int threads = (int)std::max<int64_t>(32, ((p->n[0] / 4 + 31) / 32) * 32);
  void (*kern)(PlanDev, const uint32_t*, int64_t, uint32_t*, unsigned long long*, uint32_t*, int) = nullptr;
#define RSFT_V2(LPV, MV) if (lp == LPV && mode == MV) kern = k_vote2d<LPV, MV, 4>;
  RSFT_V2(8, 0) RSFT_V2(8, 1) RSFT_V2(8, 2) RSFT_V2(16, 0) RSFT_V2(16, 1) RSFT_V2(16, 2)
  RSFT_V2(32, 0) RSFT_V2(32, 1) RSFT_V2(32, 2)
#undef RSFT_V2
  if (!kern) return RSFT_E_UNSUPPORTED;
  rsft_status s = check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  if (s) return s;
  int nb = 0;
  s = check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem), "occupancy");
  if (s) return s;
  if (nb < 1) { set_error("k_vote2d: zero occupancy"); return RSFT_E_UNSUPPORTED; }
  int64_t grid = (int64_t)nb * p->num_sms;
  if (grid > batch) grid = batch;
  if (cudaError_t le_ = pdl_launch(kern, (unsigned)grid, (unsigned)threads, smem, st, p->dev, bm, batch, det, rcount, slots,
                                   list_cap); le_ != cudaSuccess)
    return check(le_, "k_vote2d launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_vote2d launch");
}

rsft_status launch_detect(rsft_plan_s* p, const uint32_t* bm, int64_t batch, int64_t d0b, int64_t d0e,
                          uint32_t* det, uint8_t* counts, cudaStream_t st) {
  if (vote1d_ok(p, counts)) return launch_vote1d(p, bm, batch, det, nullptr, nullptr, 0, st);
  if (vote2d_ok(p, d0b, d0e, counts)) return launch_vote2d(p, bm, batch, det, nullptr, nullptr, 0, st);
  if (vote3d_ok(p, batch, d0b, d0e, counts)) return launch_vote3d(p, bm, batch, d0b, d0e, det, nullptr, nullptr, 0, st);
  return launch_vote_mode<false, false>(p, bm, batch, d0b, d0e, det, counts, st);
}

// vote (+ per-region counts) -> offset scan -> per-region sorted index writes
rsft_status launch_scan_write(rsft_plan_s* p, int64_t batch, uint32_t* det, int64_t* idx, int64_t capacity,
                              int64_t* d_count, bool list, cudaStream_t st);

rsft_status launch_detect_compact(rsft_plan_s* p, const uint32_t* bm, int64_t batch, uint32_t* det,
                                  int64_t* idx, int64_t capacity, int64_t* d_count, cudaStream_t st) {
  const int64_t n0 = p->n[0];
  // region-local index lists when a region's items fit the registers (LIST): the writer then
  // copies the lists instead of re-reading the detection bitmap
  const int D = p->D;
  const int64_t W = p->n[D - 1] / 32;
  const int mode = p->mu == p->L ? 0 : p->mu == 1 ? 1 : 2;
  const int64_t cw = (W % 8 == 0 && mode != 2) ? 8 : W % 4 == 0 ? 4 : W % 2 == 0 ? 2 : 1;
  const int64_t rows = D == 3 ? p->n[1] : D == 2 ? n0 : 1;
  const bool v1 = vote1d_ok(p, nullptr);
  const bool v3 = !v1 && vote3d_ok(p, batch, 0, n0, nullptr);
  const bool v2 = !v1 && !v3 && vote2d_ok(p, 0, n0, nullptr);
  {
    // RSFT_COMPACT=1 (read per launch): plain vote, then the single-pass look-back compaction
    // of the detection words (k_compact) instead of per-region counts / lists + scan + writer
    const char* cm = getenv("RSFT_COMPACT");
    if (cm && cm[0] == '1') {
      rsft_status s = launch_detect(p, bm, batch, 0, n0, det, nullptr, st);
      if (s) return s;
      return launch_compact(p, det, batch, idx, capacity, d_count, st);
    }
  }
  const bool list = p->dev.region_slots && (v1 || v2 || v3 || rows * (W / cw) <= (int64_t)kListIpt * kThreads);
  const int64_t np = vote_regions_per_frame(p, 0, n0);
  const int64_t nregions = np * batch;
  if (nregions > p->dev.region_capacity) return RSFT_E_WORKSPACE;
  rsft_status s = v1 ? launch_vote1d(p, bm, batch, det, p->dev.region_state, list ? p->dev.region_slots : nullptr,
                                     (int)p->dev.list_cap, st)
                : v3 ? launch_vote3d(p, bm, batch, 0, n0, det, p->dev.region_state, list ? p->dev.region_slots : nullptr,
                                     (int)p->dev.list_cap, st)
                : v2 ? launch_vote2d(p, bm, batch, det, p->dev.region_state, list ? p->dev.region_slots : nullptr,
                                     (int)p->dev.list_cap, st)
                : list ? launch_vote_mode<true, true>(p, bm, batch, 0, n0, det, nullptr, st)
                       : launch_vote_mode<true, false>(p, bm, batch, 0, n0, det, nullptr, st);
  if (s) return s;
  return launch_scan_write(p, batch, det, idx, capacity, d_count, list, st);
}


rsft_status launch_compact(rsft_plan_s* p, const uint32_t* det, int64_t batch, int64_t* idx,
                           int64_t capacity, int64_t* d_count, cudaStream_t st) {
  const int64_t nwords = batch * ((p->ntot + 31) / 32);
  const int64_t nchunks = (nwords + kChunkWords - 1) / kChunkWords;
  if (nchunks > p->dev.chunk_capacity) return RSFT_E_WORKSPACE;
  unsigned long long* state = reinterpret_cast<unsigned long long*>(p->dev.chunk_counts);
  unsigned int* ticket = reinterpret_cast<unsigned int*>(state + nchunks);
  rsft_status s = check(cudaMemsetAsync(state, 0, (size_t)(nchunks + 1) * 8, st), "compaction state reset");
  if (s) return s;
  if (cudaError_t le_ = pdl_launch(k_compact, (unsigned)nchunks, kThreads, 0, st, det, nwords, nchunks, state, ticket,
                                                   reinterpret_cast<long long*>(idx), capacity,
                                                   reinterpret_cast<long long*>(d_count)); le_ != cudaSuccess)
    return check(le_, "k_compact launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_compact launch");
}



// Offsets of the per-region detection counts (two-pass parallel scan) + the sorted index list
// writer (region lists, or the detection words when a list overflowed / is absent).
rsft_status launch_scan_write(rsft_plan_s* p, int64_t batch, uint32_t* det, int64_t* idx, int64_t capacity,
                              int64_t* d_count, bool list, cudaStream_t st) {
  const int64_t n0 = p->n[0];
  const int64_t np = vote_regions_per_frame(p, 0, n0);
  const int64_t nregions = np * batch;
  const int64_t rwords = ((p->ntot + 31) / 32) / np;
  const char* nsw = getenv("RSFT_NO_SCANWRITE");     // read per launch: tests select either path
  if (list && nregions <= kDirectRegions && !(nsw && nsw[0] == '1')) {
    // 4 warps per region list for large frames (c4: 15 vs 20 us); at c2's 2048-word frames one warp
    // per region measured faster (17 vs 21 us)
    const bool wide = rwords >= 4096;
    cudaError_t le_ = wide
        ? pdl_launch(k_region_scan_write<4>, (unsigned)((nregions + 1) / 2), 256, 0, st, det, rwords,
                     p->dev.region_state, reinterpret_cast<long long*>(d_count), nregions, p->dev.region_slots,
                     reinterpret_cast<long long*>(idx), capacity, (int)p->dev.list_cap)
        : pdl_launch(k_region_scan_write<1>, (unsigned)((nregions + 7) / 8), 256, 0, st, det, rwords,
                     p->dev.region_state, reinterpret_cast<long long*>(d_count), nregions, p->dev.region_slots,
                     reinterpret_cast<long long*>(idx), capacity, (int)p->dev.list_cap);
    if (le_ != cudaSuccess) return check(le_, "k_region_scan_write launch");
    p->last_launches += 1;
    return check(cudaGetLastError(), "k_region_scan_write launch");
  }
  {
    const int64_t ntiles = (nregions + kScanTile - 1) / kScanTile;
    if (ntiles > p->dev.chunk_capacity) return RSFT_E_WORKSPACE;
    long long* tsum = p->dev.chunk_counts;
    if (cudaError_t le_ = pdl_launch(k_scan_tiles, (unsigned)ntiles, 1024, 0, st, p->dev.region_state, nregions, tsum); le_ != cudaSuccess)
      return check(le_, "k_scan_tiles launch");
    if (cudaError_t le_ = pdl_launch(k_scan_apply, (unsigned)ntiles, 1024, 0, st, p->dev.region_state, nregions, tsum,
                                     reinterpret_cast<long long*>(d_count)); le_ != cudaSuccess)
      return check(le_, "k_scan_apply launch");
    p->last_launches += 1;
  }
  // small regions (c1: one 4096-location frame, c3: one dim-0 plane): a warp per region
  const bool warp_writer = rwords <= 1024;
  if (warp_writer) {
    if (cudaError_t le_ = pdl_launch(k_region_write_warp, (unsigned)((nregions + 7) / 8), 256, 0, st, det, rwords, p->dev.region_state,
                                     reinterpret_cast<long long*>(d_count), nregions, list ? p->dev.region_slots : nullptr,
                                     reinterpret_cast<long long*>(idx), capacity, (int)p->dev.list_cap); le_ != cudaSuccess)
      return check(le_, "k_region_write_warp launch");
  } else if (cudaError_t le_ = pdl_launch(k_region_write, (unsigned)nregions, kThreads, 0, st, det, rwords, p->dev.region_state,
                                                          reinterpret_cast<long long*>(d_count), nregions,
                                                          list ? p->dev.region_slots : nullptr,
                                                          reinterpret_cast<long long*>(idx), capacity, (int)p->dev.list_cap); le_ != cudaSuccess)
    return check(le_, "k_region_write launch");
  p->last_launches += 2;
  return check(cudaGetLastError(), "region scan/write launch");
}

}  // namespace rsft
