// Fused D = 2 path of rsft_run (c2 / c4 frames) for sm_100a: ONE warp-specialised persistent
// kernel runs both stages of Alg. 1 per frame.
//
//   fold warps (kF2vFold): pre-window + permutation + flat window + aliasing of every loop in one
//     pass over x (Alg. 1 l.5-8; Eqs. z, l P:269-279; factored form I3), exactly as
//     k_fused streams a frame: per-warp TMA rings of U-row boxes of one residue class, FFMA2
//     folds against the class-major row weights, the column weights + lane fold once per class.
//     The per-class residue sums go to a double-buffered shared slot F[fi & 1]; the warps then
//     go straight on to the next frame (mbarriers Ffull / Fempty).  No CTA barrier after the
//     prologue: the TMA stream never waits for an epilogue.
//   epilogue warps (NE): per frame, per loop: the residue -> bucket permutation with the
//     half-bucket twiddles (L1), the B0 x B1 FFT (Alg. 1 l.9) with one bucket row per lane
//     (dim 1 in registers, dim 0 across the lanes with xor shuffles), |f|^2 > gamma_l and the
//     bitmap words (l.10; Eq. tpd); then the D = 2 vote of the frame (l.11-14,
//     P:226-229; identity I1, Props. 3-4 P:437-450, as k_vote2d): E rows from the set buckets,
//     the L word lookups per detection word, the detection words, the frame count and its
//     ascending local index list (for the region scan + writer of rsft_detect_compact).
//
// Outputs are those of rsft_execute (bitmaps) + the vote kernels (detection words, counts,
// lists); the FFT runs in a different order than k_fused's shared-memory DIT (same values to
// fp32 rounding: parity is checked against the oracle, not against the other kernel's bits).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "rsft_internal.h"
#include "kcommon.cuh"
#include "hcommon.h"
#include "fold.cuh"

namespace rsft {

__constant__ float2 c_tw2v[128];   // e^{-j 2 pi k / 128} (fp64-rounded at bind)

constexpr int kF2vFold = 8;        // fold warps: 4 of the 32 residue classes of c4 each
constexpr int kF2vEpi = 8;         // epilogue (FFT + threshold + vote) warps: one per loop (L <= 8)
#ifndef RSFT_F2V_U
#define RSFT_F2V_U 16
#endif
constexpr int kF2vU = RSFT_F2V_U;   // rows per TMA box (16: 8 KiB; -DRSFT_F2V_U=4 / 8 are tuning builds, DESIGN 6.7)
constexpr int kF2vFB = 2;          // residue-sum slots F (one slot + 5 ring stages measured slower)
constexpr int kF2vMaxN0 = 1024;    // vote rows per epilogue thread: 32 / NE (N0 <= 1024)

template <int NE>
__device__ __forceinline__ void epi_sync() {
  asm volatile("bar.sync 1, %0;" :: "n"(32 * NE) : "memory");
}

// Shared-memory carve-up (byte offsets), identical on host and device.
struct F2vLayout {
  int ring, bars, F, fslot, tw, rowW, arows, Xs, E, bms, wsum, total;
};
RSFT_HD inline int f2v_align(int v, int a) { return (v + a - 1) / a * a; }
RSFT_HD inline F2vLayout f2v_layout(int S, int L, int LP, int N0, int B0, int B1, int W, int wpl) {
  F2vLayout o;
  int off = 0;
  o.ring = off; off += kF2vFold * S * kF2vU * 512;
  o.bars = off; off += (kF2vFold * S + 4) * 8;
  off = f2v_align(off, 16);
  o.fslot = L * B0 * (B1 + 1);                       // float2 per buffer
  o.F = off; off += kF2vFB * f2v_align(o.fslot, 2) * 8;
  o.tw = off; off += 128 * 8;
  // row weights class-major [B0][A0 rounded up to U][LP] (zero rows pad the last group): the U
  // rows of a box are contiguous, so the fold addresses them with immediate offsets
  o.arows = f2v_align(N0 / B0, kF2vU);
  o.rowW = off; off += B0 * o.arows * LP * 4;
  off = f2v_align(off, 16);
  o.Xs = off; off += L * B1 * W * 4;
  off = f2v_align(off, 16);
  o.E = off; off += f2v_align(L * B0 * W, 4) * 4;
  o.bms = off; off += L * wpl * 4;
  off = f2v_align(off, 16);
  o.wsum = off; off += 64;
  o.total = f2v_align(off, 128);
  return o;
}

template <int LP, int NB1, int MODE, int NE>
__global__ void __launch_bounds__(32 * (kF2vFold + NE), 1) k_fused2v(PlanDev pd, const __grid_constant__ CUtensorMap tmap,
                                                           int64_t batch, int S, uint32_t* __restrict__ bitmaps,
                                                           uint32_t* __restrict__ detect,
                                                           unsigned long long* __restrict__ rcount,
                                                           uint32_t* __restrict__ slots, int list_cap) {
  pdl_enter();
  constexpr int U = kF2vU, NF = kF2vFold, MR = 32 / NE;
  constexpr int LB1 = NB1 == 32 ? 5 : NB1 == 16 ? 4 : NB1 == 8 ? 3 : 2;
  extern __shared__ __align__(128) unsigned char smem[];
  const int L = pd.L, N0 = pd.n[0], N1 = pd.n[1], B0 = pd.b[0], A0 = pd.a[0];
  const int W = N1 >> 5, wpl = pd.wpl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const F2vLayout lay = f2v_layout(S, L, LP, N0, B0, NB1, W, wpl);
  float4* ring = reinterpret_cast<float4*>(smem + lay.ring);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bars);
  uint64_t* Ffull = bars + NF * S;                   // [FB], NF x 32 arrivals per frame
  uint64_t* Fempty = Ffull + 2;                      // [FB], NE x 32 arrivals per frame
  float2* Fbuf = reinterpret_cast<float2*>(smem + lay.F);
  const int fslot = f2v_align(lay.fslot, 2);
  float2* tw = reinterpret_cast<float2*>(smem + lay.tw);
  float* rowW = reinterpret_cast<float*>(smem + lay.rowW);
  uint32_t* Xs = reinterpret_cast<uint32_t*>(smem + lay.Xs);
  uint32_t* E = reinterpret_cast<uint32_t*>(smem + lay.E);
  uint32_t* bms = reinterpret_cast<uint32_t*>(smem + lay.bms);
  int* wsum = reinterpret_cast<int*>(smem + lay.wsum);
  constexpr int fstride = NB1 + 1;

  // prologue: twiddles, class-major row weights (row N0 = zeros), X masks, barriers
  for (int i = tid; i < 128; i += blockDim.x) tw[i] = c_tw2v[i];
  for (int i = tid; i < B0 * lay.arows * LP; i += blockDim.x) {
    const int l = i % LP, a = (i / LP) % lay.arows, kappa = i / (LP * lay.arows);
    const int s0 = kappa + B0 * a;                  // dim-0 sample of row a of class kappa
    rowW[i] = (l < L && a < A0) ? pd.h[0][(size_t)l * N0 + s0] : 0.f;
  }
  for (int i = tid; i < L * NB1 * W; i += blockDim.x) Xs[i] = __ldg(pd.xmask + i);
  if (tid == 0) {
    for (int i = 0; i < NF * S; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < kF2vFB; ++i) { mbar_init(&Ffull[i], NF * 32); mbar_init(&Fempty[i], NE * 32); }
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t nfr = batch > (int64_t)blockIdx.x ? (batch - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp < NF) {
    // ---------------------------------------------------------------- fold warps
    const float* __restrict__ hlast = pd.h[1];
    const int spt = N1 >> 6, lg_spt = __ffs(spt) - 1;        // 64-column segments per class
    const int ntw = warp < B0 ? (B0 - 1 - warp) / NF + 1 : 0;  // classes of this warp
    const int units = ntw * spt;
    const int ngrp = (A0 + U - 1) / U;
    const int64_t total = nfr * units * ngrp;
    float4* myring = ring + (size_t)warp * S * U * 32;
    uint64_t* mybar = bars + warp * S;
    const uint64_t tmap_ptr = reinterpret_cast<uint64_t>(&tmap);
    int p_fi = 0, p_unit = 0, p_grp = 0, p_st = 0;
    int64_t p_left = total;
    auto issue_next = [&]() {
      if (p_left <= 0) return;
      --p_left;
      const int frame = (int)(blockIdx.x + (int64_t)p_fi * gridDim.x);
      mbar_expect_tx(&mybar[p_st], (uint32_t)U * 512u);
      const int kappa = warp + (p_unit >> lg_spt) * NF, seg = p_unit & (spt - 1);
      tma_load_4d(myring + (size_t)p_st * U * 32, tmap_ptr, seg * 64, kappa, p_grp * U, frame, &mybar[p_st]);
      if (++p_st == S) p_st = 0;
      if (++p_grp == ngrp) {
        p_grp = 0;
        if (++p_unit == units) { p_unit = 0; ++p_fi; }
      }
    };
    if (lane == 0)
      for (int j = 0; j < S - 1; ++j) issue_next();
    int c_st = 0;
    uint32_t c_ph = 0;
    const int fold_lanes = NB1 / 2;
    float2 racc[LP][2];
    for (int64_t fi = 0; fi < nfr; ++fi) {
      const int fb = (int)(fi % kF2vFB);
      const uint32_t use = (uint32_t)(fi / kF2vFB);   // this slot's use count
      float2* F = Fbuf + (size_t)fb * fslot;
      bool waited = false;
      for (int unit = 0; unit < units; ++unit) {
        const int kappa = warp + (unit >> lg_spt) * NF, seg = unit & (spt - 1);
        if (seg == 0) {
#pragma unroll
          for (int l = 0; l < LP; ++l) racc[l][0] = racc[l][1] = make_float2(0.f, 0.f);
        }
        float2 acc[LP][2];
#pragma unroll
        for (int l = 0; l < LP; ++l) acc[l][0] = acc[l][1] = make_float2(0.f, 0.f);
        for (int grp = 0; grp < ngrp; ++grp) {
          if (lane == 0) issue_next();
          mbar_wait(&mybar[c_st], c_ph);
          const float* wbase = rowW + ((size_t)kappa * lay.arows + grp * U) * LP;
          const float* wrow[U];
#pragma unroll
          for (int u = 0; u < U; ++u) wrow[u] = wbase + u * LP;
          fold_group<LP, U>(acc, myring + (size_t)c_st * U * 32, lane, wrow);
          __syncwarp();
          if (++c_st == S) { c_st = 0; c_ph ^= 1u; }
        }
        colweight<LP>(acc, hlast, 0, L, N1, seg * 64 + 2 * lane);
#pragma unroll
        for (int l = 0; l < LP; ++l) {
          racc[l][0] = cadd(racc[l][0], acc[l][0]);
          racc[l][1] = cadd(racc[l][1], acc[l][1]);
        }
        if (seg == spt - 1) {
          lane_fold<LP>(racc, NB1);
          if (!waited) {                             // slot fb free: the epilogue gathered frame fi - FB
            mbar_wait(&Fempty[fb], (use & 1u) ^ 1u);
            waited = true;
          }
          if (lane < fold_lanes) {
            float2* slot = F + kappa * fstride + 2 * lane;
#pragma unroll
            for (int l = 0; l < LP; ++l)
              if (l < L) {
                slot[(size_t)l * B0 * fstride] = racc[l][0];
                slot[(size_t)l * B0 * fstride + 1] = racc[l][1];
              }
          }
        }
      }
      if (!waited) mbar_wait(&Fempty[fb], (use & 1u) ^ 1u);   // keeps the Ffull phases in step
      __syncwarp();
      mbar_arrive(&Ffull[fb]);
    }
    return;
  }

  // ------------------------------------------------------------------ epilogue warps
  const int ew = warp - NF, etid = tid - NF * 32;
  const int lgb0 = pd.lgb[0];
  const int b0 = lane & (B0 - 1);                    // this lane's bucket row (lanes >= B0 duplicate)
  float2 stw[5];                                     // cross-lane DIF twiddles W_{2h}^{lane & (h-1)}
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int h = 16 >> q;
    stw[q] = tw[(lane & (h - 1)) * (64 / h)];
  }
  const DifTw dt = dif_tw(lane, stw);
  const float2 h0tw = pd.shift[0] ? tw[b0 * (64 >> lgb0)] : make_float2(1.f, 0.f);   // e^{-j pi b0 / B0}
  const bool shift1 = pd.shift[1] != 0;
  const int rpw = 32 / NB1;                          // bucket rows per bitmap word
  const int lga0 = pd.lga[0], mu = pd.mu;
  const uint32_t n0m = (uint32_t)(N0 - 1);
  const int R = (N0 + NE * 32 - 1) / (NE * 32);      // vote rows per thread (<= MR)
  const int64_t fwords = (int64_t)N0 * W;
  int sg0[LP];
#pragma unroll
  for (int l = 0; l < LP; ++l) sg0[l] = l < L ? pd.loops[l].sig[0] : 0;

  for (int64_t fi = 0; fi < nfr; ++fi) {
    const int64_t frame = blockIdx.x + fi * gridDim.x;
    const int fb = (int)(fi % kF2vFB);
    const float2* F = Fbuf + (size_t)fb * fslot;
    mbar_wait(&Ffull[fb], (uint32_t)((fi / kF2vFB) & 1));
    // one loop per epilogue warp (L <= 8 = NE): gather its bucket rows, then free the slot
    const int l = ew;
    const LoopDev lp = pd.loops[l < L ? l : 0];
    float2 v[NB1];
    if (l < L) {
      const int r0 = (lp.sig[0] * b0 + lp.tau[0]) & (B0 - 1);
      const float2* Fr = F + ((size_t)l * B0 + r0) * fstride;
#pragma unroll
      for (int b1 = 0; b1 < NB1; ++b1) v[b1] = Fr[(lp.sig[1] * b1 + lp.tau[1]) & (NB1 - 1)];   // residue -> bucket (I3)
    }
    mbar_arrive(&Fempty[fb]);                        // F[fb] consumed (values in registers)
    if (l < L) {
#pragma unroll
      for (int b1 = 0; b1 < NB1; ++b1) {             // half-bucket twiddles (L1)
        float2 x = v[b1];
        if (shift1) x = cmul(x, c_tw2v[b1 * (64 / NB1)]);
        v[b1] = cmul(x, h0tw);
      }
      // dim 1: in-register radix-2 DIF (natural in, slot s = X[brev(s)])
#pragma unroll
      for (int half = NB1 / 2; half >= 1; half >>= 1)
#pragma unroll
        for (int blk = 0; blk < NB1; blk += 2 * half)
#pragma unroll
          for (int j = 0; j < half; ++j) {
            const float2 a = v[blk + j], b = v[blk + j + half];
            v[blk + j] = cadd(a, b);
            v[blk + j + half] = j == 0 ? csub(a, b) : cmul(csub(a, b), c_tw2v[j * (64 / half)]);
          }
      // dim 0: B0-point DIF across the lanes; lane p then holds bucket row brev(p mod B0)
      uint32_t mask = 0u;
#pragma unroll
      for (int s = 0; s < NB1; ++s) {
        const float2 x = warp_dif(v[s], lgb0, dt);
        if (x.x * x.x + x.y * x.y > lp.gamma) mask |= 1u << brev(s, LB1);
      }
      // bitmap words: word w holds bucket rows w rpw .. w rpw + rpw - 1 (flat k = k0 B1 + k1)
      uint32_t word = 0u;
      for (int q = 0; q < rpw; ++q) {
        const int k0 = lane * rpw + q;
        const uint32_t m = __shfl_sync(0xffffffffu, mask, brev(k0 & (B0 - 1), lgb0));
        if (k0 < B0) word |= NB1 == 32 ? m : (m << (q * NB1));
      }
      if (lane < wpl) {
        bms[l * wpl + lane] = word;
        bitmaps[(size_t)frame * L * wpl + (size_t)l * wpl + lane] = word;
      }
    }
    epi_sync<NE>();
    // E[l][k0][w] = OR of the last-dim masks X[l][k1] of the set buckets (k0, k1) of loop l (I1)
    const int lgW = __ffs(W) - 1;
    for (int j = etid; j < L * B0 * W; j += NE * 32) {
      const int w = j & (W - 1), k0 = (j >> lgW) & (B0 - 1), l = j >> (lgW + lgb0);
      const int flat = k0 * NB1;
      uint32_t pat = (bms[l * wpl + (flat >> 5)] >> (flat & 31)) & (NB1 == 32 ? 0xffffffffu : ((1u << NB1) - 1u));
      uint32_t e = 0u;
      const uint32_t* X = Xs + (size_t)l * NB1 * W + w;
      while (pat) {
        const int k = __ffs(pat) - 1;
        pat &= pat - 1;
        e |= X[k * W];
      }
      E[j] = e;
    }
    epi_sync<NE>();
    // vote rows i0 = etid R + r (Alg. 1 l.11-14)
    uint32_t acc[MR][8];
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int i0 = etid * R + r;
#pragma unroll
      for (int w = 0; w < 8; ++w) acc[r][w] = 0u;
      if (r >= R || i0 >= N0) continue;
      uint32_t pl[MODE == 2 ? 8 : 1][MODE == 2 ? 6 : 1];
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        acc[r][w] = MODE == 0 ? 0xffffffffu : 0u;
        if constexpr (MODE == 2) {
#pragma unroll
          for (int b = 0; b < 6; ++b) pl[w][b] = 0u;
        }
      }
#pragma unroll
      for (int l = 0; l < LP; ++l) {
        if (l >= L) break;
        const int k0 = (int)((((uint32_t)sg0[l] * (uint32_t)i0) & n0m) >> lga0);
        const uint32_t* er = E + ((size_t)l * B0 + k0) * W;
        uint32_t m[8];
#pragma unroll
        for (int w = 0; w < 8; w += 4) {
          if (w < W) {
            const uint4 x = *reinterpret_cast<const uint4*>(er + w);
            m[w] = x.x; m[w + 1] = x.y; m[w + 2] = x.z; m[w + 3] = x.w;
          } else {
            m[w] = m[w + 1] = m[w + 2] = m[w + 3] = 0u;
          }
        }
        uint32_t any = 0u;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          if (MODE == 0) { acc[r][w] &= m[w]; any |= acc[r][w]; }
          else if (MODE == 1) acc[r][w] |= m[w];
          else {
            uint32_t carry = m[w];
#pragma unroll
            for (int b = 0; b < 6; ++b) { const uint32_t t = pl[w][b] & carry; pl[w][b] ^= carry; carry = t; }
          }
        }
        if (MODE == 0 && any == 0u) break;           // unanimity already impossible
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
    }
    // exclusive scan of the per-thread counts over the epilogue warps -> list positions
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += x;
    }
    if (lane == 31) wsum[ew] = incl;
    epi_sync<NE>();
    int pos = incl - cnt, total = 0;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int x = wsum[i];
      if (i < ew) pos += x;
      total += x;
    }
    if (slots && total <= list_cap && cnt) {
      uint32_t* sl = slots + (size_t)frame * list_cap;
#pragma unroll
      for (int r = 0; r < MR; ++r) {
        const int i0 = etid * R + r;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          uint32_t x = acc[r][w];
          while (x) {
            const int bit = __ffs(x) - 1;
            x &= x - 1;
            sl[pos++] = (uint32_t)(i0 * N1 + (w << 5) + bit);
          }
        }
      }
    }
    if (rcount && etid == 0) rcount[frame] = (unsigned long long)total;
    epi_sync<NE>();                                      // bms / E / wsum reused by the next frame
  }
}

rsft_status upload_twiddles_2v(cudaStream_t st) {
  float2 tw[128];
  for (int k = 0; k < 128; ++k) {
    const double a = -2.0 * M_PI * (double)k / 128.0;
    tw[k] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  return check(cudaMemcpyToSymbolAsync(c_tw2v, tw, sizeof(tw), 0, cudaMemcpyHostToDevice, st), "twiddles (2v)");
}

// Shapes the kernel covers: D = 2, all L <= 8 loops, B0 <= 32, B1 in {8, 16, 32}, N1 in {128, 256},
// N0 <= 1024 (vote rows per thread), plan-constant X masks present.
bool fused2v_ok(const rsft_plan_s* p) {
  const char* off = getenv("RSFT_NO_FUSED2V");      // read per launch: tests select either path
  if (off && off[0] && off[0] != '0') return false;
  if (p->D != 2 || p->L > 8 || !p->dev.xmask) return false;
  const int64_t B0 = p->b[0], B1 = p->b[1], N0 = p->n[0], N1 = p->n[1];
  if (B0 < 2 || B0 > 32 || !(B1 == 8 || B1 == 16 || B1 == 32)) return false;
  if (N1 < 128 || N1 > 256 || N0 > kF2vMaxN0) return false;   // W = N1 / 32 in {4, 8}: 16-B E rows
  return true;
}

rsft_status fold_map(const rsft_plan_s* p, const void* d_x, int64_t batch, int64_t n0, CUtensorMap* m, int u,
                     int64_t frame_stride);   // kernels.cu

template <int LP, int NB1, int MODE, int NE>
static rsft_status launch_f2v_t(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm, uint32_t* det,
                                unsigned long long* rcount, uint32_t* slots, int list_cap, cudaStream_t st) {
  auto kern = k_fused2v<LP, NB1, MODE, NE>;
  const int W = (int)(p->n[1] / 32);
  int S = 0;
  const char* es = getenv("RSFT_F2V_STAGES");
  // ring depth per fold warp: 3 stages (2 boxes = 8 KiB ahead per warp, 64 KiB in flight per SM) measured
  // best -- c4 1.379 ms per step vs 1.399 (4 stages, the most that fit) and 1.436 (2); c2 0.728 vs 0.764
  // and 0.794 (DESIGN 6.7); the read-only TMA microbenchmark peaks at ~49 KiB in flight per SM too
  // With 16-row (8-KiB) boxes, 2 stages (one box ahead per warp, the same 64 KiB in flight, half the box issues
  // and waits): c4 1.378 ms, c2 0.710 ms (4-row boxes: 1.50 / 0.89 ms).
  const int smax = es && es[0] ? std::max(2, atoi(es)) : (kF2vU >= 16 ? 2 : 3);
  for (int s = smax; s >= 2; --s)
    if (f2v_layout(s, p->L, LP, (int)p->n[0], (int)p->b[0], NB1, W, p->dev.wpl).total <= 227 * 1024) { S = s; break; }
  if (!S) return RSFT_E_UNSUPPORTED;
  const size_t smem = f2v_layout(S, p->L, LP, (int)p->n[0], (int)p->b[0], NB1, W, p->dev.wpl).total;
  CUtensorMap tmap;
  rsft_status s = fold_map(p, d_x, batch, p->n[0], &tmap, kF2vU, 0);
  if (s) return s;
  s = check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr (2v)");
  if (s) return s;
  const int64_t grid = std::min<int64_t>(batch, p->num_sms);
  if (cudaError_t e = pdl_launch(kern, (unsigned)grid, 32 * (kF2vFold + NE), smem, st, p->dev, tmap, batch, S, bm, det, rcount,
                                 slots, list_cap); e != cudaSuccess)
    return check(e, "k_fused2v launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_fused2v launch");
}

// rsft_run on a fused2v_ok plan: bitmaps, detection words, per-frame counts + local lists.
rsft_status launch_fused2v(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm, uint32_t* det,
                           unsigned long long* rcount, uint32_t* slots, int list_cap, cudaStream_t st) {
  const int lp = p->L <= 6 ? 6 : 8;
  const int mode = p->mu == p->L ? 0 : p->mu == 1 ? 1 : 2;
  // 8 epilogue warps, one loop each (4 measured slower: c4 1.420 vs 1.404 ms per step; c2 1.054 vs
  // 0.757 ms, where 4 warps took longer per frame than the fold)
#define RSFT_F2V(LPV, B1V, MV) \
  if (lp == LPV && p->b[1] == B1V && mode == MV) \
    return launch_f2v_t<LPV, B1V, MV, kF2vEpi>(p, d_x, batch, bm, det, rcount, slots, list_cap, st);
#define RSFT_F2V_M(LPV, B1V) RSFT_F2V(LPV, B1V, 0) RSFT_F2V(LPV, B1V, 1) RSFT_F2V(LPV, B1V, 2)
  RSFT_F2V_M(6, 8) RSFT_F2V_M(6, 16) RSFT_F2V_M(6, 32)
  RSFT_F2V_M(8, 8) RSFT_F2V_M(8, 16) RSFT_F2V_M(8, 32)
#undef RSFT_F2V_M
#undef RSFT_F2V
  return RSFT_E_UNSUPPORTED;
}

}  // namespace rsft
