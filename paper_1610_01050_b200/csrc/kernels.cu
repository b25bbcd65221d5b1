// RSFT hot-path kernels for sm_100a (B200).  Hand-written CUDA; no cuFFT, no libraries.
//
//   K1 fold   : pre-window + permutation + flat window + aliasing, all L loops in ONE coalesced
//               pass over x (factored form I3): per element and loop one
//               complex x real FMA; permutation costs no data movement (identity I2).
//               Alg. 1 l.5-8; Defs. 1-2; Eqs. z, l.
//   K2 FFT    : half-bucket twiddle + B-point N-D FFT in registers + |.|^2 + NP threshold +
//               warp ballot -> bitmaps.  Alg. 1 l.9-10; Eq. tpd.
//   K3 vote   : reverse mapping + accumulation + second stage, word-parallel (32 locations
//               per lane-op) with bit-sliced counters.  Alg. 1 l.11-14; Def. 4;
//               Eq. a_i; identity I1 (Props. 3-4).
//   K4 compact: detection bitmap -> sorted flat index list (popc + scans).
//
// Fused mode (D <= 2, many frames): K1 + K2 in one persistent kernel, one CTA per frame;
// the [L][B] buckets never leave shared memory.  Split mode (D >= 2, big frames): K1 per
// (frame, outer residue class) + an outer-dimension FFT kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <string>

#include "rsft_internal.h"
#include "kcommon.cuh"
#include "hcommon.h"
#include "vote1d.cuh"
#include "fold.cuh"

namespace rsft {

__constant__ float2 c_tw128[128];   // e^{-j 2 pi k / 128}, k < 128 (fp64-rounded at bind)
__constant__ float2 c_tw512[512];   // e^{-j 2 pi k / 512}, k < 512 (k_gather1d with B_0 > 64)

// Multi-axis view of a shared-memory array: element (i_0, ..., i_{k-1}) lives at
// sum_a i_a * st[a].  Axis 0 (loops) may have any size; axes >= 1 are powers of two.
struct View {
  int k;
  int n[4], lg[4], st[4];
};

// In-place radix-2 DIT FFT along axis a (forward e^{-j...}, unnormalised; reading L7) of a
// View whose axis-a data is in bit-reversed order; output natural order.  Stage-parallel:
// every thread of the CTA takes butterflies of every line, one __syncthreads per stage.
// tw = shared copy of e^{-j 2 pi k / 128}.
__device__ __noinline__ void fft_axis(float2* A, const View v, int a, const float2* __restrict__ tw) {
  const int lgn = v.lg[a];
  if (lgn == 0) return;
  int lines = 1;
  for (int i = 0; i < v.k; ++i) if (i != a) lines *= v.n[i];
  const int nbf = lines << (lgn - 1);
  const int sa = v.st[a];
  for (int s = 1; s <= lgn; ++s) {
    const int half = 1 << (s - 1);
    for (int bf = threadIdx.x; bf < nbf; bf += blockDim.x) {
      int j = bf & (half - 1);
      int g = (bf >> (s - 1)) & ((1 << (lgn - s)) - 1);
      int rest = bf >> (lgn - 1);
      int off = 0;
      for (int i = v.k - 1; i >= 1; --i) {
        if (i == a) continue;
        off += (rest & (v.n[i] - 1)) * v.st[i];
        rest >>= v.lg[i];
      }
      off += rest * v.st[0];
      float2* e0 = A + off + ((g << s) + j) * sa;
      float2* e1 = e0 + half * sa;
      float2 u = *e0;
      float2 t = cmul(tw[j << (7 - s)], *e1);
      *e0 = cadd(u, t);
      *e1 = csub(u, t);
    }
    __syncthreads();
  }
}

// Stage-parallel radix-2 DIT along one axis with a closed-form line decomposition:
// the axis has 2^lgn points `sa` apart (bit-reversed input, natural output); line r of
// nlines starts at (r >> sh) * hs + (r & ((1 << sh) - 1)) * ls.  One barrier per stage.
__device__ __noinline__ void fft_axis_fast(float2* A, int lgn, int sa, int nlines, int sh, int hs, int ls,
                                           const float2* __restrict__ tw) {
  if (lgn == 0) return;
  const int nbf = nlines << (lgn - 1);
  const int lmask = (1 << sh) - 1;
  for (int s = 1; s <= lgn; ++s) {
    const int hm = (1 << (s - 1)) - 1;
    const int gm = (1 << (lgn - s)) - 1;
    const int half = 1 << (s - 1);
    for (int bf = threadIdx.x; bf < nbf; bf += blockDim.x) {
      const int j = bf & hm;
      const int g = (bf >> (s - 1)) & gm;
      const int r = bf >> (lgn - 1);
      const int off = (r >> sh) * hs + (r & lmask) * ls;
      float2* e0 = A + off + ((g << s) + j) * sa;
      float2* e1 = e0 + half * sa;
      const float2 u = *e0;
      const float2 t = cmul(tw[j << (7 - s)], *e1);
      *e0 = cadd(u, t);
      *e1 = csub(u, t);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void load_twiddles(float2* tw) {
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tw[i] = c_tw128[i];
}

// Residue fold through shared memory (reduce over the lanes that share residues, written
// to slot[l][r]; segments add).  Same sums as lane_fold, a quarter of its instructions at
// B_last = 8: every lane stores its LP float4 (acc[l][0], acc[l][1]) to scr[l][lane] (odd l
// xor-swizzled by 4 slots, so the reads below are bank-conflict free), then each lane sums
// the 32 / (B_last / 2) entries of an item (l, q) and writes residues 2q, 2q + 1.
// 2 <= B_last <= 32; scr holds LP x 32 float4 and is free (a consumed TMA stage).
template <int LP>
__device__ __forceinline__ void fold_smem(const float2 (&acc)[LP][2], float4* scr, float2* slot, int lane, int blast,
                                          int lghq, int nl, bool first) {
#pragma unroll
  for (int l = 0; l < LP; ++l)
    scr[l * 32 + (lane ^ ((l & 1) << 2))] = make_float4(acc[l][0].x, acc[l][0].y, acc[l][1].x, acc[l][1].y);
  __syncwarp();
  const int hq = 1 << lghq, G = 32 >> lghq;
  for (int it = lane; it < LP * hq; it += 32) {
    const int l = it >> lghq, q = it & (hq - 1);
    const float4* src = scr + l * 32;
    const int sw = (l & 1) << 2;
    float2 s0 = make_float2(0.f, 0.f), s1 = s0;
    for (int g = 0; g < G; ++g) {
      const float4 v = src[(g * hq + q) ^ sw];
      s0 = __fadd2_rn(s0, make_float2(v.x, v.y));
      s1 = __fadd2_rn(s1, make_float2(v.z, v.w));
    }
    if (l < nl) {
      float4* d = reinterpret_cast<float4*>(slot + l * blast + 2 * q);
      if (first) *d = make_float4(s0.x, s0.y, s1.x, s1.y);
      else {
        const float4 o = *d;
        *d = make_float4(o.x + s0.x, o.y + s0.y, o.z + s1.x, o.w + s1.y);
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // scr is a TMA stage again
  __syncwarp();
}

template <int LP>
__device__ __forceinline__ void colweight_fold(float2 (&acc)[LP][2], const float* __restrict__ hlast,
                                               int l0, int nl, int nlast, int col, int blast) {
  colweight<LP>(acc, hlast, l0, nl, nlast, col);
  lane_fold<LP>(acc, blast);
}

// fold_group with per-row weights formed on the fly: w[l] = h0v[l] * wrow[u][l] (D == 3,
// more loops than two accumulator sets fit in registers).
template <int LP, int U>
__device__ __forceinline__ void fold_group_prod(float2 (&acc)[LP][2], const float4* __restrict__ buf, int lane,
                                                const float* const (&wrow)[U], const float (&h0v)[LP]) {
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = buf[u * 32 + lane];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const float4* wr = reinterpret_cast<const float4*>(wrow[u]);
#pragma unroll
    for (int l4 = 0; l4 < LP / 4; ++l4) {
      const float4 w = wr[l4];
      const float wv[4] = {w.x * h0v[4 * l4], w.y * h0v[4 * l4 + 1], w.z * h0v[4 * l4 + 2], w.w * h0v[4 * l4 + 3]};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        mac(acc[4 * l4 + i][0], wv[i], v[u].x, v[u].y);
        mac(acc[4 * l4 + i][1], wv[i], v[u].z, v[u].w);
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// Fused mode: persistent CTAs, one frame at a time per CTA.  D in {1, 2}, N_last >= 64.
// Warp task = (outer residue class kappa, segment group g); unit = (task, 64-column
// segment); a unit folds the A0 rows of class kappa over its segment (D == 1: one row).
// smem: ring [nwarps][S][U][32] float4 | bars [nwarps][S] | F [G][nl][bouter][blast+1] |
//       tw[128] | rowW [N0+1][LP] float (row N0 = zeros)
// ------------------------------------------------------------------------------------
template <int LP, int U, int S, int T, int C>
__global__ void __launch_bounds__(T, C) k_fused(PlanDev pd, const __grid_constant__ CUtensorMap tmap,
                                                    int64_t batch, int l0, int nl,
                                                    uint32_t* __restrict__ bitmaps,
                                                    float2* __restrict__ spectra, int64_t bm_stride,
                                                    int64_t sp_stride) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smem[];
  const int D = pd.D;
  const int blast = pd.blast, nlast = pd.nlast, bouter = pd.bouter;
  const int fstride = blast + 1;
  const int nseg = nlast >> 6;
  const int G = (D == 1) ? (nseg < 8 ? nseg : 8) : 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  float4* ring = reinterpret_cast<float4*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (size_t)nwarps * S * U * 32);
  float2* F = reinterpret_cast<float2*>(bars + nwarps * S);
  const int fslot = nl * bouter * fstride;
  float2* tw = F + (((size_t)G * fslot + 1) & ~size_t(1));   // keep rowW 16-B aligned
  float* rowW = reinterpret_cast<float*>(tw + 128);
  float4* myring = ring + (size_t)warp * S * U * 32;
  uint64_t* mybar = bars + warp * S;

  const int n0 = D == 2 ? pd.n[0] : 1;
  load_twiddles(tw);
  for (int i = tid; i < (n0 + 1) * LP; i += blockDim.x) {
    int s0 = i / LP, l = i - s0 * LP;
    float w = 0.f;
    if (l < nl && s0 < n0) w = D == 2 ? pd.h[0][(size_t)(l0 + l) * n0 + s0] : 1.f;
    rowW[i] = w;
  }
  if (lane == 0) {
    for (int st = 0; st < S; ++st) mbar_init(&mybar[st], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const float* __restrict__ hlast = pd.h[D - 1];
  const int ntasks = bouter * G;
  const int A0 = D == 2 ? pd.a[0] : 1, B0 = D == 2 ? pd.b[0] : 1;
  const int spt = nseg / G;                        // segments per task
  const int ntw = warp < ntasks ? (ntasks - 1 - warp) / nwarps + 1 : 0;
  // D == 2: unit = (task, segment), groups of U rows of the class.  D == 1: unit = task,
  // groups of U consecutive 64-column segments of the single row.
  const int units = D == 2 ? ntw * spt : ntw;
  const int ngrp = D == 2 ? (A0 + U - 1) / U : (spt + U - 1) / U;
  const int64_t nfr = batch > (int64_t)blockIdx.x ? (batch - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = nfr * units * ngrp;
  const int fold_lanes = blast >= 2 ? blast / 2 : 1;
  const int fold_e = blast >= 2 ? 2 : 1;
  const uint64_t tmap_ptr = reinterpret_cast<uint64_t>(&tmap);
  const int lg_spt = __ffs(spt) - 1;               // spt is a power of two

  // producer cursor (lane 0): next group to load, advanced without divisions
  int p_fi = 0, p_unit = 0, p_grp = 0, p_st = 0;
  int64_t p_left = total;
  auto issue_next = [&]() {
    if (p_left <= 0) return;
    --p_left;
    const int frame = (int)(blockIdx.x + (int64_t)p_fi * gridDim.x);
    mbar_expect_tx(&mybar[p_st], (uint32_t)U * 512u);
    float4* dst = myring + (size_t)p_st * U * 32;
    if (D == 2) {                                  // box [64 cols][U rows a] of class kappa
      const int kappa = warp + (p_unit >> lg_spt) * nwarps, seg = p_unit & (spt - 1);
      tma_load_4d(dst, tmap_ptr, seg * 64, kappa, p_grp * U, frame, &mybar[p_st]);
    } else {                                       // box [64 cols][U segments]
      const int g = warp + p_unit * nwarps;
      tma_load_3d(dst, tmap_ptr, 0, g * spt + p_grp * U, frame, &mybar[p_st]);
    }
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
  float2 racc[LP][2];                              // per-lane residue sums of one class
  for (int64_t fi = 0; fi < nfr; ++fi) {
    const int64_t frame = blockIdx.x + fi * gridDim.x;
    for (int unit = 0; unit < units; ++unit) {
      if (D == 2) {
        const int kappa = warp + (unit >> lg_spt) * nwarps, seg = unit & (spt - 1);
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
          const int a0 = grp * U;
          const float* wrow[U];
#pragma unroll
          for (int u = 0; u < U; ++u) wrow[u] = rowW + (a0 + u < A0 ? kappa + B0 * (a0 + u) : n0) * LP;
          fold_group<LP, U>(acc, myring + (size_t)c_st * U * 32, lane, wrow);
          __syncwarp();
          if (++c_st == S) { c_st = 0; c_ph ^= 1u; }
        }
        // column weights per segment; the lanes' residues are the same for every segment,
        // so segments accumulate per lane and the cross-lane fold runs once per class
        colweight<LP>(acc, hlast, l0, nl, nlast, seg * 64 + 2 * lane);
#pragma unroll
        for (int l = 0; l < LP; ++l) {
          racc[l][0] = cadd(racc[l][0], acc[l][0]);
          racc[l][1] = cadd(racc[l][1], acc[l][1]);
        }
        if (seg == spt - 1) {
          lane_fold<LP>(racc, blast);
          if (lane < fold_lanes) {
            float2* slot = F + kappa * fstride + 2 * lane;
#pragma unroll
            for (int l = 0; l < LP; ++l)
              if (l < nl)
                for (int e = 0; e < fold_e; ++e) slot[(size_t)l * bouter * fstride + e] = racc[l][e];
          }
        }
      } else {
        const int g = warp + unit * nwarps;
        for (int grp = 0; grp < ngrp; ++grp) {
          if (lane == 0) issue_next();
          mbar_wait(&mybar[c_st], c_ph);
          const int cnt = spt - grp * U < U ? spt - grp * U : U;
          for (int u = 0; u < cnt; ++u) {
            const int seg = g * spt + grp * U + u;
            float4 v = myring[((size_t)c_st * U + u) * 32 + lane];
            float2 acc[LP][2];
#pragma unroll
            for (int l = 0; l < LP; ++l) {
              acc[l][0] = make_float2(v.x, v.y);
              acc[l][1] = make_float2(v.z, v.w);
            }
            colweight_fold<LP>(acc, hlast, l0, nl, nlast, seg * 64 + 2 * lane, blast);
            if (lane < fold_lanes) {
              float2* slot = F + (size_t)g * fslot + 2 * lane;
#pragma unroll
              for (int l = 0; l < LP; ++l)
                if (l < nl)
                  for (int e = 0; e < fold_e; ++e) {
                    float2* dst = slot + (size_t)l * fstride + e;
                    *dst = (grp == 0 && u == 0) ? acc[l][e] : cadd(*dst, acc[l][e]);
                  }
            }
          }
          __syncwarp();
          if (++c_st == S) { c_st = 0; c_ph ^= 1u; }
        }
      }
    }
    __syncthreads();
    if (G > 1) {                                  // deterministic combine of segment groups
      for (int i = tid; i < fslot; i += blockDim.x) {
        float2 sum = F[i];
        for (int gg = 1; gg < G; ++gg) sum = cadd(sum, F[(size_t)gg * fslot + i]);
        F[i] = sum;
      }
      __syncthreads();
    }
    // residue -> bucket (b_d = sigma^{-1}(r_d - tau_d) mod B_d, I3) with the half-bucket
    // twiddles e^{-j pi b_d / B_d} (L1); the permutation goes through registers, landing
    // bit-reversed for the in-place DIT FFT.
    {
      constexpr int PMAX = 8;                      // elements per thread per round
      const int dl = D - 1;
      const int lgbl = pd.lgb[dl], lgb0 = pd.lgb[0];
      const int per_loop = bouter * blast;
      int lchunk = (PMAX * (int)blockDim.x) / per_loop;
      if (lchunk < 1) lchunk = 1;
      for (int lb = 0; lb < nl; lb += lchunk) {
        const int le = lb + lchunk < nl ? lb + lchunk : nl;
        const int nel = (le - lb) * per_loop;
        float2 pv[PMAX];
        int pdst[PMAX];
#pragma unroll
        for (int j = 0; j < PMAX; ++j) {
          int i = tid + j * blockDim.x;
          pdst[j] = -1;
          if (i < nel) {
            int l = lb + i / per_loop, rem = i - (l - lb) * per_loop;
            int ro = rem >> lgbl, rl = rem & (blast - 1);
            const LoopDev& lp = pd.loops[l0 + l];
            int bl = (lp.sinv[dl] * (rl - lp.tau[dl])) & (blast - 1);
            float2 v = F[((size_t)l * bouter + ro) * fstride + rl];
            if (pd.shift[dl]) v = cmul(v, tw[bl << (6 - lgbl)]);
            int bo = 0;
            if (D == 2) {
              bo = (lp.sinv[0] * (ro - lp.tau[0])) & (bouter - 1);
              if (pd.shift[0]) v = cmul(v, tw[bo << (6 - lgb0)]);
              bo = brev(bo, lgb0);
            }
            pv[j] = v;
            pdst[j] = ((l * bouter + bo) * fstride) + brev(bl, lgbl);
          }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < PMAX; ++j)
          if (pdst[j] >= 0) F[pdst[j]] = pv[j];
        __syncthreads();
      }
    }
    {
      // F is [nl][bouter][fstride]: last-dim lines r = (l, bo) start at r * fstride; dim-0
      // lines r = (l, k_last) start at (r >> lg B_last) * bouter * fstride + (r & (B_last-1))
      const int lgbl = pd.lgb[D - 1];
      fft_axis_fast(F, lgbl, 1, nl * bouter, 0, fstride, 0, tw);
      if (D == 2) fft_axis_fast(F, pd.lgb[0], fstride, nl * blast, lgbl, bouter * fstride, 1, tw);
    }
    // |fhat|^2 > gamma_l -> ballot -> bitmap words (Alg. 1 l.10)
    const int wpl = pd.wpl;
    const int nitems = nl * wpl * 32;
    for (int it = tid; it < nitems; it += blockDim.x) {
      int l = it / (wpl * 32), k = it - l * wpl * 32;   // flat bucket index
      bool bit = false;
      if (k < pd.btot) {
        int ko = k / blast, kl = k - ko * blast;
        float2 v = F[((size_t)l * bouter + ko) * fstride + kl];
        bit = v.x * v.x + v.y * v.y > pd.loops[l0 + l].gamma;
        if (spectra) spectra[(size_t)frame * sp_stride + (size_t)l * pd.btot + k] = v;
      }
      unsigned word = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) bitmaps[(size_t)frame * bm_stride + (size_t)l * wpl + (k >> 5)] = word;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------
// Fused mode, D == 1 with a short flat-window support (W <= 1024; c1: N = 4096, W = 512):
// GATHER form of Alg. 1 l.5-10.  Per loop only the W permuted times t with |t_c| <= W/2
// carry a non-zero flat-window weight, so the fold is f_l[b] = sum over the W/B taps
// t = b (mod B) of h_l[s] x[s], s = sigma_l t + tau_l (mod N) (Def. 1, Def. 2
// P:89-91, Eqs. z/l P:272-279; h = w g (-1)^floor(t/B) as in I3): L W complex x real MACs per
// frame instead of L N.  Each warp owns one loop (two when L > 16); lane j owns taps
// i = j + 32 k (t_c = i - W/2), whose sources s sit in registers with their weights for the
// whole kernel (they depend on the loop only).  Consecutive t across the lanes of a warp map
// to s = sigma t + tau with sigma odd, i.e. to 32 distinct banks mod 32: every gather from the
// shared-memory frame is bank-conflict free.
// A producer warp streams whole frames (N x 8 B, one cp.async.bulk each; SASS UBLKCP) into an
// S-slot ring; a slot is released as soon as every loop warp has gathered from it, and the
// warp then runs its loop's half-bucket twiddle (L1), B-point FFT (radix-2 DIF with xor
// shuffles, no barrier), |.|^2 > gamma_l and the ballot to bitmap words in registers
// (Alg. 1 l.9-10; Eq. tpd).  No CTA barrier after the prologue.
// ------------------------------------------------------------------------------------
// Fused c1 path (VL > 0; rsft_run): `nv` vote warps per CTA vote the frames the loop warps just
// finished -- each loop warp also drops its bitmap words into a BS-slot shared ring (mbarriers
// bfull / bempty), a vote warp takes frame fi = v, v + nv, ... and runs the per-frame D = 1 vote
// (vote1d.cuh) while the loop warps fold the next frames: the second stage hides under the HBM
// stream.  Outputs as k_vote1d: detection words, per-frame counts, local index lists.
constexpr int kG1BS = 16;                             // bitmap ring slots (>= vote warps)
// MB = buckets per lane: 2 for B <= 64 (B = 64: lane j owns buckets j and j + 32; B <= 32: the
// lanes' sums are folded by shuffles), B / 32 for B = 128 and 256 (lane j owns buckets j + 32 m;
// the B-point FFT is an in-lane MB-point DIF, the twiddles W_B^{j k1} and a 32-point DIF across
// the lanes: lane p slot r then holds X[brev_MB(r) + MB brev5(p)]).
// seg != 0: segment mode (x [batch][L][N]): loop l0 + l runs on segment l0 + l of each
// frame; the producer streams the nl segments of every frame, each gathered by its loop's warp.
template <int TAPS, int LPW, int VL = 0, int MB = 2>
__global__ void __launch_bounds__(VL ? 672 : 544, 1) k_gather1d(PlanDev pd, const float2* __restrict__ x, int64_t batch,
                                                      int l0, int nl, int W, int S, int chunk, uint32_t* __restrict__ bitmaps,
                                                      float2* __restrict__ spectra, int64_t bm_stride,
                                                      int64_t sp_stride, int nv, uint32_t* __restrict__ vdet,
                                                      unsigned long long* __restrict__ rcount, uint32_t* __restrict__ slots,
                                                      int list_cap, int seg) {
  constexpr int TWN = MB > 2 ? 512 : 128;            // twiddle table W_TWN^k in shared memory
  constexpr int LM = MB == 8 ? 3 : MB == 4 ? 2 : 1;
  extern __shared__ __align__(128) unsigned char smem[];
  const int N = pd.n[0], B = pd.b[0], lgb = pd.lgb[0];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncw = (blockDim.x >> 5) - 1 - (VL ? nv : 0);   // loop warps; then the producer, then vote warps
  const uint32_t fbytes = (uint32_t)N * 8u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + S;
  float2* tw = reinterpret_cast<float2*>(smem + 16 * S + 128 - ((16 * S) & 127));  // 128-B aligned
  unsigned char* ring = reinterpret_cast<unsigned char*>(tw + TWN);
  // fused vote state after the ring: bfull / bempty [BS] | bitmap slots [BS][L wpl] | sinv [VL] |
  // per vote warp: detection words [N/32], ent [32], queue [64]
  uint64_t* bfull = reinterpret_cast<uint64_t*>(ring + (size_t)S * fbytes);
  uint64_t* bempty = bfull + kG1BS;
  const int bsw = pd.L * pd.wpl;
  uint32_t* bslot = reinterpret_cast<uint32_t*>(bempty + kG1BS);
  int* vsinv = reinterpret_cast<int*>(bslot + kG1BS * bsw);
  uint32_t* vbase = reinterpret_cast<uint32_t*>(vsinv + (VL ? VL : 1));
  for (int i = tid; i < TWN; i += blockDim.x) tw[i] = MB > 2 ? c_tw512[i] : c_tw128[i];
  if (tid == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], ncw); }
    if (VL) for (int s = 0; s < kG1BS; ++s) { mbar_init(&bfull[s], ncw); mbar_init(&bempty[s], 1); }
    fence_mbar_init();
  }
  pdl_enter();
  if (VL)
    for (int l = tid; l < VL; l += blockDim.x) vsinv[l] = l < pd.L ? pd.loops[l].sinv[0] : 0;
  __syncthreads();
  const int64_t nfr = batch > (int64_t)blockIdx.x ? (batch - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if constexpr (VL > 0) {
    if (warp > ncw) {                               // ---- vote warps
      const int vw = warp - ncw - 1;
      const int nw = N >> 5;
      uint32_t* dw = vbase + (size_t)vw * (nw + 96);
      int* ent = reinterpret_cast<int*>(dw + nw);
      uint32_t* q = dw + nw + 32;
      for (int w = lane; w < nw; w += 32) dw[w] = 0u;
      int sg[VL];
#pragma unroll
      for (int l = 0; l < VL; ++l) sg[l] = l < pd.L ? pd.loops[l].sig[0] : 0;
      __syncwarp();
      const int L = pd.L, wpl = pd.wpl;
      for (int64_t fi = vw; fi < nfr; fi += nv) {
        const int slot = (int)(fi & (kG1BS - 1));
#ifndef RSFT_G1_SLEEP
#define RSFT_G1_SLEEP 0
#endif
        if (RSFT_G1_SLEEP) mbar_wait_backoff(&bfull[slot], (uint32_t)((fi / kG1BS) & 1), RSFT_G1_SLEEP);
        else mbar_wait(&bfull[slot], (uint32_t)((fi / kG1BS) & 1));
        const uint32_t* b = bslot + slot * bsw;
        uint32_t mlo[VL], mhi[VL];
#pragma unroll
        for (int l = 0; l < VL; ++l) {
          mlo[l] = l < L ? b[l * wpl] : 0u;
          mhi[l] = (l < L && wpl > 1) ? b[l * wpl + 1] : 0u;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bempty[slot]);
        vote1d_frame<VL>(pd, mlo, mhi, sg, vsinv, ent, q, dw, (int64_t)blockIdx.x + fi * gridDim.x, vdet, rcount,
                         slots, list_cap);
        __syncwarp();
      }
      return;
    }
  }

  if (warp == ncw) {                                // ---- producer: whole frames (segments), S-deep ring
    if (lane == 0) {
      int s = 0, j = 0;
      uint32_t ph = 0;                              // empty-barrier parity of slot s's previous use
      int64_t fi = 0;
      const int64_t nit = seg ? nfr * nl : nfr;
      for (int64_t g = 0; g < nit; ++g) {           // item g = (frame fi, segment j)
        if (g >= S) {
          if (RSFT_G1_SLEEP) mbar_wait_backoff(&empty[s], ph, RSFT_G1_SLEEP);
          else mbar_wait(&empty[s], ph);
        }
        mbar_expect_tx(&full[s], fbytes);
        const int64_t frame = blockIdx.x + fi * gridDim.x;
        const int64_t row = seg ? frame * pd.L + l0 + j : frame;
        const char* src = reinterpret_cast<const char*>(x + (size_t)row * N);
        for (uint32_t o = 0; o < fbytes; o += (uint32_t)chunk)
          tma_load_1d(ring + (size_t)s * fbytes + o, src + o, (uint32_t)chunk, &full[s]);
        if (++s == S) { s = 0; if (g >= 2 * S - 1) ph ^= 1u; }   // use u + 1 waits for parity u & 1
        if (!seg || ++j == nl) { j = 0; ++fi; }
      }
    }
    return;
  }

  // ---- loop warps: taps, weights and twiddles in registers for the whole kernel
  const bool shift = pd.shift[0] != 0;
  uint32_t off[LPW][TAPS];
  float wt[LPW][TAPS];
  int lid[LPW];
  float gam[LPW];
#pragma unroll
  for (int q = 0; q < LPW; ++q) {
    const int l = warp + q * ncw;
    lid[q] = l < nl ? l : -1;
    gam[q] = pd.loops[l0 + (l < nl ? l : 0)].gamma;
    const LoopDev& lp = pd.loops[l0 + (l < nl ? l : 0)];
    const float* __restrict__ h = pd.h[0] + (size_t)(l0 + (l < nl ? l : 0)) * N;
#pragma unroll
    for (int k = 0; k < TAPS; ++k) {
      const int i = lane + 32 * k;
      const uint32_t t = shift ? (uint32_t)(i - W / 2) & (uint32_t)(N - 1) : (uint32_t)i;
      const uint32_t s = ((uint32_t)lp.sig[0] * t + (uint32_t)lp.tau[0]) & (uint32_t)(N - 1);
      const bool ok = l < nl && i < W;
      off[q][k] = ok ? s * 8u : 0u;
      wt[q][k] = ok ? h[s] : 0.f;
    }
  }
  float2 stw[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int hh = 16 >> q;
    stw[q] = tw[((lane & (hh - 1)) * (TWN / 2)) / hh];
  }
  const DifTw dt = dif_tw(lane, stw);
  // the fused-vote build (VL > 0, 96 registers) keeps the select-form DIF: the packed form's per-lane
  // constants spill there (c1 rsft_run 0.92 vs 0.85 ms)
  auto dif = [&](float2 x, int lg) -> float2 {
    if constexpr (VL > 0) return warp_dif_sel(x, lane, lg, stw);
    else return warp_dif(x, lg, dt);
  };
  // half-bucket twiddles e^{-j pi b / B} of the lane's buckets (L1), stage-1 twiddle (B = 64)
  const float2 sh0 = MB > 2 ? make_float2(1.f, 0.f) : shift ? tw[(lane & (B - 1)) << (6 - lgb)] : make_float2(1.f, 0.f);
  const float2 sh1 = MB > 2 ? make_float2(1.f, 0.f) : shift ? tw[((lane + 32) & (B - 1)) << (6 - lgb)] : make_float2(1.f, 0.f);
  const float2 w64 = tw[2 * lane];
  const int wpl = pd.wpl;

  int s = 0;
  uint32_t ph = 0;
  for (int64_t fi = 0; fi < nfr; ++fi) {
    const int64_t frame = blockIdx.x + fi * gridDim.x;
    const int bsl = (int)(fi & (kG1BS - 1));
    if (VL && fi >= kG1BS) mbar_wait(&bempty[bsl], (uint32_t)(((fi / kG1BS) - 1) & 1));   // slot voted
    // tap k -> bucket lane + 32 (k mod MB) (B = 32 MB; B = 64: even / odd taps); for B <= 32
    // both parities land in bucket lane mod B and are added below (compile-time register indices)
    float2 acc[LPW][MB];
    if (seg) {
      // one ring slot per (frame, loop j): every loop warp passes every slot in order (so no
      // warp runs two phases ahead of a slot's barrier); the owner of loop j gathers from it
#pragma unroll
      for (int q = 0; q < LPW; ++q)
#pragma unroll
        for (int m = 0; m < MB; ++m) acc[q][m] = make_float2(0.f, 0.f);
      for (int j = 0; j < nl; ++j) {
        mbar_wait(&full[s], ph);
        const unsigned char* xs = ring + (size_t)s * fbytes;
#pragma unroll
        for (int q = 0; q < LPW; ++q) {
          if (lid[q] != j) continue;                // warp-uniform
#pragma unroll
          for (int k = 0; k < TAPS; ++k) {
            const float2 v = *reinterpret_cast<const float2*>(xs + off[q][k]);
            acc[q][k % MB] = __ffma2_rn(make_float2(wt[q][k], wt[q][k]), v, acc[q][k % MB]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    } else {
      mbar_wait(&full[s], ph);
      const unsigned char* xs = ring + (size_t)s * fbytes;
#pragma unroll
      for (int q = 0; q < LPW; ++q) {
#pragma unroll
        for (int m = 0; m < MB; ++m) acc[q][m] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < TAPS; ++k) {
          const float2 v = *reinterpret_cast<const float2*>(xs + off[q][k]);
          acc[q][k % MB] = __ffma2_rn(make_float2(wt[q][k], wt[q][k]), v, acc[q][k % MB]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);        // slot free: the rest is in registers
      if (++s == S) { s = 0; ph ^= 1u; }
    }

#pragma unroll
    for (int q = 0; q < LPW; ++q) {
      if (lid[q] < 0) continue;                     // warp-uniform
      const int l = lid[q];
      const float gamma = gam[q];
      uint32_t* bmw = bitmaps + (size_t)frame * bm_stride + (size_t)l * wpl;
      float2* sp = spectra ? spectra + (size_t)frame * sp_stride + (size_t)l * pd.btot : nullptr;
      if constexpr (MB > 2) {                       // B = 32 MB (128, 256)
        float2 v[MB];
#pragma unroll
        for (int m = 0; m < MB; ++m)                // half-bucket twiddles e^{-j pi b / B} (L1)
          v[m] = shift ? cmul(acc[q][m], tw[(lane + 32 * m) << (8 - lgb)]) : acc[q][m];
#pragma unroll
        for (int st = 0; st < LM; ++st) {           // in-lane MB-point DIF over m (bit-reversed out)
#pragma unroll
          for (int e = 0; e < MB / 2; ++e) {
            const int span = MB >> (st + 1);
            const int j = e & (span - 1), blk = (e / span) * 2 * span;
            const float2 a = v[blk + j], b = v[blk + j + span];
            v[blk + j] = cadd(a, b);
            v[blk + j + span] = j == 0 ? csub(a, b) : cmul(csub(a, b), tw[j * (256 / span)]);
          }
        }
#pragma unroll
        for (int r = 1; r < MB; ++r) {              // W_B^{lane k1}, k1 = brev_MB(r)
          const int k1 = brev(r, LM);
          v[r] = cmul(v[r], tw[((lane * k1) & (B - 1)) << (9 - lgb)]);
        }
        int val = 0;
#pragma unroll
        for (int r = 0; r < MB; ++r) {
          v[r] = dif(v[r], 5);
          val |= (v[r].x * v[r].x + v[r].y * v[r].y > gamma ? 1 : 0) << r;
          if (sp) sp[brev(r, LM) + MB * brev(lane, 5)] = v[r];
        }
        uint32_t wd[MB];
#pragma unroll
        for (int t = 0; t < MB; ++t) {              // word t: bucket k = 32 t + lane
          const int k = 32 * t + lane;
          const int vq = __shfl_sync(0xffffffffu, val, brev(k >> LM, 5));
          wd[t] = __ballot_sync(0xffffffffu, (vq >> brev(k & (MB - 1), LM)) & 1);
        }
        if (lane == 0) {
#pragma unroll
          for (int t = 0; t < MB; t += 4)
            *reinterpret_cast<uint4*>(bmw + t) = make_uint4(wd[t], wd[t + 1], wd[t + 2], wd[t + 3]);
        }
      } else if (B == 64) {
        const float2 a = cmul(acc[q][0], sh0), c = cmul(acc[q][1], sh1);
        float2 u = cadd(a, c), v = cmul(csub(a, c), w64);   // X[2k] <- u, X[2k+1] <- v
        u = dif(u, 5);
        v = dif(v, 5);
        const int kb = 2 * brev(lane, 5);                   // lane p holds X[kb], X[kb + 1]
        if (sp) { sp[kb] = u; sp[kb + 1] = v; }
        const int val = (u.x * u.x + u.y * u.y > gamma ? 1 : 0) | (v.x * v.x + v.y * v.y > gamma ? 2 : 0);
        const int sl = brev(lane >> 1, 5);
        const int va = __shfl_sync(0xffffffffu, val, sl), vb = __shfl_sync(0xffffffffu, val, sl ^ 1);
        const uint32_t w0 = __ballot_sync(0xffffffffu, (va >> (lane & 1)) & 1);
        const uint32_t w1 = __ballot_sync(0xffffffffu, (vb >> (lane & 1)) & 1);
        if (lane == 0) *reinterpret_cast<uint2*>(bmw) = make_uint2(w0, w1);
        if (VL && lane == 0) { bslot[bsl * bsw + l * wpl] = w0; bslot[bsl * bsw + l * wpl + 1] = w1; }
      } else {
        float2 a = cadd(acc[q][0], acc[q][1]);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1)
          if (o >= B) a = cadd(a, shfl_xor2(a, o));         // lanes with equal lane mod B
        a = cmul(a, sh0);
        a = dif(a, lgb);
        const int kb = brev(lane & (B - 1), lgb);
        if (sp && lane < B) sp[kb] = a;
        const int val = a.x * a.x + a.y * a.y > gamma ? 1 : 0;
        const int vq = __shfl_sync(0xffffffffu, val, brev(lane & (B - 1), lgb));
        const uint32_t w0 = __ballot_sync(0xffffffffu, lane < B && vq);
        if (lane == 0) bmw[0] = w0;
        if (VL && lane == 0) bslot[bsl * bsw + l * wpl] = w0;
      }
    }
    if (VL) {                                       // this warp's loops of frame fi are in the slot
      __syncwarp();
      if (lane == 0) mbar_arrive(&bfull[bsl]);
    }
  }
}

// ------------------------------------------------------------------------------------
// Split mode, kernel 1: persistent, per-WARP work units (frame, outer residue class kappa,
// dim-0 chunk c); D in {2, 3}.  Unit u of warp gw = blockIdx.x * nwarps + warp is
// gw + i * (gridDim.x * nwarps).  Each warp streams its unit's rows through its own TMA ring
// (RPW = 64/N_last rows of N_last < 64 complex packed per 512 B slot); lane 0 issues boxes
// S-1 ahead across unit boundaries, so HBM keeps streaming with no CTA barrier anywhere.
// Row weights: D == 2 -> h0[a0][l] (staged per unit); D == 3 -> h0[a0][l] h1[a1][l] (I3),
// applied in two levels (a1 rows with h1, then each a0 group with h0).  Output: the residue sums R[frame][l][kappa][r_last] (identity I2:
// the class of every sample is fixed by its residues) BEFORE the per-loop residue -> bucket
// relabelling and half-bucket twiddles, which k_split_fft applies.  With several chunks
// per class each warp writes its chunk partial and the class's last warp to finish sums the
// partials in chunk order (deterministic) into R.  The sums are linear in x, so partial sums
// of dim-0 slabs (a0_base, a0_count) add up to the whole frame's (variant B).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int LP, int U, int RPW>
__global__ void __launch_bounds__(kThreadsSplit, LP >= 24 ? 1 : kCtasSplit)
k_split_fold(PlanDev pd, const __grid_constant__ CUtensorMap tmap, int l0, int nl, int64_t batch,
             int a0_base, int a0_count, int lg_chunk, float2* __restrict__ R, uint32_t* __restrict__ zero_bm,
             int64_t zero_words, int seg_L) {
  // seg_L > 0 (segment mode): `batch` counts (frame, segment) pseudo-frames f L + s, each
  // folded for the single loop l0 + s (nl == 1); the tables then hold all seg_L loops
  const int LT = seg_L > 0 ? seg_L : LP;             // loops in the column-weight / DFT tables
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int S = kStagesSplit;
  constexpr int BR = U * RPW;                        // run rows per TMA box
  constexpr int LPR = 32 / RPW;                      // lanes per row
  const int D = pd.D;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int lane_row = lane / LPR, lane_c4 = lane - lane_row * LPR;
  const int blast = pd.blast, nlast = pd.nlast, bouter = pd.bouter;
  const int B0 = pd.b[0], B1 = D == 3 ? pd.b[1] : 1;
  const int lgb1 = D == 3 ? pd.lgb[1] : 0;
  const int A0 = pd.a[0], A1 = D == 3 ? pd.a[1] : 1;
  const int nchunk = 1 << lg_chunk;
  const int A0c = a0_count >> lg_chunk;              // dim-0 residue rows per unit
  const int nseg = RPW == 1 ? nlast >> 6 : 1;
  const int fold_lanes = blast >= 2 ? blast / 2 : 1;
  const int fold_e = blast >= 2 ? 2 : 1;
  const int AR = D == 3 ? A1 : A0c;                  // run length: a1 (D == 3) or the chunk's a0
  const int nb_run = AR > BR ? AR / BR : 1;
  const int per_a0 = D == 3 ? A0c : 1;               // a0 groups per segment
  // D == 3 with short a1 runs (A1 < BR, e.g. c3: A1 = 8, 32-row boxes): each box spans
  // G = BR / A1 whole a0 groups (5-D tensor map {N_last, r1, a1, r0, frame a0_count + a0}), so
  // no box row is out of bounds (the 4-D map zero-filled BR - A1 rows per box and folded them)
  const int MG = split_multi_g(D, LP, A1, A0c, RPW, nseg);
  const int plane_stride = a0_count * B0;            // dim-0 planes per frame in this launch

  const SplitWarpLayout wl = split_warp_layout(D, LP, nl, A0c, A1, blast, nseg, RPW);
  unsigned char* wbase = smem + (size_t)warp * wl.total;
  float4* ring = reinterpret_cast<float4*>(wbase + wl.ring);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + wl.bars);
  float* hsb = reinterpret_cast<float*>(wbase + wl.hs);
  const int hs_f = wl.hs_stride / 4;                 // floats per hs buffer
  float2* slot = reinterpret_cast<float2*>(wbase + wl.slot);

  const int64_t TW = (int64_t)gridDim.x * nwarps;
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t nunits = (batch * bouter) << lg_chunk;
  const int64_t my_units = nunits > gw ? (nunits - 1 - gw) / TW + 1 : 0;

  // k_split_fft ORs bits into the bitmaps: zero them first (stream order)
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < zero_words; w += (int64_t)gridDim.x * blockDim.x)
    zero_bm[w] = 0u;

  // column weights h_last[l0 + l][col] for the whole launch in shared memory (if small):
  // rows l >= nl are zero (padded loops)
  const float* hl_smem = nullptr;
  const int LH = seg_L > 0 ? seg_L + LP : LP;        // rows (segment mode: + LP zero rows)
  const int nlh = seg_L > 0 ? seg_L : nl;
  if ((size_t)LH * nlast * 4 <= kSplitHlastBytes) {
    float* t = reinterpret_cast<float*>(smem + (size_t)nwarps * wl.total);
    for (int i = threadIdx.x; i < LH * nlast; i += blockDim.x) {
      const int l = i / nlast, c = i - l * nlast;
      t[i] = l < nlh ? pd.h[D - 1][(size_t)(l0 + l) * nlast + c] : 0.f;
    }
    __syncthreads();
    hl_smem = t;
  }
  float2* tws = reinterpret_cast<float2*>(smem + (size_t)nwarps * wl.total +
                                         ((size_t)LH * nlast * 4 <= kSplitHlastBytes ? (size_t)LH * nlast * 4 : 0));
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tws[i] = c_tw128[i];
  __syncthreads();
  // last-dim DFT factors e^{-j pi b_l(r) (2k + 1) / B} [or e^{-j 2 pi b_l(r) k / B}],
  // b_l(r) = sigma^{-1}(r - tau) mod B_last, as (T, jT) float4 [r][l][k] (I3, L1)
  const int dl = D - 1, lgbl = pd.lgb[dl], shl = pd.shift[dl];
  const float4* dtab = nullptr;
  if ((size_t)LT * blast * blast * 16 <= kSplitDftBytes) {
    float4* t = reinterpret_cast<float4*>(tws + 128);
    const int m2 = shl ? 2 * blast - 1 : blast - 1;
    const int tsh = shl ? 6 - lgbl : 7 - lgbl;
    for (int i = threadIdx.x; i < LT * blast * blast; i += blockDim.x) {
      const int r = i / (LT * blast), rem = i - r * (LT * blast);
      const int l = rem >> lgbl, k = rem & (blast - 1);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (l < nlh) {
        const LoopDev& lp = pd.loops[l0 + l];
        const int b = (lp.sinv[dl] * (r - lp.tau[dl])) & (blast - 1);
        const float2 w = tws[((b * (shl ? 2 * k + 1 : k)) & m2) << tsh];
        v = make_float4(w.x, w.y, -w.y, w.x);
      }
      t[i] = v;
    }
    __syncthreads();
    dtab = t;
  }
  // zero the parts of the weight tables cp.async never writes: padded loops and pad rows
  for (int i = lane; i < 2 * hs_f; i += 32) hsb[i] = 0.f;

  struct Unit { int frame, kappa, r0, r1, chunk; };
  auto decode = [&](int64_t ui) {
    const int64_t u = gw + ui * TW;
    Unit t;
#if RSFT_SPLIT_ORDER
    const int64_t ncls = batch * bouter;
    t.chunk = (int)(u / ncls);
    const int64_t cu = u - (int64_t)t.chunk * ncls;
#else
    t.chunk = (int)(u & (nchunk - 1));
    const int64_t cu = u >> lg_chunk;
#endif
    t.frame = (int)(cu / bouter);
    t.kappa = (int)(cu - (int64_t)t.frame * bouter);
    t.r0 = t.kappa >> lgb1;
    t.r1 = t.kappa & (B1 - 1);
    return t;
  };
  // stage h0[l0 + l][(a0_base + chunk A0c + a) B0 + r0] (a < A0c) [and h1[l0 + l][r1 + B1 a1]]
  // from the class-major tables into hs with an LP row stride (cp.async, waited per unit)
  const bool stage16 = seg_L == 0 && ((nl | l0 | pd.L) & 3) == 0;
  auto uloop = [&](const Unit& t) { return seg_L > 0 ? l0 + t.frame % seg_L : l0; };   // unit's first loop
  auto stage = [&](const Unit& t, float* h) {
    const int lu = uloop(t);
    const float* s0 = pd.ht[0] + ((size_t)t.r0 * A0 + a0_base + t.chunk * A0c) * pd.L + lu;
    if (stage16) {                                   // 16-B copies: rows of nl loops, 16-B aligned
      const int nl4 = nl >> 2;
      for (int i = lane; i < A0c * nl4; i += 32) {
        const int a = i / nl4, l = (i - a * nl4) << 2;
        cp_async16(h + a * LP + l, s0 + (size_t)a * pd.L + l);
      }
      if (D == 3) {
        const float* s1 = pd.ht[1] + (size_t)t.r1 * A1 * pd.L + lu;
        float* h1 = h + A0c * LP;
        for (int i = lane; i < A1 * nl4; i += 32) {
          const int a = i / nl4, l = (i - a * nl4) << 2;
          cp_async16(h1 + a * LP + l, s1 + (size_t)a * pd.L + l);
        }
      }
      return;
    }
    for (int i = lane; i < A0c * nl; i += 32) {
      const int a = i / nl, l = i - a * nl;
      cp_async4(h + a * LP + l, s0 + (size_t)a * pd.L + l);
    }
    if (D == 3) {
      const float* s1 = pd.ht[1] + (size_t)t.r1 * A1 * pd.L + lu;
      float* h1 = h + A0c * LP;
      for (int i = lane; i < A1 * nl; i += 32) {
        const int a = i / nl, l = i - a * nl;
        cp_async4(h1 + a * LP + l, s1 + (size_t)a * pd.L + l);
      }
    }
  };

  if (lane == 0) {
    for (int st = 0; st < S; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncwarp();

  // producer cursor (lane 0): box coordinates advanced incrementally, unit by unit
  int64_t p_ui = 0;
  int p_st = 0, p_rb = 0, p_a0l = 0, p_seg = 0;
  int p_c0 = 0, p_c1 = 0, p_c2 = 0, p_c3 = 0, p_c2b = 0, p_c3b = 0;
  auto p_unit = [&]() {
    const Unit t = decode(p_ui);
    p_c0 = 0;
    p_c1 = D == 3 ? t.r1 : t.r0;
    p_c2b = D == 3 ? 0 : t.chunk * A0c;
    p_c3b = D == 3 ? t.frame * plane_stride + t.r0 + B0 * t.chunk * A0c : t.frame;
    if (MG) { p_c2b = t.r0; p_c3b = t.frame * a0_count + t.chunk * A0c; }   // 5-D: (0, r1, 0, r0, a0)
    p_c2 = p_c2b;
    p_c3 = p_c3b;
    p_rb = p_a0l = p_seg = 0;
  };
  if (my_units > 0) p_unit();
  const uint64_t tmap_ptr = reinterpret_cast<uint64_t>(&tmap);
  auto issue_next = [&]() {                         // run by all lanes; lane 0 issues
    if (p_ui >= my_units) return;
    if (MG) {
      tma_load_5d_lane0(lane, ring + (size_t)p_st * U * 32, tmap_ptr, 0, p_c1, 0, p_c2, p_c3, &bars[p_st],
                        (uint32_t)U * 512u);
      if (++p_st == S) p_st = 0;
      p_c3 += MG;
      if (++p_a0l < A0c / MG) return;
      if (++p_ui < my_units) p_unit();
      return;
    }
    tma_load_4d_lane0(lane, ring + (size_t)p_st * U * 32, tmap_ptr, p_c0, p_c1, p_c2, p_c3, &bars[p_st],
                      (uint32_t)U * 512u);
    if (++p_st == S) p_st = 0;
    if (++p_rb < nb_run) { p_c2 += BR; return; }
    p_rb = 0;
    p_c2 = p_c2b;
    if (++p_a0l < per_a0) { p_c3 += B0; return; }
    p_a0l = 0;
    p_c3 = p_c3b;
    if (++p_seg < nseg) { p_c0 += 64; return; }
    if (++p_ui < my_units) p_unit();
  };
#if !RSFT_NO_TMA
  for (int j = 0; j < S - 1; ++j) issue_next();
#endif
  if (my_units > 0) stage(decode(0), hsb);

  int c_st = 0;
  uint32_t c_ph = 0;
  const float* __restrict__ hlast = pd.h[D - 1];
  for (int64_t ui = 0; ui < my_units; ++ui) {
    const Unit t = decode(ui);
    float* hcur = hsb + (ui & 1) * hs_f;
    cp_async_wait_all();
    __syncwarp();
    if (ui + 1 < my_units) stage(decode(ui + 1), hsb + ((ui + 1) & 1) * hs_f);
    float2 acc[LP][2];
    for (int seg = 0; seg < nseg; ++seg) {
#pragma unroll
      for (int l = 0; l < LP; ++l) acc[l][0] = acc[l][1] = make_float2(0.f, 0.f);
      if constexpr (LP <= 16) {
        if (MG) {                                    // boxes of MG whole a0 groups (A1 rows each)
          const int UA = A1 / RPW;                   // ring slots per a0 group
          const float* h1b = hcur + (A0c + lane_row) * LP;
          for (int bx = 0; bx < A0c / MG; ++bx) {
            issue_next();
            mbar_wait(&bars[c_st], c_ph);
            const float4* buf = ring + (size_t)c_st * U * 32;
            for (int g = 0; g < MG; ++g) {
              float2 inn[LP][2];
              const float4* gb = buf + g * UA * 32;
              switch (UA) {                          // warp-uniform; h1 rows a1 = u RPW + lane_row
                case 1: { const float* w[1] = {h1b}; fold_group<LP, 1, true>(inn, gb, lane, w); break; }
                case 2: { const float* w[2] = {h1b, h1b + RPW * LP}; fold_group<LP, 2, true>(inn, gb, lane, w); break; }
                case 4: { const float* w[4] = {h1b, h1b + RPW * LP, h1b + 2 * RPW * LP, h1b + 3 * RPW * LP};
                          fold_group<LP, 4, true>(inn, gb, lane, w); break; }
                default: { const float* w[8];
#pragma unroll
                           for (int u = 0; u < 8; ++u) w[u] = h1b + u * RPW * LP;
                           fold_group<LP, 8, true>(inn, gb, lane, w); break; }
              }
              const float2* h0r = reinterpret_cast<const float2*>(hcur + (bx * MG + g) * LP);
#pragma unroll
              for (int l2 = 0; l2 < LP / 2; ++l2) {
                const float2 w = h0r[l2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  acc[2 * l2][e] = __ffma2_rn(make_float2(w.x, w.x), inn[2 * l2][e], acc[2 * l2][e]);
                  acc[2 * l2 + 1][e] = __ffma2_rn(make_float2(w.y, w.y), inn[2 * l2 + 1][e], acc[2 * l2 + 1][e]);
                }
              }
            }
            __syncwarp();
            if (++c_st == S) { c_st = 0; c_ph ^= 1u; }
          }
        }
      }
      for (int a0l = 0; a0l < (MG ? 0 : per_a0); ++a0l) {
        // D == 3: rows (a0, a1) carry h0[a0][l] h1[a1][l] (I3).  LP <= 16: fold the a1 rows
        // with h1 into `inn`, then acc += h0[a0] * inn (two-level, +1/A1 FMAs); LP > 16: the
        // product weight is formed per row (registers do not hold two accumulator sets).
        // D == 2: rows a0 of the chunk carry h0[a0][l] directly.
        const float* wb = hcur + ((D == 3 ? A0c : 0) + lane_row) * LP;
        if (D == 3 && LP <= 16) {
          float2 inn[LP][2];                         // set by the first box (INIT)
          {                                          // box 0 peeled: inn = h1 x (no zero fill)
#if !RSFT_NO_TMA
            issue_next();
            mbar_wait(&bars[c_st], c_ph);
#endif
            const float* wrow[U];
#pragma unroll
            for (int u = 0; u < U; ++u) wrow[u] = wb + u * RPW * LP;
            fold_group<LP, U, true>(inn, ring + (size_t)c_st * U * 32, lane, wrow);
            __syncwarp();
            if (++c_st == S) { c_st = 0; c_ph ^= 1u; }
            wb += BR * LP;
          }
          for (int rb = 1; rb < nb_run; ++rb, wb += BR * LP) {
#if !RSFT_NO_TMA
            issue_next();
            mbar_wait(&bars[c_st], c_ph);
#endif
            const float* wrow[U];
#pragma unroll
            for (int u = 0; u < U; ++u) wrow[u] = wb + u * RPW * LP;
            fold_group<LP, U>(inn, ring + (size_t)c_st * U * 32, lane, wrow);
            __syncwarp();
            if (++c_st == S) { c_st = 0; c_ph ^= 1u; }
          }
          const float2* h0r = reinterpret_cast<const float2*>(hcur + a0l * LP);
#pragma unroll
          for (int l2 = 0; l2 < LP / 2; ++l2) {
            const float2 w = h0r[l2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              acc[2 * l2][e] = __ffma2_rn(make_float2(w.x, w.x), inn[2 * l2][e], acc[2 * l2][e]);
              acc[2 * l2 + 1][e] = __ffma2_rn(make_float2(w.y, w.y), inn[2 * l2 + 1][e], acc[2 * l2 + 1][e]);
            }
          }
        } else {
          float h0v[LP];
#pragma unroll
          for (int l = 0; l < LP; ++l) h0v[l] = D == 3 ? hcur[a0l * LP + l] : 1.f;
          for (int rb = 0; rb < nb_run; ++rb, wb += BR * LP) {
#if !RSFT_NO_TMA
            issue_next();
            mbar_wait(&bars[c_st], c_ph);
#endif
            const float* wrow[U];
#pragma unroll
            for (int u = 0; u < U; ++u) wrow[u] = wb + u * RPW * LP;
            if constexpr (LP % 4 == 0) {
              if (D == 3) fold_group_prod<LP, U>(acc, ring + (size_t)c_st * U * 32, lane, wrow, h0v);
              else fold_group<LP, U>(acc, ring + (size_t)c_st * U * 32, lane, wrow);
            } else
              fold_group<LP, U>(acc, ring + (size_t)c_st * U * 32, lane, wrow);
            __syncwarp();
            if (++c_st == S) { c_st = 0; c_ph ^= 1u; }
          }
        }
      }
      // column weights of this segment + cross-lane residue fold -> slot[l][r] (segments add)
      const int lofs = uloop(t) - l0;                // segment mode: the unit's loop
      if (hl_smem) colweight_plain<LP>(acc, hl_smem + (size_t)lofs * nlast, nlast, seg * 64 + 2 * lane_c4);
      else colweight<LP>(acc, hlast, l0 + lofs, nl, nlast, seg * 64 + 2 * lane_c4);
      if (LP <= kUSplit && blast >= 2 && blast <= 32) {
        fold_smem<LP>(acc, ring + (size_t)((c_st + S - 1) % S) * U * 32, slot, lane, blast, lgbl - 1, nl, seg == 0);
        continue;
      }
      lane_fold<LP>(acc, blast);
      if (lane < fold_lanes) {
#pragma unroll
        for (int l = 0; l < LP; ++l)
          if (l < nl)
            for (int e = 0; e < fold_e; ++e) {
              float2* d = slot + l * blast + 2 * lane + e;
              *d = seg == 0 ? acc[l][e] : cadd(*d, acc[l][e]);
            }
      }
    }
    __syncwarp();
    // last-dim DFT of the unit's residue sums with the residue -> bucket relabelling and the
    // half-bucket twiddle merged into one factor per (loop, residue, k_last) (I3, L1):
    //   F[l][k][kappa] = sum_r slot[l][r] e^{-j pi b_l(r) (2k + 1) / B},  b_l(r) = sigma^{-1}(r - tau)
    // (no shift when B_last = N_last: e^{-j 2 pi b k / B}).  Written per dim-0 chunk;
    // k_split_fft adds the chunks in order (deterministic, no atomics).
    if (dtab) {
      float2* dst = R + (size_t)t.frame * nl * blast * nchunk * bouter + (size_t)t.chunk * bouter + t.kappa;
      for (int i = lane; i < nl * blast; i += 32) {
        const int l = i >> lgbl, k = i & (blast - 1);
        const float2* row = slot + l * blast;
        const float4* tk = dtab + (l + uloop(t) - l0) * blast + k;
        float2 v = make_float2(0.f, 0.f);
#pragma unroll 8
        for (int r = 0; r < blast; ++r) {
          const float2 x = row[r];
          const float4 w = tk[r * LT * blast];
          v = __ffma2_rn(make_float2(x.x, x.x), make_float2(w.x, w.y), v);
          v = __ffma2_rn(make_float2(x.y, x.y), make_float2(w.z, w.w), v);
        }
        dst[(size_t)i * nchunk * bouter] = v;
      }
    } else {
      float2* dst = R + (size_t)t.frame * nl * blast * nchunk * bouter + (size_t)t.chunk * bouter + t.kappa;
      const int m2 = shl ? 2 * blast - 1 : blast - 1;     // twiddle index mod 2B (shift) or B
      const int tsh = shl ? 6 - lgbl : 7 - lgbl;
      for (int i = lane; i < nl * blast; i += 32) {
        const int l = i >> lgbl, k = i & (blast - 1);
        const LoopDev& lp = pd.loops[uloop(t) + l];
        const float2* row = slot + l * blast;
        // twiddle index b(r) (2k + 1) mod 2B [or b(r) k mod B], b(r) = sigma^{-1} (r - tau) mod B
        const int f = shl ? 2 * k + 1 : k;
        int b = (lp.sinv[dl] * (0 - lp.tau[dl])) & (blast - 1);
        const int db = lp.sinv[dl] & (blast - 1);
        float2 v = make_float2(0.f, 0.f);
        for (int r = 0; r < blast; ++r, b = (b + db) & (blast - 1)) v = cadd(v, cmul(row[r], tws[((b * f) & m2) << tsh]));
        dst[(size_t)i * nchunk * bouter] = v;
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------
// Split-mode fold on the tensor cores (D == 3, N_last == 64, L <= 16, A_1 % 16 == 0).
// Per residue class the fold is the dense contraction C[m][l] = sum_rows X[row][m] W[row][l]
// (m = 128 real columns of the 64 complex samples of a row, l = loop, W[row][l] =
// h0_l[a0] h1_l[a1], identity I3), run as 3xTF32 tcgen05.mma (kind::tf32, fp32 accumulators
// in TMEM): X = Xh + Xl, W = Wh + Wl with Xh, Wh the tf32 truncations (the tensor core
// truncates fp32 operands, scripts/micro/umma_tf32.cu) and Xl, Wl the exact fp32 remainders;
// C = Xh (Wh | Wl) + Xl Wh, relative error ~2^-20 (the dropped Xl Wl term).  A = X^T comes
// from TMEM (lane m = real column m, one TMEM column per row): shared-memory operand tiles
// would have to be K-major (tcgen05 takes tf32 from shared memory K-major only; MN-major
// returned zeros in scripts/micro/umma_tf32.cu) and their extra traffic made the kernel
// shared-memory bound; B = the weights, K-major in shared memory.
// Persistent, one CTA per SM, 14 warps:
//   warps 0-7   workers, two groups of 4 taking alternate stage PAIRS: thread m of the
//               group reads column m of the X stage (TMA box, row-major), splits it into
//               Xh / Xl and stores both to its TMEM lane (tcgen05.st); the group writes the
//               K-major weight tiles (Wh | Wl); after a group barrier the group's first warp
//               issues the pair's 8 MMAs into the GROUP's accumulator (one per group: the two
//               groups' partial sums are added in a fixed order, so results are deterministic)
//   warp 8      TMA producer (lane 0): one 5-D tensor-map box (32 rows = 2 stages, 16 KiB)
//               per stage pair into a kMmaSX/2-deep ring
//   warp 9      TMEM owner: accumulators (2 classes in flight x 2 groups x 32 columns) and
//               the A stages (kMmaSP pairs x 2 stages x 32 columns)
//   warps 10-13 epilogue: TMEM -> (Wh | Wl) halves and groups summed, column weights h_last,
//               residue fold (shared memory), last-dim DFT (factor table) -> R
// One class = a0_count x A_1 rows of one (frame, r0, r1); one stage = 16 rows (one a0).
// ------------------------------------------------------------------------------------
// X ring: kMmaSX stage slots; operand ring (TMEM A + shared-memory W): kMmaSP pair slots
#ifndef RSFT_MMA_SX
#define RSFT_MMA_SX 16
#endif
#ifndef RSFT_MMA_SP
#define RSFT_MMA_SP 4
#endif
#ifndef RSFT_MMA_QB
#define RSFT_MMA_QB 2
#endif
constexpr int kMmaSX = RSFT_MMA_SX, kMmaSP = RSFT_MMA_SP, kMmaThreads = 448, kMmaLP = 16, kMmaEStride = 144;
constexpr int kMmaQB = RSFT_MMA_QB;                  // stages per TMA box (2: one pair, 4: two pairs)
constexpr int kMmaNB = kMmaSX / kMmaQB;              // box slots in the X ring
constexpr int kMmaWorkers = 8, kMmaProd = 8, kMmaTmem = 9, kMmaEpi0 = 10;   // warp roles
constexpr int kMmaWStage = 2048;                                           // (Wh | Wl) per stage
static_assert(128 + kMmaSP * 2 * 32 <= 512, "TMEM columns");

struct MmaLayout {
  int x, op, tab, tab_stride, hl, tws, dtab, e, slot, bar, taddr, total;
};
RSFT_HD inline MmaLayout mma_layout(int a0c, int a1, int nlast, int blast) {
  MmaLayout L;
  int off = 0;
  L.x = off; off += kMmaSX * 8192;
  L.op = off; off += kMmaSP * 2 * kMmaWStage;
  L.tab = off; L.tab_stride = (a0c + a1) * kMmaLP * 4; off += 2 * L.tab_stride;
  L.hl = off; off += kMmaLP * nlast * 4;
  L.tws = off; off += 128 * 8;
  L.dtab = off; off += kMmaLP * blast * blast * 16;
  L.e = off; off += kMmaLP * kMmaEStride * 4;
  L.slot = off; off += kMmaLP * blast * 8;
  off = (off + 15) / 16 * 16;
  L.bar = off; off += (2 * kMmaSX + 2 * kMmaSP + 4) * 8;
  L.taddr = off; off += 16;
  L.total = off;
  return L;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // no swizzle, K-major canonical layout; version 1 (sm_100)
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
// warp-wide call sites (uniform descriptors stay in uniform registers); one elected lane issues
__device__ __forceinline__ void umma_tf32_elect(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
               "setp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               :: "r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                  "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                  "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                  "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
               : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
               :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
}

__global__ void __launch_bounds__(kMmaThreads, 1)
k_split_mma(PlanDev pd, const __grid_constant__ CUtensorMap tmap, int l0, int nl, int64_t batch, int a0_base,
            int a0_count, float2* __restrict__ R, uint32_t* __restrict__ zero_bm, int64_t zero_words, int mbar_issue) {
  pdl_enter();
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int LP = kMmaLP;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int D = pd.D;                                  // == 3
  const int nlast = pd.nlast, blast = pd.blast, bouter = pd.bouter;
  const int B1 = pd.b[1], A0 = pd.a[0], A1 = pd.a[1], lgb1 = pd.lgb[1];
  const int nst = a0_count * (A1 >> 4);               // 16-row stages per class (one a0, 16 a1 each)
  const int npairs = nst >> 1;                         // even, >= 2 (launcher)
  const MmaLayout ly = mma_layout(a0_count, A1, nlast, blast);
  uint64_t* xfull = reinterpret_cast<uint64_t*>(smem + ly.bar);
  uint64_t* xempty = xfull + kMmaSX;
  uint64_t* opempty = xempty + kMmaSX;
  uint64_t* accfull = opempty + kMmaSP;
  uint64_t* accempty = accfull + 2;
  uint64_t* opfull = accempty + 2;                     // [kMmaSP]: the 4 group warps' operands written
  uint32_t* taddr_s = reinterpret_cast<uint32_t*>(smem + ly.taddr);
  float* hl = reinterpret_cast<float*>(smem + ly.hl);
  float2* tws = reinterpret_cast<float2*>(smem + ly.tws);
  float4* dtab = reinterpret_cast<float4*>(smem + ly.dtab);
  const int64_t nunits = batch * bouter;

  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + t; w < zero_words; w += (int64_t)gridDim.x * blockDim.x)
    zero_bm[w] = 0u;
  // column weights h_last[l0 + l][c] (zero rows for padded loops), twiddles
  for (int i = t; i < LP * nlast; i += blockDim.x) {
    const int l = i / nlast, c = i - l * nlast;
    hl[i] = l < nl ? pd.h[D - 1][(size_t)(l0 + l) * nlast + c] : 0.f;
  }
  for (int i = t; i < 128; i += blockDim.x) tws[i] = c_tw128[i];
  // zero both class-table buffers (padded loops stay zero; cp.async writes l < nl)
  for (int i = t; i < 2 * ly.tab_stride / 4; i += blockDim.x) reinterpret_cast<float*>(smem + ly.tab)[i] = 0.f;
  if (t == 0) {
    for (int i = 0; i < kMmaNB; ++i) { mbar_init(&xfull[i], 1); mbar_init(&xempty[i], 4 * (kMmaQB / 2)); }  // consuming warps
    for (int i = 0; i < kMmaSP; ++i) mbar_init(&opempty[i], 1);                              // MMA commit
    for (int i = 0; i < 2; ++i) { mbar_init(&accfull[i], 2); mbar_init(&accempty[i], 4); }  // 2 groups / 4 epi warps
    for (int i = 0; i < kMmaSP; ++i) mbar_init(&opfull[i], 4);                               // group warps
    fence_mbar_init();
  }
  if (warp == kMmaTmem) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t taddr = *taddr_s;
  {  // last-dim DFT factors e^{-j pi b_l(r) (2k + 1) / B} [or e^{-j 2 pi b_l(r) k / B}] as (T, jT) [r][l][k]
    const int dl = D - 1, lgbl = pd.lgb[dl], shl = pd.shift[dl];
    const int m2 = shl ? 2 * blast - 1 : blast - 1;
    const int tsh = shl ? 6 - lgbl : 7 - lgbl;
    for (int i = t; i < LP * blast * blast; i += blockDim.x) {
      const int r = i / (LP * blast), rem = i - r * (LP * blast);
      const int l = rem >> lgbl, k = rem & (blast - 1);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (l < nl) {
        const LoopDev& lp = pd.loops[l0 + l];
        const int b = (lp.sinv[dl] * (r - lp.tau[dl])) & (blast - 1);
        const float2 w = tws[((b * (shl ? 2 * k + 1 : k)) & m2) << tsh];
        v = make_float4(w.x, w.y, -w.y, w.x);
      }
      dtab[i] = v;
    }
  }
  __syncthreads();

  if (warp < kMmaWorkers) {
    // ---------------- workers (+ MMA issue by each group's first warp) ----------------
    float* tab = reinterpret_cast<float*>(smem + ly.tab);
    const int tabf = ly.tab_stride / 4;
    const int nl4 = nl >> 2;
    auto stage_tables = [&](int64_t u, float* dst) {
      const int kappa = (int)(u % bouter);
      const int r0 = kappa >> lgb1, r1 = kappa & (B1 - 1);
      const float* s0 = pd.ht[0] + ((size_t)r0 * A0 + a0_base) * pd.L + l0;
      for (int i = t; i < a0_count * nl4; i += 32 * kMmaWorkers) {
        const int a = i / nl4, l = (i - a * nl4) << 2;
        cp_async16(dst + a * LP + l, s0 + (size_t)a * pd.L + l);
      }
      const float* s1 = pd.ht[1] + (size_t)r1 * A1 * pd.L + l0;
      float* d1 = dst + a0_count * LP;
      for (int i = t; i < A1 * nl4; i += 32 * kMmaWorkers) {
        const int a = i / nl4, l = (i - a * nl4) << 2;
        cp_async16(d1 + a * LP + l, s1 + (size_t)a * pd.L + l);
      }
    };
    constexpr uint32_t id32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t id16 = (1u << 4) | (2u << 7) | (2u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t dw0 = umma_desc(smem_u32(smem + ly.op), 512, 128);
    const int kq = warp & 3, grp = warp >> 2;
    const int m = kq * 32 + lane;                      // this thread's real column = TMEM lane
    const uint32_t lane_off = (uint32_t)(kq * 32) << 16;
    int lgJ = 0;
    while ((16 << lgJ) < A1) ++lgJ;
    // pair P = (ci nst + gl) / 2 goes to group P & 1 and uses x slots 2 (P mod SX/2) + {0, 1}
    // and operand pair slot P mod SP (TMEM A columns, shared-memory W tiles)
    int64_t ci = 0;
    if ((int64_t)blockIdx.x < nunits) stage_tables(blockIdx.x, tab);
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++ci) {
      cp_async_wait_all();
      named_bar(1, 32 * kMmaWorkers);
      if (u + gridDim.x < nunits) stage_tables(u + gridDim.x, tab + ((ci + 1) & 1) * tabf);
      const float* h0s = tab + (ci & 1) * tabf;
      const float* h1s = h0s + a0_count * LP;
      const int buf = (int)(ci & 1);
      const uint32_t dacc = taddr + (uint32_t)(buf * 2 + grp) * 32;
      const int pl0 = (int)((grp + ci * npairs) & 1);
      for (int pl = pl0; pl < npairs; pl += 2) {
        const uint32_t P = (uint32_t)(ci * npairs + pl);
        const uint32_t bx = P / (kMmaQB / 2);         // TMA box of this pair
        const int px = (int)(bx % kMmaNB), x = px * kMmaQB + 2 * (int)(P % (kMmaQB / 2)), op = (int)(P % kMmaSP);
        const uint32_t xph = (bx / kMmaNB) & 1, oph = (P / kMmaSP) & 1;
        float* wsl = reinterpret_cast<float*>(smem + ly.op + op * 2 * kMmaWStage);
        const uint32_t acol = taddr + 128 + (uint32_t)(op * 2) * 32;
        mbar_wait(&opempty[op], oph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int h = 0; h < 2; ++h) {                  // weight tiles: rows 4 kq + j, column n = lane
          const int gl = 2 * pl + h;
          const int a0l = gl >> lgJ, a1b = (gl & ((1 << lgJ) - 1)) << 4;
          const int n = lane, l = n & 15;
          const float h0v = h0s[a0l * LP + l];
          float wv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float w = h0v * h1s[(a1b + 4 * kq + j) * LP + l];
            wv[j] = n < 16 ? w : w - tf32_trunc(w);
          }
          *reinterpret_cast<float4*>(wsl + h * (kMmaWStage / 4) + (((kq * 4 + (n >> 3)) * 8 + (n & 7)) << 2)) =
              make_float4(wv[0], wv[1], wv[2], wv[3]);
        }
        // A = X^T: column m of both stages -> TMEM lane m (Xh: the tensor core truncates; Xl exact)
        mbar_wait(&xfull[px], xph);
        float xv[2][16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float* xs = reinterpret_cast<const float*>(smem + ly.x + (x + h) * 8192) + m;
#pragma unroll
          for (int r = 0; r < 16; ++r) xv[h][r] = xs[r * 128];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[px]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t v[32];
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            v[r] = __float_as_uint(xv[h][r]);
            v[16 + r] = __float_as_uint(xv[h][r] - tf32_trunc(xv[h][r]));
          }
          tmem_st32(acol + h * 32 + lane_off, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");    // W tiles -> tensor core
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        if (mbar_issue) {                              // only the issuing warp waits for the group
          __syncwarp();
          if (lane == 0) mbar_arrive(&opfull[op]);
        } else {
          named_bar(2 + grp, 128);                     // the group's operands are complete
        }
        if (kq == grp) {                               // issuing warp: SMSP 0 (group 0) / 1 (group 1)
          if (mbar_issue) mbar_wait(&opfull[op], oph);
          if (pl == pl0) mbar_wait(&accempty[buf], (((uint32_t)(ci >> 1)) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#if RSFT_MMA_DEBUG != 3
          const uint64_t so = (uint64_t)((op * 2 * kMmaWStage) >> 4);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const uint64_t sw = so + (uint64_t)((h * kMmaWStage + c * 1024) >> 4);
              const uint32_t ah = acol + h * 32 + c * 8;
              umma_tf32_elect(dacc, ah, dw0 + sw, id32, (pl > pl0 || h > 0 || c > 0) ? 1u : 0u);
              umma_tf32_elect(dacc, ah + 16, dw0 + sw, id16, 1u);
            }
#endif
          umma_commit_elect(&opempty[op]);
          if (pl + 2 >= npairs) umma_commit_elect(&accfull[buf]);
        }
      }
    }
  } else if (warp == kMmaProd) {
    // ---------------- TMA producer ----------------
    // map dims {N_last, r1, a1, r0, frame * a0_count + a0}; a box = kMmaQB stages = 16 kMmaQB
    // rows: (16 kMmaQB / A_1) a0 x A_1 a1, or 1 a0 x 16 kMmaQB a1 when A_1 is larger
    if (lane == 0) {
      int px = 0;
      uint32_t ph = 0;
      const uint64_t tm = reinterpret_cast<uint64_t>(&tmap);
      const int lgJ = __ffs(A1 >> 4) - 1;
      const int nbox = nst / kMmaQB;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int frame = (int)(u / bouter), kappa = (int)(u % bouter);
        const int r0 = kappa >> lgb1, r1 = kappa & (B1 - 1);
        for (int bi = 0; bi < nbox; ++bi) {
          const int gl = kMmaQB * bi, a0l = gl >> lgJ, a1b = (gl & ((1 << lgJ) - 1)) << 4;
          mbar_wait(&xempty[px], ph ^ 1);
#if RSFT_MMA_DEBUG == 2                               // compute ceiling: no HBM traffic
          mbar_arrive(&xfull[px]);
#else
          mbar_expect_tx(&xfull[px], 8192u * kMmaQB);
          tma_load_5d(smem + ly.x + px * 8192 * kMmaQB, tm, 0, r1, a1b, r0, frame * a0_count + a0l, &xfull[px]);
#endif
          if (++px == kMmaNB) { px = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp >= kMmaEpi0) {
    // ---------------- epilogue ----------------
    const int e = t - kMmaEpi0 * 32, quarter = warp & 3, m = quarter * 32 + lane, c = m >> 1;
    float* E = reinterpret_cast<float*>(smem + ly.e);
    float* slotf = reinterpret_cast<float*>(smem + ly.slot);
    const float2* slot = reinterpret_cast<const float2*>(slotf);
    const int lgbl = pd.lgb[D - 1];
    const int per = 64 / blast;                        // columns per residue (N_last = 64)
    int64_t ci = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++ci) {
      const int frame = (int)(u / bouter), kappa = (int)(u % bouter);
      const int buf = (int)(ci & 1);
      mbar_wait(&accfull[buf], ((uint32_t)(ci >> 1)) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r0v[32], r1v[32];
      const uint32_t ta = taddr + (uint32_t)(buf * 64) + ((uint32_t)(quarter * 32) << 16);
      tmem_ld32(ta, r0v);
      tmem_ld32(ta + 32, r1v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[buf]);
      // group 0 + group 1, each (Xh Wh + Xl Wh) + Xh Wl, then the column weight
#pragma unroll
      for (int l = 0; l < LP; ++l)
        E[l * kMmaEStride + m] = ((__uint_as_float(r0v[l]) + __uint_as_float(r0v[16 + l])) +
                                  (__uint_as_float(r1v[l]) + __uint_as_float(r1v[16 + l]))) * hl[l * nlast + c];
      named_bar(4, 128);
      for (int it = e; it < LP * 2 * blast; it += 128) {         // (l, r, part): residue sums
        const int l = it / (2 * blast), rp = it - l * 2 * blast;
        const float* src = E + l * kMmaEStride + rp;
        float acc = 0.f;
        for (int j = 0; j < per; ++j) acc += src[2 * blast * j];
        slotf[it] = acc;
      }
      named_bar(4, 128);
      float2* dst = R + (size_t)frame * nl * blast * bouter + kappa;
      for (int i = e; i < nl * blast; i += 128) {                // last-dim DFT (I3, L1)
        const int l = i >> lgbl, k = i & (blast - 1);
        const float2* row = slot + l * blast;
        const float4* tk = dtab + l * blast + k;
        float2 v = make_float2(0.f, 0.f);
        for (int rr = 0; rr < blast; ++rr) {
          const float2 xv = row[rr];
          const float4 w = tk[rr * LP * blast];
          v = __ffma2_rn(make_float2(xv.x, xv.x), make_float2(w.x, w.y), v);
          v = __ffma2_rn(make_float2(xv.y, xv.y), make_float2(w.z, w.w), v);
        }
        dst[(size_t)i * bouter] = v;
      }
      named_bar(4, 128);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == kMmaTmem) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(taddr));
}

// Split mode, kernel 2: one CTA per (loop, k_last, frame).  From the folded spectra F (k_last
// domain, one slice per dim-0 chunk): sum the chunks in order, outer relabelling
// b_d = sigma^{-1}(r_d - tau_d) mod B_d + half twiddles e^{-j pi b_d / B_d} (I3, L1), outer-dims
// FFT in smem (forward, unnormalised, L7), |.|^2 > gamma_l -> bitmap bits (atomicOr; words
// zeroed by the fold kernel or the caller), optional spectra.  Alg. 1 l.9-10;
// Eq. tpd.  F holds loops [rl0, rl0 + rnl) of the plan.
// smem: tw[128] | V [B0][B1 + 1]
__global__ void __launch_bounds__(kThreadsFft) k_split_fft(PlanDev pd, const float2* __restrict__ F, int rl0,
                                                           int rnl, int nchunk, int l0, int nl,
                                                           uint32_t* __restrict__ bitmaps,
                                                           float2* __restrict__ spectra, int seg_L) {
  pdl_enter();
  extern __shared__ float4 smem_f4[];
  float2* tw = reinterpret_cast<float2*>(smem_f4);
  float2* V = tw + 128;
  const int D = pd.D;
  const int blast = pd.blast, lgbl = pd.lgb[D - 1];
  const int l = blockIdx.x >> lgbl, kl = blockIdx.x & (blast - 1);   // l relative to l0
  const int64_t frame = blockIdx.y;
  const int tid = threadIdx.x;
  const int b0 = pd.b[0], b1 = D == 3 ? pd.b[1] : 1;
  const int vstride = b1 + 1;                        // padded rows [B0][B1+1]
  const int lgb0 = pd.lgb[0], lgb1 = D == 3 ? pd.lgb[1] : 0;
  const int bouter = pd.bouter;
  // segment mode: pseudo-frame f L + s runs loop l0 + s (nl == rnl == 1)
  const LoopDev& lp = pd.loops[seg_L > 0 ? l0 + (int)(frame % seg_L) : l0 + l];
  const float2* src = F + ((((size_t)frame * rnl + (l0 + l - rl0)) * blast + kl) * nchunk) * bouter;
  load_twiddles(tw);
  __syncthreads();
  for (int o = tid; o < bouter; o += blockDim.x) {
    float2 v = __ldg(src + o);
    for (int c = 1; c < nchunk; ++c) v = cadd(v, __ldg(src + (size_t)c * bouter + o));
    const int o0 = o >> lgb1, o1 = o & (b1 - 1);
    const int bb0 = (lp.sinv[0] * (o0 - lp.tau[0])) & (b0 - 1);
    if (pd.shift[0]) v = cmul(v, tw[bb0 << (6 - lgb0)]);
    int bb1 = 0;
    if (D == 3) {
      bb1 = (lp.sinv[1] * (o1 - lp.tau[1])) & (b1 - 1);
      if (pd.shift[1]) v = cmul(v, tw[bb1 << (6 - lgb1)]);
    }
    V[brev(bb0, lgb0) * vstride + brev(bb1, lgb1)] = v;
  }
  __syncthreads();
  if (D == 3) fft_axis_fast(V, lgb1, 1, b0, 0, vstride, 0, tw);
  fft_axis_fast(V, lgb0, vstride, b1, lgb1, 0, 1, tw);
  const float gamma = lp.gamma;
  uint32_t* bm = bitmaps + ((size_t)frame * nl + l) * pd.wpl;
  for (int o = tid; o < bouter; o += blockDim.x) {
    int o0 = o >> lgb1, o1 = o & (b1 - 1);
    float2 v = V[o0 * vstride + o1];
    int64_t k = (int64_t)o * blast + kl;
    if (v.x * v.x + v.y * v.y > gamma) atomicOr(bm + (k >> 5), 1u << (k & 31));
    if (spectra) spectra[((size_t)frame * nl + l) * pd.btot + k] = v;
  }
}

// Split mode, kernel 2, warp form for B_0 = 32 outer grids (D == 3, c3: 32 x 16): one WARP per
// (frame, loop, k_last) line, no barrier.  Lane b0 loads its relabelled dim-0 row
// r0 = sigma0 b0 + tau0 (mod B0) of the summed folded spectra, does the dim-1 DFT as a direct
// B1 x B1 product with a per-loop factor table T[l][r1][k1] = e^{-j pi b1(r1) / B1} W^{b1(r1) k1},
// b1(r1) = sigma1^{-1}(r1 - tau1) (the relabelling and half twiddle folded in, I3 / L1), applies its
// dim-0 half twiddle and runs the 32-point dim-0 DFT across the lanes (xor shuffles); lane p then
// holds k0 = brev5(p), k1 = 0..B1-1: |.|^2 > gamma_l -> atomicOr into the bitmap words.
template <int B1>
__global__ void __launch_bounds__(256) k_split_fft_w32(PlanDev pd, const float2* __restrict__ F, int rl0, int rnl,
                                                        int nchunk, int l0, int nl, int64_t batch,
                                                        uint32_t* __restrict__ bitmaps, float2* __restrict__ spectra,
                                                        int seg_L) {
  pdl_enter();
  extern __shared__ __align__(16) float2 fw[];
  const int LT = seg_L > 0 ? seg_L : nl;             // loops in the factor table
  float2* T = fw;                                      // [LT][B1][B1]
  float2* tw = fw + (size_t)LT * B1 * B1;             // [128]
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tw[i] = c_tw128[i];
  __syncthreads();
  const int lgb1 = pd.lgb[1], sh1 = pd.shift[1];
  for (int i = threadIdx.x; i < LT * B1 * B1; i += blockDim.x) {
    const int l = i / (B1 * B1), r1 = (i / B1) % B1, k1 = i % B1;
    const LoopDev& lp = pd.loops[l0 + l];
    const int b1 = (lp.sinv[1] * (r1 - lp.tau[1])) & (B1 - 1);
    // e^{-j pi b1 / B1} e^{-j 2 pi b1 k1 / B1} = e^{-j 2 pi b1 (2 k1 + 1) / (2 B1)} (shift) or W^{b1 k1}
    const int idx = sh1 ? ((b1 * (2 * k1 + 1)) & (2 * B1 - 1)) << (6 - lgb1) : ((b1 * k1) & (B1 - 1)) << (7 - lgb1);
    T[i] = tw[idx];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int blast = pd.blast, bouter = pd.bouter, sh0 = pd.shift[0];
  float2 stw[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int h = 16 >> q;
    stw[q] = tw[((lane & (h - 1)) * 64) / h];          // W_{2h}^{lane mod h}
  }
  const DifTw dt = dif_tw(lane, stw);
  const int64_t lines = batch * nl * blast;
  for (int64_t li = (int64_t)blockIdx.x * nw + warp; li < lines; li += (int64_t)gridDim.x * nw) {
    const int64_t frame = li / (nl * blast);
    const int rem = (int)(li - frame * nl * blast), l = rem / blast, kl = rem - l * blast;
    const int lg = seg_L > 0 ? (int)(frame % seg_L) : l;            // loop index into the tables
    const LoopDev& lp = pd.loops[l0 + lg];
    const float2* src = F + ((((size_t)frame * rnl + (l0 + l - rl0)) * blast + kl) * nchunk) * bouter;
    const int r0 = (lp.sig[0] * lane + lp.tau[0]) & 31;             // b0 = lane
    float2 y[B1];
#pragma unroll
    for (int q = 0; q < B1; q += 2) {                  // the row's loads all in flight
      const float4 a = __ldg(reinterpret_cast<const float4*>(src + r0 * B1 + q));
      y[q] = make_float2(a.x, a.y);
      y[q + 1] = make_float2(a.z, a.w);
    }
    for (int c = 1; c < nchunk; ++c) {
#pragma unroll
      for (int q = 0; q < B1; q += 2) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(src + (size_t)c * bouter + r0 * B1 + q));
        y[q] = cadd(y[q], make_float2(a.x, a.y));
        y[q + 1] = cadd(y[q + 1], make_float2(a.z, a.w));
      }
    }
    const float2* Tl = T + (size_t)lg * B1 * B1;
    const float2 t0 = sh0 ? tw[lane << 1] : make_float2(1.f, 0.f);  // e^{-j pi b0 / 32}
    float2 X[B1];
#pragma unroll
    for (int k1 = 0; k1 < B1; ++k1) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int r1 = 0; r1 < B1; ++r1) {
        const float2 t = Tl[r1 * B1 + k1];
        acc = __ffma2_rn(make_float2(y[r1].x, y[r1].x), t, acc);
        acc = __ffma2_rn(make_float2(-y[r1].y, y[r1].y), make_float2(t.y, t.x), acc);
      }
      X[k1] = cmul(acc, t0);
    }
#pragma unroll
    for (int k1 = 0; k1 < B1; ++k1) X[k1] = warp_dif(X[k1], 5, dt);   // dim-0 DFT across the lanes (DIF)
    const int k0 = brev(lane, 5);
    const float gamma = lp.gamma;
    uint32_t* bm = bitmaps + ((size_t)frame * nl + l) * pd.wpl;
    float2* sp = spectra ? spectra + ((size_t)frame * nl + l) * pd.btot : nullptr;
#pragma unroll
    for (int k1 = 0; k1 < B1; ++k1) {
      const int64_t k = (int64_t)(k0 * B1 + k1) * blast + kl;
      if (X[k1].x * X[k1].x + X[k1].y * X[k1].y > gamma) atomicOr(bm + (k >> 5), 1u << (k & 31));
      if (sp) sp[k] = X[k1];
    }
  }
}

// Split mode, kernel 2, warp-register form for B_0 = 32 / 64 outer grids (D == 3; c3: 32 x 16,
// c5: 64 x 32): a 256-thread CTA per (frame, loop, k_last) line, two barriers.  Rows: warp w takes
// bucket rows b0 = w, w + 8, ...; lane j = bucket b1 gathers residue (sigma_0 b0 + tau_0,
// sigma_1 b1 + tau_1) (mod B) of the summed folded spectra (I3), applies both half-bucket
// twiddles (L1) and the warp runs the B1-point dim-1 DIF across its lanes (B0 / 8 rows in flight
// per warp).  Columns: warp w takes columns k1 = w, w + 8, ...; lane j holds row j (B0 = 32: one
// 32-point lane DIF, lane p then holds k0 = brev5(p)) or rows j and j + 32 (B0 = 64: the first
// radix-2 stage of the 64-point dim-0 DIF in-lane, the two 32-point halves across the lanes:
// lane p then holds k0 = 2 brev5(p) (+1)).  |.|^2 > gamma_l -> atomicOr into the bitmap
// words (zeroed by the fold kernel).  Alg. 1 l.9-10; Eq. tpd.
template <int B0, int B1>
__global__ void __launch_bounds__(256) k_split_fft_wr(PlanDev pd, const float2* __restrict__ F, int rl0, int rnl,
                                                        int nchunk, int l0, int nl, int64_t batch,
                                                        uint32_t* __restrict__ bitmaps, float2* __restrict__ spectra,
                                                        int seg_L) {
  pdl_enter();
  constexpr int LB1 = B1 == 32 ? 5 : B1 == 16 ? 4 : 3;
  __shared__ float2 tw[128];
  constexpr int RQ = B0 / 8;                            // rows per warp
  __shared__ float2 V[B0][B1 + 1];
  for (int i = threadIdx.x; i < 128; i += blockDim.x) tw[i] = c_tw128[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int blast = pd.blast, bouter = pd.bouter;
  const bool sh0 = pd.shift[0] != 0, sh1 = pd.shift[1] != 0;
  float2 stw[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int h = 16 >> q;
    stw[q] = tw[((lane & (h - 1)) * 64) / h];          // W_{2h}^{lane mod h}
  }
  const DifTw dt = dif_tw(lane, stw);
  const float2 w64 = tw[2 * lane];                      // W_64^j (first dim-0 stage)
  const int b1 = lane & (B1 - 1);                       // lanes >= B1 duplicate
  const float2 t1 = sh1 ? tw[b1 * (64 / B1)] : make_float2(1.f, 0.f);   // e^{-j pi b1 / B1}
  const int k1_of_lane = brev(b1, LB1);
  const int64_t lines = batch * nl * blast;
  for (int64_t li = blockIdx.x; li < lines; li += gridDim.x) {
    const int64_t frame = li / (nl * blast);
    const int rem = (int)(li - frame * nl * blast), l = rem / blast, kl = rem - l * blast;
    const int lg = seg_L > 0 ? (int)(frame % seg_L) : l;
    const LoopDev lp = pd.loops[l0 + lg];
    const float2* src = F + ((((size_t)frame * rnl + (l0 + l - rl0)) * blast + kl) * nchunk) * bouter;
    const int r1 = (lp.sig[1] * b1 + lp.tau[1]) & (B1 - 1);
    float2 v[RQ];
#pragma unroll
    for (int q = 0; q < RQ; ++q) {                     // rows b0 = warp + 8 q: all gathers in flight
      const int b0 = warp + 8 * q;
      v[q] = __ldg(src + ((lp.sig[0] * b0 + lp.tau[0]) & (B0 - 1)) * B1 + r1);
    }
    for (int c = 1; c < nchunk; ++c) {
#pragma unroll
      for (int q = 0; q < RQ; ++q) {
        const int b0 = warp + 8 * q;
        v[q] = cadd(v[q], __ldg(src + (size_t)c * bouter + ((lp.sig[0] * b0 + lp.tau[0]) & (B0 - 1)) * B1 + r1));
      }
    }
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int b0 = warp + 8 * q;
      float2 x = cmul(v[q], t1);
      if (sh0) x = cmul(x, tw[b0 * (64 / B0)]);       // e^{-j pi b0 / B0}
      x = warp_dif(x, LB1, dt);
      if (lane < B1) V[b0][k1_of_lane] = x;
    }
    __syncthreads();
    const float gamma = lp.gamma;
    uint32_t* bm = bitmaps + ((size_t)frame * nl + l) * pd.wpl;
    float2* sp = spectra ? spectra + ((size_t)frame * nl + l) * pd.btot : nullptr;
    if constexpr (B0 == 64) {
      const int k0e = 2 * brev(lane, 5);
#pragma unroll
      for (int k1 = warp; k1 < B1; k1 += 8) {
        const float2 a = V[lane][k1], b = V[lane + 32][k1];
        const float2 u = warp_dif(cadd(a, b), 5, dt);
        const float2 t = warp_dif(cmul(csub(a, b), w64), 5, dt);
        const int64_t ke = (int64_t)(k0e * B1 + k1) * blast + kl, ko = ke + (int64_t)B1 * blast;
        if (u.x * u.x + u.y * u.y > gamma) atomicOr(bm + (ke >> 5), 1u << (ke & 31));
        if (t.x * t.x + t.y * t.y > gamma) atomicOr(bm + (ko >> 5), 1u << (ko & 31));
        if (sp) { sp[ke] = u; sp[ko] = t; }
      }
    } else {
      const int k0 = brev(lane, 5);
#pragma unroll
      for (int k1 = warp; k1 < B1; k1 += 8) {
        const float2 u = warp_dif(V[lane][k1], 5, dt);
        const int64_t k = (int64_t)(k0 * B1 + k1) * blast + kl;
        if (u.x * u.x + u.y * u.y > gamma) atomicOr(bm + (k >> 5), 1u << (k & 31));
        if (sp) sp[k] = u;
      }
    }
    __syncthreads();                                     // V reused by the next line
  }
}

// Variant B helper: sum the dim-0 chunks of the folded spectra F [L][B_last][nchunk][B_outer]
// into the canonical partial [L][B_last][B_outer] (in chunk order).
__global__ void k_chunk_sum(const float2* __restrict__ F, int nchunk, int64_t bouter, int64_t n, float2* __restrict__ out) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / bouter, o = i - row * bouter;
    const float2* s = F + row * nchunk * bouter + o;
    float2 v = s[0];
    for (int c = 1; c < nchunk; ++c) v = cadd(v, s[(size_t)c * bouter]);
    out[i] = v;
  }
}

// ------------------------------------------------------------------------------------
// K3 vote (persistent).  Reverse mapping + accumulation + second stage (Alg. 1 l.11-14,
// P:226-229; Def. 4; Eq. a_i), evaluated through identity I1 (Props. 3-4,
// P:437-450): abar[i] = sum_l c_l[M_l(i)] with M_l separable per dimension.  A region is
// (frame, prefix): prefix = i0 for D == 3 (k_pre = M_l,0(i0)); one region per frame for
// D <= 2.  Word-parallel: for the row dim rd = D-2 and the last dim ld = D-1,
//   E[l][k_rd][w] = {j : c_l[k_pre, k_rd, M_l,ld(32 w + j)] = 1}
// (32 locations per word: OR of the plan-constant last-dim bucket masks X[l][k][w] over the
// set bits of the bucket row, or one ballot per word), so each (row, CW words) item costs
// one shared load per loop plus an AND (mu = L), OR (mu = 1) or a bit-sliced counter add
// and compare (L10).  CTAs loop over regions; COUNT also stores each region's detection
// count (rcount[region]) for the offset scan of rsft_detect_compact.
// smem: bm [L][lw] | E [L][B_rd][W] | sig_rd [32] | X [L][B_last][W]
// ------------------------------------------------------------------------------------
rsft_status fold_map(const rsft_plan_s* p, const void* d_x, int64_t batch, int64_t n0, CUtensorMap* m, int u,
                            int64_t frame_stride = 0) {
  const int D = p->D;
  const uint64_t e = 8;
  if (frame_stride == 0) frame_stride = p->ntot;
  if (D == 1) {
    cuuint64_t dims[3] = {64, (cuuint64_t)(p->n[0] / 64), (cuuint64_t)batch};
    cuuint64_t str[2] = {64 * e, (cuuint64_t)frame_stride * e};
    cuuint32_t box[3] = {64, (cuuint32_t)u, 1};
    return make_map(m, d_x, 3, dims, str, box);
  }
  const int64_t nl = p->n[D - 1], no = D == 3 ? p->n[D - 2] : n0, bo = p->b[D - 2], ao = no / bo;
  const int64_t planes = D == 3 ? batch * n0 : batch;
  const int64_t rpw = nl >= 64 ? 1 : 64 / nl;
  cuuint64_t dims[4] = {(cuuint64_t)nl, (cuuint64_t)bo, (cuuint64_t)ao, (cuuint64_t)planes};
  cuuint64_t str[3] = {(cuuint64_t)(nl * e), (cuuint64_t)(bo * nl * e),
                       (cuuint64_t)(D == 2 ? frame_stride * e : no * nl * e)};
  cuuint32_t box[4] = {(cuuint32_t)(nl >= 64 ? 64 : nl), 1, (cuuint32_t)(u * rpw), 1};
  return make_map(m, d_x, 4, dims, str, box);
}


template <int TAPS, int LPW, int VL = 0, int MB = 2>
static rsft_status launch_gather1d_t(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl, uint32_t* bm,
                                     void* spectra, cudaStream_t st, int64_t bm_stride, int64_t sp_stride,
                                     uint32_t* vdet = nullptr, unsigned long long* rcount = nullptr,
                                     uint32_t* slots = nullptr, int list_cap = 0, int seg = 0) {
  auto kern = k_gather1d<TAPS, LPW, VL, MB>;
  const int ncw = (nl + LPW - 1) / LPW;
  const char* env_v = getenv("RSFT_G1_VOTE_WARPS");
  const int nv = VL ? (env_v && env_v[0] ? std::max(1, std::min(atoi(env_v), kG1BS)) : 8) : 0;   // 6-12 measured alike, 4 slower
  const int threads = 32 * (ncw + 1 + nv);
  const int W = (int)(p->b[0] < p->n[0] ? p->W[0] : p->n[0]);
  const size_t fbytes = (size_t)p->n[0] * 8;
  const char* env_s = getenv("RSFT_G1_STAGES");
  const char* env_c = getenv("RSFT_G1_CTAS");
  int ctas = env_c && env_c[0] ? atoi(env_c) : (VL ? 1 : 2);
  const size_t vbytes = VL ? (size_t)16 * kG1BS + (size_t)kG1BS * p->L * p->dev.wpl * 4 + (size_t)VL * 4 +
                                 (size_t)nv * (p->n[0] / 32 + 96) * 4
                           : 0;
  int S = env_s && env_s[0] ? atoi(env_s) : 0;
  if (S <= 0) S = (int)std::min<size_t>(8, std::max<size_t>(2, (200 * 1024 / ctas - 2048 - vbytes) / fbytes));
  const size_t smem = 16 * S + 128 + (MB > 2 ? 4096 : 1024) + S * fbytes + vbytes;
  const char* env_k = getenv("RSFT_G1_CHUNK");        // bytes per bulk copy (divides the frame)
  // c1 (32-KiB frames), whole rsft_run step: 2048-B copies 0.901 ms, 4096 0.861, 8192 0.849, 16384 0.842,
  // 32768 (one copy per frame) 0.840
  int chunk = env_k && env_k[0] ? atoi(env_k) : (int)std::min<size_t>(fbytes, 32768);
  if (chunk <= 0 || chunk % 16 || fbytes % chunk) chunk = (int)fbytes;
  rsft_status s = check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  if (s) return s;
  int nb = 0;
  s = check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem), "occupancy");
  if (s) return s;
  if (nb < 1) { set_error("k_gather1d: zero occupancy"); return RSFT_E_UNSUPPORTED; }
  int64_t grid = (int64_t)std::min(nb, ctas) * p->num_sms;
  if (grid > batch) grid = batch;
  if (cudaError_t le_ = pdl_launch(kern, (unsigned)grid, (unsigned)threads, smem, st, p->dev,
                                   reinterpret_cast<const float2*>(d_x), batch, l0, nl, W, S, chunk, bm,
                                   reinterpret_cast<float2*>(spectra), bm_stride, sp_stride, nv, vdet, rcount, slots,
                                   list_cap, seg); le_ != cudaSuccess)
    return check(le_, "k_gather1d launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_gather1d launch");
}

static rsft_status launch_gather1d(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl, uint32_t* bm,
                                   void* spectra, cudaStream_t st, int64_t bm_stride, int64_t sp_stride, int seg = 0) {
  const int taps = gather1d_taps(p);
  const int lpw = nl > 16 ? 2 : 1;
  const int mb = p->b[0] <= 64 ? 2 : (int)(p->b[0] / 32);
#define RSFT_G1(T, M) \
  if (taps == T && mb == M) \
    return lpw == 1 ? launch_gather1d_t<T, 1, 0, M>(p, d_x, batch, l0, nl, bm, spectra, st, bm_stride, sp_stride, nullptr, nullptr, nullptr, 0, seg) \
                    : launch_gather1d_t<T, 2, 0, M>(p, d_x, batch, l0, nl, bm, spectra, st, bm_stride, sp_stride, nullptr, nullptr, nullptr, 0, seg);
  RSFT_G1(4, 2) RSFT_G1(8, 2) RSFT_G1(16, 2) RSFT_G1(32, 2)
  RSFT_G1(4, 4) RSFT_G1(8, 4) RSFT_G1(16, 4) RSFT_G1(32, 4)
  RSFT_G1(8, 8) RSFT_G1(16, 8) RSFT_G1(32, 8)
#undef RSFT_G1
  return RSFT_E_UNSUPPORTED;
}

// Segment mode for D = 1 gather plans: one launch per <= 32 loops, loop l on segment l of every
// frame (x [batch][L][N]); bitmaps [batch][L][wpl], spectra [batch][L][B].
static rsft_status launch_gather1d_segments(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm,
                                            void* spectra, cudaStream_t st) {
  const int L = p->L;
  const int c = (L + kMaxLaunchLoops - 1) / kMaxLaunchLoops, per = (L + c - 1) / c;
  int launches = 0;
  for (int a = 0; a < L; a += per) {
    const int m = std::min(per, L - a);
    void* sp = spectra ? reinterpret_cast<char*>(spectra) + (size_t)a * p->btot * 8 : nullptr;
    p->last_launches = 0;
    rsft_status s = launch_gather1d(p, d_x, batch, a, m, bm + (size_t)a * p->dev.wpl, sp, st,
                                    (int64_t)L * p->dev.wpl, (int64_t)L * p->btot, 1);
    if (s) return s;
    launches += p->last_launches;
  }
  p->last_launches = launches;
  return RSFT_OK;
}

// rsft_run for D = 1 gather plans: the fold kernel with vote warps (first and second stage in one
// launch), all L <= 16 loops; returns E_UNSUPPORTED when the shape does not qualify.
static rsft_status launch_gather1d_voted(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm, uint32_t* det,
                                         unsigned long long* rcount, uint32_t* slots, int list_cap, cudaStream_t st) {
  const int taps = gather1d_taps(p);
  if (p->L > 16 || !taps) return RSFT_E_UNSUPPORTED;
  const int64_t bs = (int64_t)p->L * p->dev.wpl;
#define RSFT_G1V(T) \
  if (taps == T) return p->L <= 8 ? launch_gather1d_t<T, 1, 8>(p, d_x, batch, 0, p->L, bm, nullptr, st, bs, 0, det, rcount, slots, list_cap) \
                                  : launch_gather1d_t<T, 1, 16>(p, d_x, batch, 0, p->L, bm, nullptr, st, bs, 0, det, rcount, slots, list_cap);
  RSFT_G1V(4) RSFT_G1V(8) RSFT_G1V(16) RSFT_G1V(32)
#undef RSFT_G1V
  return RSFT_E_UNSUPPORTED;
}

// frame_stride (complex elements between frames), bm_stride (words) and sp_stride (complex)
// default to the dense layouts; segment mode (rsft_execute_segments) strides over segments.
template <int LP>
static rsft_status launch_fused_t(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl,
                                  uint32_t* bm, void* spectra, cudaStream_t st, int64_t frame_stride = 0,
                                  int64_t bm_stride = 0, int64_t sp_stride = 0) {
  constexpr FusedCfg F2 = kFused2D, F1 = kFused1D;
  const FusedCfg fc = fused_cfg(p->D);
  {
    const char* g1 = getenv("RSFT_NO_GATHER1D");      // read per launch: tests select either kernel
    if (p->D == 1 && (frame_stride == 0 || frame_stride == p->ntot) && gather1d_taps(p) && !(g1 && g1[0] && g1[0] != '0'))
      return launch_gather1d(p, d_x, batch, l0, nl, bm, spectra, st, bm_stride ? bm_stride : (int64_t)nl * p->dev.wpl,
                             sp_stride ? sp_stride : (int64_t)nl * p->btot);
    if (p->D == 1 && p->b[0] > 64) {                 // the streaming 1-D form folds B <= 64 only
      set_error("k_fused: D = 1 with B > 64 needs the gather form (support W <= 1024)");
      return RSFT_E_UNSUPPORTED;
    }
  }
  auto kern = p->D == 2 ? k_fused<LP, F2.u, F2.stages, F2.threads, F2.ctas> : k_fused<LP, F1.u, F1.stages, F1.threads, F1.ctas>;
  size_t smem = fused_smem_bytes(p, nl, LP);
  {
    // D = 2 frames whose tables leave room: a third ring stage per warp keeps a box in flight
    // through the per-frame epilogue (RSFT_F2_STAGES=2 keeps two)
    const char* es = getenv("RSFT_F2_STAGES");
    const size_t s3 = fused_smem_bytes(p, nl, LP, F2.stages + 1);
    if (p->D == 2 && s3 <= 227 * 1024 && !(es && es[0] == '2')) {
      kern = k_fused<LP, F2.u, F2.stages + 1, F2.threads, F2.ctas>;
      smem = s3;
    }
  }
  if (bm_stride == 0) bm_stride = (int64_t)nl * p->dev.wpl;
  if (sp_stride == 0) sp_stride = (int64_t)nl * p->btot;
  CUtensorMap tmap;
  rsft_status s = fold_map(p, d_x, batch, p->n[0], &tmap, fc.u, frame_stride);
  if (s) return s;
  s = check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  if (s) return s;
  int nb = 0;
  s = check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, fc.threads, smem), "occupancy");
  if (s) return s;
  if (nb < 1) { set_error("k_fused: zero occupancy"); return RSFT_E_UNSUPPORTED; }
  int64_t grid = (int64_t)nb * p->num_sms;
  if (grid > batch) grid = batch;
  if (cudaError_t le_ = pdl_launch(kern, (unsigned)grid, fc.threads, smem, st, p->dev, tmap, batch, l0, nl, bm, reinterpret_cast<float2*>(spectra),
                                               bm_stride, sp_stride); le_ != cudaSuccess)
    return check(le_, "kern launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_fused launch");
}

// Split-mode fold of dim-0 rows [a0_base*B0, (a0_base + a0_count)*B0) of `batch` frames
// into residue sums R [batch][nl][B_outer][B_last]; zeroes zero_words bitmap words.
// Tensor-core split fold (k_split_mma): c5-like shapes, one class per CTA iteration (no chunks).
static bool mma_fold_ok(const rsft_plan_s* p, int64_t batch, int l0, int nl, int64_t a0_count) {
  const char* off = getenv("RSFT_NO_MMA");          // read per launch: tests select either kernel
  if ((off && off[0] && off[0] != '0') || p->D != 3 || p->n[2] != 64 || p->a[1] % 16 != 0 || nl > kMmaLP || (nl | l0 | p->L) % 4 != 0) return false;
  const int64_t nst = a0_count * (p->a[1] / 16);                   // 16-row stages per class
  if (nst % kMmaQB != 0 || nst < 4) return false;                  // whole boxes of stage pairs, both groups busy
  const int64_t blast = p->b[2];
  if ((int64_t)kMmaLP * blast * blast * 16 > kSplitDftBytes) return false;
  if (batch * nl * p->btot > p->dev.fbuf_capacity) return false;
  return mma_layout((int)a0_count, (int)p->a[1], 64, (int)blast).total <= 227 * 1024;
}

static rsft_status launch_split_mma(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl, int64_t a0_base,
                                    int64_t a0_count, uint32_t* zero_bm, int64_t zero_words, cudaStream_t st) {
  const size_t smem = (size_t)mma_layout((int)a0_count, (int)p->a[1], 64, (int)p->b[2]).total;
  // x [batch][a0_count B0][N1][64] as {64, r1 (B1), a1 (A1), r0 (B0), frame a0_count + a0}
  const uint64_t e = 8, row = 64 * e;
  const int64_t N1 = p->n[1], B1 = p->b[1], A1 = p->a[1], B0 = p->b[0];
  cuuint64_t dims[5] = {64, (cuuint64_t)B1, (cuuint64_t)A1, (cuuint64_t)B0, (cuuint64_t)(batch * a0_count)};
  cuuint64_t str[4] = {row, (cuuint64_t)(B1 * row), (cuuint64_t)(N1 * row), (cuuint64_t)(B0 * N1 * row)};
  const int64_t rows = 16 * kMmaQB, ba1 = A1 < rows ? A1 : rows;
  cuuint32_t box[5] = {64, 1, (cuuint32_t)ba1, 1, (cuuint32_t)(rows / ba1)};
  CUtensorMap tmap;
  rsft_status s = make_map(&tmap, d_x, 5, dims, str, box);
  if (s) return s;
  s = check(cudaFuncSetAttribute(k_split_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  if (s) return s;
  const int64_t units = batch * p->dev.bouter;
  const int64_t grid = units < p->num_sms ? units : p->num_sms;
  const char* mb = getenv("RSFT_MMA_MBAR");             // issue behind an mbarrier (1) or a group barrier (0)
  const int mbar_issue = mb && mb[0] == '1' ? 1 : 0;
  if (cudaError_t le_ = pdl_launch(k_split_mma, (unsigned)grid, kMmaThreads, smem, st, p->dev, tmap, l0, nl, batch, (int)a0_base, (int)a0_count,
                                                         p->dev.fbuf, zero_bm, zero_words, mbar_issue); le_ != cudaSuccess)
    return check(le_, "k_split_mma launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_split_mma launch");
}

template <int LP>
static rsft_status launch_split_fold_t(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl,
                                       int64_t a0_base, int64_t a0_count, int* lg_out, uint32_t* zero_bm,
                                       int64_t zero_words, cudaStream_t st, int seg_L = 0) {
  if (seg_L == 0 && LP <= kMmaLP && mma_fold_ok(p, batch, l0, nl, a0_count)) {
    *lg_out = 0;
    return launch_split_mma(p, d_x, batch, l0, nl, a0_base, a0_count, zero_bm, zero_words, st);
  }
  auto kern = p->n[p->D - 1] >= 64 ? k_split_fold<LP, kUSplit, 1> : k_split_fold<LP, kUSplit, 2>;
  const int64_t per = (int64_t)nl * p->btot;          // folded spectrum elements per frame and chunk
  int lg = split_lg_chunks(p, batch, nl, a0_count, (int64_t)p->num_sms * (kThreadsSplit / 32) * (LP >= 24 ? 1 : kCtasSplit));
  while (lg > 0 && (batch << lg) * per > p->dev.fbuf_capacity) --lg;
  if (batch * per > p->dev.fbuf_capacity) { set_error("split fold: batch exceeds the workspace"); return RSFT_E_ARG; }
  // more chunks if the per-warp weight tables do not fit (smaller dim-0 chunk per unit)
  const int64_t amin = p->D == 3 ? 1 : (int64_t)kUSplit * (p->n[p->D - 1] >= 64 ? 1 : 64 / p->n[p->D - 1]);
  while (split_smem_bytes(p, nl, LP, a0_count >> lg, seg_L) > 227 * 1024 && (a0_count >> (lg + 1)) >= amin &&
         (batch << (lg + 1)) * per <= p->dev.fbuf_capacity)
    ++lg;
  const size_t smem = split_smem_bytes(p, nl, LP, a0_count >> lg, seg_L);
  if (smem > 227 * 1024) { set_error("k_split_fold: tables beyond shared memory"); return RSFT_E_UNSUPPORTED; }
  CUtensorMap tmap;
  const int rpw = p->n[p->D - 1] >= 64 ? 1 : (int)(64 / p->n[p->D - 1]);
  const int nseg = rpw == 1 ? (int)(p->n[p->D - 1] >> 6) : 1;
  const int mg = split_multi_g(p->D, LP, p->D == 3 ? (int)p->a[1] : 1, (int)(a0_count >> lg), rpw, nseg);
  rsft_status s;
  if (mg) {                // 5-D map {N_last, r1, a1, r0, frame a0_count + a0}, box {N_last, 1, A1, 1, mg}
    const uint64_t e = 8, nl = (uint64_t)p->n[2];
    cuuint64_t dims[5] = {(cuuint64_t)nl, (cuuint64_t)p->b[1], (cuuint64_t)p->a[1], (cuuint64_t)p->b[0],
                          (cuuint64_t)(batch * a0_count)};
    cuuint64_t str[4] = {nl * e, (cuuint64_t)(p->b[1] * nl * e), (cuuint64_t)(p->n[1] * nl * e),
                         (cuuint64_t)(p->b[0] * p->n[1] * nl * e)};
    cuuint32_t box[5] = {(cuuint32_t)nl, 1, (cuuint32_t)p->a[1], 1, (cuuint32_t)mg};
    s = make_map(&tmap, d_x, 5, dims, str, box);
  } else {
    s = fold_map(p, d_x, batch, a0_count * p->b[0], &tmap, kUSplit);
  }
  if (s) return s;
  s = check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr");
  if (s) return s;
  int nb = 0;
  s = check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreadsSplit, smem), "occupancy");
  if (s) return s;
  if (nb < 1) { set_error("k_split_fold: zero occupancy"); return RSFT_E_UNSUPPORTED; }
  const int64_t wunits = (batch * p->dev.bouter) << lg;
  int64_t grid = (int64_t)nb * p->num_sms;
  const int64_t need = (wunits + kThreadsSplit / 32 - 1) / (kThreadsSplit / 32);
  if (grid > need) grid = need;
  if (cudaError_t le_ = pdl_launch(kern, (unsigned)grid, kThreadsSplit, smem, st, p->dev, tmap, l0, nl, batch, (int)a0_base, (int)a0_count, lg,
                                                    p->dev.fbuf, zero_bm, zero_words, seg_L); le_ != cudaSuccess)
    return check(le_, "kern launch");
  p->last_launches += 1;
  *lg_out = lg;
  return check(cudaGetLastError(), "k_split_fold launch");
}

// Folded spectra F (loops [rl0, rl0 + rnl), nchunk chunks) -> bitmaps / spectra of loops [l0, l0 + nl).
static rsft_status launch_split_fft(rsft_plan_s* p, const float2* F, int rl0, int rnl, int nchunk, int64_t batch,
                                    int l0, int nl, uint32_t* bm, void* spectra, cudaStream_t st, int seg_L = 0) {
  const int D = p->D;
  const int64_t blast = p->b[D - 1];
  const int64_t b1 = D == 3 ? p->b[1] : 1;
  {
    // warp form with a direct dim-1 DFT for 32 x B1 outer grids (RSFT_FFT_W32DFT=1; the register
    // form below is the default); RSFT_FFT_WARP=0 (read per launch) keeps the CTA form
    const char* ew = getenv("RSFT_FFT_WARP");
    const char* eo = getenv("RSFT_FFT_W32DFT");
    const int LT = seg_L > 0 ? seg_L : nl;
    const size_t smw = ((size_t)LT * b1 * b1 + 128) * 8;
    if (eo && eo[0] == '1' && D == 3 && p->b[0] == 32 && (b1 == 8 || b1 == 16) && smw <= 64 * 1024 &&
        !(ew && ew[0] == '0')) {
      auto kw = b1 == 8 ? k_split_fft_w32<8> : k_split_fft_w32<16>;
      rsft_status s = check(cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw), "smem attr");
      if (s) return s;
      const int64_t lines = batch * nl * blast;
      const int64_t grid = std::min<int64_t>((lines + 7) / 8, 8 * (int64_t)p->num_sms);
      if (cudaError_t le_ = pdl_launch(kw, (unsigned)grid, 256, smw, st, p->dev, F, rl0, rnl, nchunk, l0, nl, batch, bm,
                                       reinterpret_cast<float2*>(spectra), seg_L); le_ != cudaSuccess)
        return check(le_, "k_split_fft_w32 launch");
      p->last_launches += 1;
      return check(cudaGetLastError(), "k_split_fft_w32 launch");
    }
  }
  {
    // register form for 32 / 64 x B1 outer grids (c3, c5); RSFT_FFT_WARP=0 (read per launch) keeps the CTA form
    const char* ew = getenv("RSFT_FFT_WARP");
    const char* eo = getenv("RSFT_FFT_W32DFT");         // 1: B_0 = 32 grids use k_split_fft_w32 (direct dim-1 DFT)
    const bool w32dft = eo && eo[0] == '1';
    if (D == 3 && (p->b[0] == 64 || (p->b[0] == 32 && !w32dft)) && (b1 == 8 || b1 == 16 || b1 == 32) &&
        !(ew && ew[0] == '0')) {
      auto kw = p->b[0] == 64 ? (b1 == 8 ? k_split_fft_wr<64, 8> : b1 == 16 ? k_split_fft_wr<64, 16> : k_split_fft_wr<64, 32>)
                              : (b1 == 8 ? k_split_fft_wr<32, 8> : b1 == 16 ? k_split_fft_wr<32, 16> : k_split_fft_wr<32, 32>);
      const int64_t lines = batch * nl * blast;
      const int64_t grid = std::min<int64_t>(lines, 8 * (int64_t)p->num_sms);
      if (cudaError_t le_ = pdl_launch(kw, (unsigned)grid, 256, 0, st, p->dev, F, rl0, rnl, nchunk, l0, nl, batch, bm,
                                       reinterpret_cast<float2*>(spectra), seg_L); le_ != cudaSuccess)
        return check(le_, "k_split_fft_wr launch");
      p->last_launches += 1;
      return check(cudaGetLastError(), "k_split_fft_wr launch");
    }
  }
  size_t smem2 = 128 * 8 + (size_t)p->b[0] * (b1 + 1) * 8;
  rsft_status s = check(cudaFuncSetAttribute(k_split_fft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2),
                        "smem attr");
  if (s) return s;
  dim3 grid2((unsigned)(nl * blast), (unsigned)batch);
  // small outer grids (c3: 512 points) run 4 points per thread so that many CTAs are resident;
  // large ones (c5: 2048) keep one L2 round trip per thread
  const char* env_t = getenv("RSFT_FFT_THREADS");
  int threads = env_t && env_t[0] ? atoi(env_t) : 0;
  if (threads <= 0) threads = p->dev.bouter >= 2048 ? kThreadsFft : (int)std::max<int64_t>(64, p->dev.bouter / 4);
  threads = std::min(threads, kThreadsFft);
  if (cudaError_t le_ = pdl_launch(k_split_fft, grid2, (unsigned)threads, smem2, st, p->dev, F, rl0, rnl, nchunk, l0, nl, bm,
                                                 reinterpret_cast<float2*>(spectra), seg_L); le_ != cudaSuccess)
    return check(le_, "k_split_fft launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_split_fft launch");
}

template <int LP>
static rsft_status launch_split_t(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl,
                                  uint32_t* bm, void* spectra, cudaStream_t st) {
  int lg = 0;
  rsft_status s = launch_split_fold_t<LP>(p, d_x, batch, l0, nl, 0, p->a[0], &lg, bm,
                                          batch * nl * (int64_t)p->dev.wpl, st);
  if (s) return s;
  return launch_split_fft(p, p->dev.fbuf, l0, nl, 1 << lg, batch, l0, nl, bm, spectra, st);
}

#define RSFT_DISPATCH_LP(FN, LPV, ...)                   \
  switch (LPV) {                                         \
    case 2: return FN<2>(__VA_ARGS__);                   \
    case 4: return FN<4>(__VA_ARGS__);                   \
    case 6: return FN<6>(__VA_ARGS__);                   \
    case 8: return FN<8>(__VA_ARGS__);                   \
    case 12: return FN<12>(__VA_ARGS__);                 \
    case 16: return FN<16>(__VA_ARGS__);                 \
    case 24: return FN<24>(__VA_ARGS__);                 \
    case 32: return FN<32>(__VA_ARGS__);                 \
    default: return RSFT_E_UNSUPPORTED;                  \
  }

template <int LP>
static rsft_status launch_partial_t(rsft_plan_s* p, const void* d_x, int64_t off, int64_t len, void* d_partial,
                                    cudaStream_t st) {
  int lg = 0;
  rsft_status s = launch_split_fold_t<LP>(p, d_x, 1, 0, p->L, off / p->b[0], len / p->b[0], &lg, nullptr, 0, st);
  if (s) return s;
  const int64_t bouter = p->dev.bouter;
  const int64_t n = (int64_t)p->L * p->btot;
  if (cudaError_t le_ = pdl_launch(k_chunk_sum, (unsigned)std::min<int64_t>((n + 255) / 256, 4 * p->num_sms), 256, 0, st, p->dev.fbuf, 1 << lg, bouter, n, reinterpret_cast<float2*>(d_partial)); le_ != cudaSuccess)
    return check(le_, "k_chunk_sum launch");
  p->last_launches += 1;
  return check(cudaGetLastError(), "k_chunk_sum launch");
}

rsft_status launch_partial(rsft_plan_s* p, const void* d_x, int64_t off, int64_t len, void* d_partial,
                           cudaStream_t st) {
  if (p->L > kMaxLaunchLoops) { set_error("rsft_bucketize_partial: more than 32 loops"); return RSFT_E_UNSUPPORTED; }
  RSFT_DISPATCH_LP(launch_partial_t, loop_pad(p->L), p, d_x, off, len, d_partial, st);
}

rsft_status launch_finalize(rsft_plan_s* p, const void* d_folded, int l0, int nl, uint32_t* bm, void* spectra,
                            cudaStream_t st) {
  rsft_status s = check(cudaMemsetAsync(bm, 0, (size_t)nl * p->dev.wpl * 4, st), "bitmap reset");
  if (s) return s;
  return launch_split_fft(p, reinterpret_cast<const float2*>(d_folded), l0, nl, 1, 1, l0, nl, bm, spectra, st);
}

// Segment mode (second mode; Eq. sig_model): x [batch][L][N...], loop l runs on
// segment l of every frame; bitmaps [batch][L][wpl], spectra [batch][L][B_tot].
template <int LP>
static rsft_status launch_segments_fused_t(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm,
                                           void* spectra, cudaStream_t st) {
  const int64_t L = p->L, wpl = p->dev.wpl;
  for (int64_t l = 0; l < L; ++l) {
    const char* x = reinterpret_cast<const char*>(d_x) + (size_t)l * p->ntot * 8;
    void* sp = spectra ? reinterpret_cast<char*>(spectra) + (size_t)l * p->btot * 8 : nullptr;
    rsft_status s = launch_fused_t<LP>(p, x, batch, (int)l, 1, bm + l * wpl, sp, st, L * p->ntot, L * wpl,
                                       L * p->btot);
    if (s) return s;
  }
  return RSFT_OK;
}

rsft_status launch_execute(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl, uint32_t* bm,
                           void* spectra, cudaStream_t st);

static rsft_status launch_fused_lp(rsft_plan_s* p, int lp, const void* d_x, int64_t batch, int l0, int nl, uint32_t* bm,
                                   void* spectra, cudaStream_t st, int64_t bm_stride, int64_t sp_stride) {
  RSFT_DISPATCH_LP(launch_fused_t, lp, p, d_x, batch, l0, nl, bm, spectra, st, 0, bm_stride, sp_stride);
}

rsft_status launch_segments(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm, void* spectra,
                            cudaStream_t st) {
  {
    const char* g1 = getenv("RSFT_NO_GATHER1D");      // read per launch
    if (p->D == 1 && gather1d_taps(p) && !(g1 && g1[0] && g1[0] != '0'))
      return launch_gather1d_segments(p, d_x, batch, bm, spectra, st);
  }
  if (resolve_mode(p, batch) == RSFT_MODE_FUSED && loop_pad(1) == 2) {
    return launch_segments_fused_t<2>(p, d_x, batch, bm, spectra, st);
  }
  // split mode: the batch x L segments are batch L contiguous pseudo-frames f L + s, each
  // folded for loop s (one fold + one outer-FFT launch for the whole step)
  const int64_t L = p->L, wpl = p->dev.wpl;
  if (L <= kMaxLaunchLoops && batch * L * p->btot <= p->dev.fbuf_capacity) {
    int lg = 0;
    rsft_status s = launch_split_fold_t<2>(p, d_x, batch * L, 0, 1, 0, p->a[0], &lg, bm, batch * L * wpl, st, (int)L);
    if (s) return s;
    return launch_split_fft(p, p->dev.fbuf, 0, 1, 1 << lg, batch * L, 0, 1, bm, spectra, st, (int)L);
  }
  for (int64_t f = 0; f < batch; ++f)               // fallback: one launch per (frame, segment)
    for (int64_t l = 0; l < L; ++l) {
      const char* x = reinterpret_cast<const char*>(d_x) + (size_t)(f * L + l) * p->ntot * 8;
      void* sp = spectra ? reinterpret_cast<char*>(spectra) + (size_t)(f * L + l) * p->btot * 8 : nullptr;
      rsft_status s = launch_execute(p, x, 1, (int)l, 1, bm + (f * L + l) * wpl, sp, st);
      if (s) return s;
    }
  return RSFT_OK;
}

rsft_status launch_execute(rsft_plan_s* p, const void* d_x, int64_t batch, int l0, int nl, uint32_t* bm,
                           void* spectra, cudaStream_t st) {
  if (nl > kMaxLaunchLoops) {                        // > 32 loops: one pass over x per <= 32 loops
    const int c = (nl + kMaxLaunchLoops - 1) / kMaxLaunchLoops;
    const int per = (nl + c - 1) / c;
    const bool fused = resolve_mode(p, batch) == RSFT_MODE_FUSED;
    int launches = 0;
    for (int a = 0; a < nl; a += per) {
      const int m = std::min(per, nl - a);
      // loops [a, a + m) of the [batch][nl][...] outputs: frame-strided (fused kernels take
      // the strides; split mode runs one frame per launch)
      for (int64_t f = 0; f < (fused ? 1 : batch); ++f) {
        const char* xf = reinterpret_cast<const char*>(d_x) + (size_t)f * p->ntot * 8;
        uint32_t* bmf = bm + ((size_t)f * nl + a) * p->dev.wpl;
        void* spf = spectra ? reinterpret_cast<char*>(spectra) + ((size_t)f * nl + a) * p->btot * 8 : nullptr;
        p->last_launches = 0;
        rsft_status s = fused ? launch_fused_lp(p, loop_pad(m), xf, batch, l0 + a, m, bmf, spf, st,
                                                (int64_t)nl * p->dev.wpl, (int64_t)nl * p->btot)
                              : launch_execute(p, xf, 1, l0 + a, m, bmf, spf, st);
        if (s) return s;
        launches += p->last_launches;
      }
    }
    p->last_launches = launches;
    return RSFT_OK;
  }
  int mode = resolve_mode(p, batch);
  int lp = loop_pad(nl);
  if (mode == RSFT_MODE_FUSED) { RSFT_DISPATCH_LP(launch_fused_t, lp, p, d_x, batch, l0, nl, bm, spectra, st); }
  if (mode == RSFT_MODE_SPLIT) { RSFT_DISPATCH_LP(launch_split_t, lp, p, d_x, batch, l0, nl, bm, spectra, st); }
  return RSFT_E_UNSUPPORTED;
}

rsft_status launch_detect_compact(rsft_plan_s* p, const uint32_t* bm, int64_t batch, uint32_t* det,
                                  int64_t* idx, int64_t capacity, int64_t* d_count, cudaStream_t st);   // vote.cu
bool vote1d_usable(const rsft_plan_s* p);                                                              // vote.cu
rsft_status launch_scan_write(rsft_plan_s* p, int64_t batch, uint32_t* det, int64_t* idx, int64_t capacity,
                              int64_t* d_count, bool list, cudaStream_t st);                          // vote.cu
bool fused2v_ok(const rsft_plan_s* p);                                                                 // fused2v.cu
rsft_status launch_fused2v(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm, uint32_t* det,
                           unsigned long long* rcount, uint32_t* slots, int list_cap, cudaStream_t st);
rsft_status upload_twiddles_2v(cudaStream_t st);

// Whole pipeline on one batch.  Fused-mode plans: one fold kernel that also votes (D = 1:
// k_gather1d with vote warps; D = 2: k_fused2v, whose epilogue warps FFT and vote frame f while
// the fold warps stream frame f + 1 -- the synchronous per-frame epilogue vote measured slower at
// c4 because the CTA's TMA stream stalled while it voted) + the scan / writer; other plans:
// execute (all loops) + detect_compact.
rsft_status launch_run(rsft_plan_s* p, const void* d_x, int64_t batch, uint32_t* bm, uint32_t* det, int64_t* idx,
                       int64_t capacity, int64_t* d_count, cudaStream_t st) {
  {
    // D = 1 gather plans: fold + vote in one kernel (RSFT_FUSED_RUN=0, read per launch, splits them)
    const char* fr = getenv("RSFT_FUSED_RUN");
    if (!(fr && fr[0] == '0') && p->D == 1 && gather1d_taps(p) && vote1d_usable(p) && batch <= p->dev.region_capacity) {
      const bool list = p->dev.region_slots != nullptr;
      rsft_status s = launch_gather1d_voted(p, d_x, batch, bm, det, p->dev.region_state,
                                            list ? p->dev.region_slots : nullptr, (int)p->dev.list_cap, st);
      if (s == RSFT_OK) return launch_scan_write(p, batch, det, idx, capacity, d_count, list, st);
      if (s != RSFT_E_UNSUPPORTED) return s;
    }
  }
  {
    // D = 2 fused plans (c2 / c4): fold warps + epilogue / vote warps in one kernel (fused2v.cu)
    const char* fr = getenv("RSFT_FUSED_RUN");
    if (!(fr && fr[0] == '0') && fused2v_ok(p) && resolve_mode(p, batch) == RSFT_MODE_FUSED &&
        batch <= p->dev.region_capacity) {
      const bool list = p->dev.region_slots != nullptr;
      rsft_status s = launch_fused2v(p, d_x, batch, bm, det, p->dev.region_state, list ? p->dev.region_slots : nullptr,
                                     (int)p->dev.list_cap, st);
      if (s == RSFT_OK) return launch_scan_write(p, batch, det, idx, capacity, d_count, list, st);
      if (s != RSFT_E_UNSUPPORTED) return s;
    }
  }
  rsft_status s = launch_execute(p, d_x, batch, 0, p->L, bm, nullptr, st);
  if (s) return s;
  return launch_detect_compact(p, bm, batch, det, idx, capacity, d_count, st);
}

rsft_status upload_twiddles(cudaStream_t st) {
  float2 tw[128];
  for (int k = 0; k < 128; ++k) {
    double a = -2.0 * M_PI * (double)k / 128.0;
    tw[k] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  rsft_status s = check(cudaMemcpyToSymbolAsync(c_tw128, tw, sizeof(tw), 0, cudaMemcpyHostToDevice, st), "twiddles");
  if (s) return s;
  float2 t5[512];
  for (int k = 0; k < 512; ++k) {
    double a = -2.0 * M_PI * (double)k / 512.0;
    t5[k] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  s = check(cudaMemcpyToSymbolAsync(c_tw512, t5, sizeof(t5), 0, cudaMemcpyHostToDevice, st), "twiddles");
  if (s) return s;
  return upload_twiddles_2v(st);
}

}  // namespace rsft
