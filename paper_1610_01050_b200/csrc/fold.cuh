// Fold / FFT device helpers shared by the fused fold kernels (kernels.cu: k_fused, k_gather1d,
// the split folds; fused2v.cu: the warp-specialised D = 2 rsft_run kernel).  Header-only.
#pragma once
#include "kcommon.cuh"

namespace rsft {

// Column weights + lane fold.  Lane owns columns c = base + 2*lane_col + e (e = 0,1); its
// residues (2*lane + e) mod B_last (B_last <= 64 divides 64).  Lanes whose index agrees
// mod B_last/2 share residues and are summed with xor shuffles.  After the call lanes
// < max(B_last/2,1) hold residue sums for residues 2*lane + e (e < min(B_last,2)).
template <int LP>
__device__ __forceinline__ void colweight(float2 (&acc)[LP][2], const float* __restrict__ hlast,
                                          int l0, int nl, int nlast, int col) {
#pragma unroll
  for (int l = 0; l < LP; ++l) {
    float2 hc = make_float2(0.f, 0.f);
    if (l < nl) hc = __ldg(reinterpret_cast<const float2*>(hlast + (size_t)(l0 + l) * nlast + col));
    acc[l][0].x *= hc.x; acc[l][0].y *= hc.x;
    acc[l][1].x *= hc.y; acc[l][1].y *= hc.y;
  }
}

template <int LP>
__device__ __forceinline__ void colweight_plain(float2 (&acc)[LP][2], const float* hl, int nlast, int col) {
#pragma unroll
  for (int l = 0; l < LP; ++l) {
    const float2 hc = *reinterpret_cast<const float2*>(hl + (size_t)l * nlast + col);
    acc[l][0].x *= hc.x; acc[l][0].y *= hc.x;
    acc[l][1].x *= hc.y; acc[l][1].y *= hc.y;
  }
}

template <int LP>
__device__ __forceinline__ void lane_fold(float2 (&acc)[LP][2], int blast) {
  for (int off = blast >= 2 ? blast / 2 : 1; off < 32; off <<= 1) {
#pragma unroll
    for (int l = 0; l < LP; ++l)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, acc[l][e].x, off),
                                     __shfl_xor_sync(0xffffffffu, acc[l][e].y, off));
        acc[l][e] = __fadd2_rn(acc[l][e], o);
      }
  }
  if (blast == 1) {
#pragma unroll
    for (int l = 0; l < LP; ++l) acc[l][0] = __fadd2_rn(acc[l][0], acc[l][1]);
  }
}

// ------------------------------------------------------------------------------------
// TMA bulk-copy pipeline (per warp): lane 0 streams row segments of x global -> shared
// with cp.async.bulk (SASS UBLKCP) into an S-deep ring, completion tracked by one
// mbarrier per stage (expect_tx / complete_tx); all lanes wait on the stage's phase, read
// their 16 B with LDS.128 and run the FFMA2 fold.  Bytes in flight per warp are explicit
// ((S-1) x U x 512 B), independent of registers and of ptxas scheduling.
// One row group: U row-loads of 32 float4 (512 B) per warp, already in the stage buffer.
// acc[l] += w_row[l] * x for each row.  Rows past the end of a class are zero-filled by
// the TMA (out-of-bounds box rows) and carry the zero weight row, so they add nothing.
template <int LP, int U, bool INIT = false>
__device__ __forceinline__ void fold_group(float2 (&acc)[LP][2], const float4* __restrict__ buf, int lane,
                                           const float* const (&wrow)[U]) {
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = buf[u * 32 + lane];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if constexpr (LP % 4 == 0) {                   // 16-B weight loads (rows are 16-B aligned)
      const float4* wr = reinterpret_cast<const float4*>(wrow[u]);
#pragma unroll
      for (int l4 = 0; l4 < LP / 4; ++l4) {
        const float4 w = wr[l4];
        const float wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (INIT && u == 0) {                    // first row of the group: acc = w * v
            acc[4 * l4 + i][0] = __fmul2_rn(make_float2(wv[i], wv[i]), make_float2(v[u].x, v[u].y));
            acc[4 * l4 + i][1] = __fmul2_rn(make_float2(wv[i], wv[i]), make_float2(v[u].z, v[u].w));
          } else {
            mac(acc[4 * l4 + i][0], wv[i], v[u].x, v[u].y);
            mac(acc[4 * l4 + i][1], wv[i], v[u].z, v[u].w);
          }
        }
      }
    } else {
      const float2* wr = reinterpret_cast<const float2*>(wrow[u]);
#pragma unroll
      for (int l2 = 0; l2 < LP / 2; ++l2) {
        const float2 w = wr[l2];
        const float wv[2] = {w.x, w.y};
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (INIT && u == 0) {
            acc[2 * l2 + i][0] = __fmul2_rn(make_float2(wv[i], wv[i]), make_float2(v[u].x, v[u].y));
            acc[2 * l2 + i][1] = __fmul2_rn(make_float2(wv[i], wv[i]), make_float2(v[u].z, v[u].w));
          } else {
            mac(acc[2 * l2 + i][0], wv[i], v[u].x, v[u].y);
            mac(acc[2 * l2 + i][1], wv[i], v[u].z, v[u].w);
          }
        }
      }
    }
  }
}

__device__ __forceinline__ float2 shfl_xor2(float2 v, int m) {
  return make_float2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// Select form of warp_dif below (no per-lane constants beyond stw: for register-capped kernels).
__device__ __forceinline__ float2 warp_dif_sel(float2 x, int lane, int lgb, const float2 (&stw)[5]) {
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int h = 16 >> q;
    if ((2 * h) > (1 << lgb)) continue;           // warp-uniform
    const float2 p = shfl_xor2(x, h);
    x = (lane & h) ? cmul(csub(p, x), stw[q]) : cadd(x, p);
  }
  return x;
}

// 2^lgb-point DIF across lanes (x = element lane mod 2^lgb, lgb <= 5): lane p ends with
// X[brev(p mod 2^lgb)].  Stage q (h = 16 >> q) pairs lanes p, p ^ h: the lower one keeps x + p,
// the upper one (p - x) W_{2h}^{lane mod h}.  Written branch-free with per-lane constants (DifTw):
// y = sg x + partner, then y w with w = 1 on the lower lane -- one FFMA2 + one FMUL2 + one FFMA2
// per stage and value in SASS (the select form issued 4 FADD + 4 FMUL/FFMA + 4 moves).
struct DifTw {
  float2 cd[5], mdc[5];                              // w = (c, d) and (-d, c)
  float sg[5];                                       // +1 lower lane, -1 upper lane
};
// stw[q] = W_{2h}^{lane & (h-1)} for h = 16 >> q
__device__ __forceinline__ DifTw dif_tw(int lane, const float2 (&stw)[5]) {
  DifTw t;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const bool up = (lane & (16 >> q)) != 0;
    const float2 w = up ? stw[q] : make_float2(1.f, 0.f);
    t.cd[q] = w;
    t.mdc[q] = make_float2(-w.y, w.x);
    t.sg[q] = up ? -1.f : 1.f;
  }
  return t;
}
__device__ __forceinline__ float2 warp_dif(float2 x, int lgb, const DifTw& t) {
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int h = 16 >> q;
    if ((2 * h) > (1 << lgb)) continue;           // warp-uniform
    const float2 p = shfl_xor2(x, h);
    const float2 y = __ffma2_rn(make_float2(t.sg[q], t.sg[q]), x, p);
    x = __ffma2_rn(make_float2(y.y, y.y), t.mdc[q], __fmul2_rn(make_float2(y.x, y.x), t.cd[q]));
  }
  return x;
}

}  // namespace rsft
