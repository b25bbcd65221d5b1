// Internal definitions shared by the host plan (plan.cpp) and the CUDA side (kernels.cu).
// Product code only: nothing here is shared with the oracle (oracle/ is NumPy).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <vector_types.h>

#include "../../include/rsft.h"

namespace rsft {

constexpr int kMaxDim = 3;
constexpr int kMaxLoops = 64;         // L <= 63: 6 bit planes of vote counts
constexpr int kMaxLaunchLoops = 32;   // loops per fold launch (more loops: several passes)
constexpr int kSizingSms = 148;     // host-only plan: workspace sized for a B200 (rsft.h)
constexpr int kMaxB = 64;          // register FFT lines and lane folds support B_d <= 64
constexpr int kMaxB1d = 256;       // D = 1 gather form (k_gather1d): B = 128, 256 as 4 / 8 buckets per lane
constexpr int64_t kChunkWords = 8192;  // compaction chunk: words of the detection bitmap
constexpr int kThreads = 256;          // CTA size of most kernels
constexpr int kThreadsFft = 1024;      // split-mode outer FFT: one L2 round trip per thread
// Fused fold kernel shapes (threads per CTA, CTAs per SM, ring stages per warp, 512-B rows per
// stage), chosen by dimension (fused_cfg): D = 2 frames stream long residue classes, so one
// 16-warp CTA per SM with 4-KiB boxes (2 stages) keeps the most bytes in flight per box issued
// (c4: 1.40 vs 1.44 ms); D = 1 frames are short and favour two 8-warp CTAs with 2-KiB boxes.
struct FusedCfg { int threads, ctas, stages, u; };
#ifndef RSFT_F2
#define RSFT_F2 512, 1, 2, 8
#endif
constexpr FusedCfg kFused2D = {RSFT_F2};
constexpr FusedCfg kFused1D = {256, 2, 3, 4};
#ifndef RSFT_NO_TMA
#define RSFT_NO_TMA 0
#endif
#ifndef RSFT_SPLIT_ORDER
#define RSFT_SPLIT_ORDER 1
#endif
#ifndef RSFT_NO_FOLD_COMPUTE
#define RSFT_NO_FOLD_COMPUTE 0
#endif
#ifndef RSFT_SPLIT_STAGES
#define RSFT_SPLIT_STAGES 2
#endif
#ifndef RSFT_SPLIT_U
#define RSFT_SPLIT_U 16
#endif
#ifndef RSFT_SPLIT_THREADS
#define RSFT_SPLIT_THREADS 256
#endif
#ifndef RSFT_SPLIT_CTAS
#define RSFT_SPLIT_CTAS 1
#endif
constexpr int kStagesSplit = RSFT_SPLIT_STAGES;   // split-mode fold: per-warp ring depth of ...
constexpr int kUSplit = RSFT_SPLIT_U;             // ... U-slot (U x 512 B) TMA boxes
constexpr int kThreadsSplit = RSFT_SPLIT_THREADS; // threads per CTA ...
constexpr int kCtasSplit = RSFT_SPLIT_CTAS;       // ... and CTAs per SM the kernel is built for
constexpr int kSplitUnitsPerWarp = 4;
constexpr int kListCapMin = 2048;                // vote: region-local index slots per region, at least ...
constexpr int kListCapMax = 8192;                // ... and at most (as many as 256 MiB of slots allow)
constexpr size_t kListSlotsBytes = 256ull << 20;
constexpr int kSplitDftBytes = 16384;            // split-mode last-dim DFT factor table [r][l][k] (float4) up to this size
constexpr int kSplitHlastBytes = 16384;          // column-weight table kept in smem up to this size             // chunking target: >= this many units per warp

#ifdef __CUDACC__
#ifndef RSFT_MMA_DEBUG
#define RSFT_MMA_DEBUG 0   // k_split_mma measurement variants: 1 = no operand work, 2 = no TMA, 3 = no MMA
#endif
#define RSFT_HD __host__ __device__
#else
#define RSFT_HD
#endif

// Per-warp shared-memory carve-up of the split-mode fold (byte offsets inside a warp's
// region): TMA ring, its mbarriers, double-buffered staged weights hs and the segment slot.
// D == 2: hs rows = the chunk's a0 rows (row weights h0), zero-padded to a whole box;
// D == 3: hs = A0c h0 rows + A1 h1 rows (zero-padded to a whole box).  slot [nl][B_last]:
// the unit's folded residue sums (segments accumulate there).
struct SplitWarpLayout {
  int ring, bars, hs, hs_stride, slot, total;
};
RSFT_HD inline int split_pad_rows(int rows, int br) { return rows < br ? br : rows; }
RSFT_HD inline SplitWarpLayout split_warp_layout(int D, int lpad, int nl, int a0c, int a1, int blast, int nseg,
                                                 int rpw) {
  SplitWarpLayout w;
  const int br = kUSplit * rpw;
  int off = 0;
  w.ring = off; off += kStagesSplit * kUSplit * 512;
  w.bars = off; off += ((kStagesSplit * 8 + 15) / 16) * 16;
  const int hs_rows = D == 3 ? a0c + split_pad_rows(a1, br) : split_pad_rows(a0c, br);
  w.hs = off; w.hs_stride = ((hs_rows * lpad * 4 + 15) / 16) * 16; off += 2 * w.hs_stride;
  w.slot = off; off += nl * blast * 8;
  w.total = ((off + 127) / 128) * 128;
  return w;
}

// Split fold, D == 3 with short a1 runs: a TMA box of BR = kUSplit * rpw rows spans
// G = BR / A1 whole a0 groups (returns G, or 0 when the 4-D a1-run boxes are used).
RSFT_HD inline int split_multi_g(int D, int lpad, int a1, int a0c, int rpw, int nseg) {
  const int br = kUSplit * rpw;
  if (D != 3 || lpad > 16 || nseg != 1 || a1 >= br || br % a1 != 0 || a1 % rpw != 0) return 0;
  const int g = br / a1;
  if (a1 / rpw > 8 || a0c % g != 0) return 0;
  return g;
}

// Per-loop device record: schedule + threshold (Def. 1; Eq. tpd).
struct LoopDev {
  int32_t sig[kMaxDim];
  int32_t sinv[kMaxDim];
  int32_t tau[kMaxDim];
  float gamma;
  int32_t pad;
};

// Plan view passed by value to every kernel.
struct PlanDev {
  int32_t D;
  int32_t L;                       // loops in the plan
  int32_t mu;
  int32_t nplanes;                 // bit planes of the vote counter (L < 2^nplanes)
  int32_t n[kMaxDim], b[kMaxDim], a[kMaxDim];
  int32_t lgn[kMaxDim], lgb[kMaxDim], lga[kMaxDim];
  int32_t shift[kMaxDim];          // 1 if B_d < N_d (half-bucket twiddle, L1), else 0
  int64_t ntot, btot;
  int32_t wpl;                     // bitmap words per loop = ceil(btot/32)
  int32_t nlast, blast;            // N_{D-1}, B_{D-1}
  int64_t rows;                    // ntot / nlast
  int32_t bouter;                  // prod_{d<D-1} B_d
  int32_t aouter;                  // prod_{d<D-1} A_d (rows per outer residue class)
  const LoopDev* loops;            // [L]
  const float* h[kMaxDim];         // [L][N_d] fp32 weight tables h_{l,d}[s] (I3)
  float2* fbuf;                    // split mode folded spectra [batch][L][B_last][nchunk][B_outer] (fold -> FFT)
  int64_t fbuf_capacity;           // float2 elements
  const float* ht[kMaxDim];        // d < D-1: class-major weights [B_d][A_d][L], ht[r][a][l] = h[l][r + B_d a]
  long long* chunk_counts;         // compaction scratch
  int64_t chunk_capacity;
  const uint32_t* xmask;           // [L][B_last][N_last/32] last-dim bucket masks, or null
  const uint32_t* ntab;            // nibble tables of the masks [L][B_last/4][16][N_last/32], or null
  unsigned long long* region_state; // per-region detection counts -> offsets (rsft_detect_compact)
  int64_t region_capacity;
  uint32_t* region_slots;          // per-region local index lists [region_capacity][list_cap] (or null)
  int32_t list_cap;                // index slots per region
  uint32_t* etab;                  // D == 3 vote: E words for every dim-0 bucket [batch][L][B0][B1][W] (or null)
  int64_t etab_frames;             // frames etab holds
  const float* bwin[kMaxDim];      // Bartlett: fp32 pre-windows w_d [N_d]
  const float* bone;               // 1.0f (window of an absent dimension)
  const float2* btw;               // e^{-j 2 pi k / 4096}, k < 2048 (Bartlett FFTs)
};

constexpr size_t kMaxXmaskBytes = 48 * 1024;   // vote expansion masks kept in smem
constexpr size_t kMaxNibbleBytes = 64 * 1024;  // vote nibble tables (4x the masks) kept in smem
constexpr size_t kMaxEtabBytes = 64ull << 20;  // D == 3 vote: precomputed E table for all dim-0 buckets, up to this

struct Workspace {
  size_t loops_off, h_off[kMaxDim], ht_off[kMaxDim], fbuf_off, fbuf_bytes, chunk_off, xmask_off, xmask_bytes, region_off, slots_off, slots_bytes, etab_off, etab_bytes, ntab_off, ntab_bytes, bwin_off[kMaxDim], bone_off, btw_off, total;
  int64_t region_capacity;
  int64_t list_cap;
  int64_t chunk_capacity;
};

}  // namespace rsft

struct rsft_plan_s {
  rsft_params P;
  int D = 1, L = 1, mu = 1;
  int64_t n[3] = {1, 1, 1}, b[3] = {1, 1, 1}, a[3] = {1, 1, 1}, W[3] = {0, 0, 0};
  int64_t ntot = 1, btot = 1;
  std::vector<int64_t> sigma, sinv, tau;          // [L*D]
  std::vector<double> prewin[3], flatg[3];        // fp64 windows [N_d]
  std::vector<double> hd[3];                      // fp64 weights [L][N_d]
  std::vector<float> hf[3];                       // fp32 weights [L][N_d]
  std::vector<double> beta, gamma;                // [L]
  std::vector<uint32_t> xmask;                    // [L][B_last][N_last/32] (may be empty)
  std::vector<uint32_t> ntab;                     // vote nibble tables [L][B_last/4][16][N_last/32] (may be empty)
  rsft::Workspace ws{};
  // binding
  bool bound = false;
  int device = -1;
  int want_device = -1;                           // rsft_plan(device): bind only there
  int num_sms = 148;
  void* d_ws = nullptr;
  rsft::PlanDev dev{};
  int32_t last_launches = 0;
};

namespace rsft {
// plan.cpp
rsft_status rebuild_tables(rsft_plan_s* p);
void layout_workspace(rsft_plan_s* p);
int resolve_mode(const rsft_plan_s* p, int64_t batch);
int gather1d_taps(const rsft_plan_s* p);
int loop_pad(int nl);
size_t fused_smem_bytes(const rsft_plan_s* p, int nl, int lpad, int stages = 0);
inline FusedCfg fused_cfg(int D) { return D == 2 ? kFused2D : kFused1D; }
size_t split_smem_bytes(const rsft_plan_s* p, int nl, int lpad, int64_t a0c, int seg_L = 0);
int split_lg_chunks(const rsft_plan_s* p, int64_t batch, int nl, int64_t a0_count, int64_t warps_total);
void set_error(const std::string& s);
}  // namespace rsft
