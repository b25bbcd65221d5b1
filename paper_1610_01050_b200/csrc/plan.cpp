// Host plan of the RSFT hot path: validation, sigma/tau schedule, windows, the per-loop
// weight tables of the factored fold, beta_l and gamma_l.  Host only (no CUDA calls).
//
// Independent of the oracle (oracle/rsft_ref.py, NumPy): same definitions, written again.
// Citations: P:<line> = /root/reference/PAPER.md; Lnn = DESIGN.md readings.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>

#include "rsft_internal.h"

namespace rsft {

static thread_local std::string g_err;
void set_error(const std::string& s) { g_err = s; }

static bool is_pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }
static int ilog2(int64_t v) { int r = 0; while ((int64_t(1) << r) < v) ++r; return r; }

// SplitMix64 draw #ctr of stream `seed` (reading L5; Alg. 1 l.2 "Generate a set of sigma
// randomly for each dimension").
static uint64_t splitmix64(uint64_t seed, uint64_t ctr) {
  uint64_t z = seed + (ctr + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// sigma^{-1} mod 2^k by Newton iteration x <- x (2 - s x) (Eq. mod_inv).
static int64_t inv_mod_pow2(int64_t s, int64_t n) {
  if (n == 1) return 0;
  uint64_t x = 1, us = (uint64_t)s;
  for (int i = 0; i < 7; ++i) x = x * (2 - us * x);
  return (int64_t)(x & (uint64_t)(n - 1));
}

// Periodic Hann, w[n] = sin^2(pi n / N) (reading L3).
static std::vector<double> hann(int64_t n) {
  std::vector<double> w(n);
  for (int64_t i = 0; i < n; ++i) { double s = std::sin(M_PI * (double)i / (double)n); w[i] = s * s; }
  return w;
}

// Symmetric Dolph-Chebyshev taper of odd length M, peak 1.  Frequency
// samples What[k] = T_{M-1}(x0 cos(pi k / M)), x0 = cosh(arccosh(10^{A/20}) / (M-1)), real
// inverse DFT, centred at m = (M-1)/2 (reading L19).
static std::vector<double> dolph_chebyshev(int64_t m, double atten_db) {
  std::vector<double> out(m, 1.0);
  if (m == 1) return out;
  const int64_t order = m - 1;
  const double r = std::pow(10.0, atten_db / 20.0);
  const double x0 = std::cosh(std::acosh(r) / (double)order);
  std::vector<double> t(m), ctab(m), w(m);
  for (int64_t k = 0; k < m; ++k) {
    double x = x0 * std::cos(M_PI * (double)k / (double)m);
    double ax = std::fabs(x);
    if (ax <= 1.0) t[k] = std::cos((double)order * std::acos(x));
    else t[k] = std::cosh((double)order * std::acosh(ax)) * ((order % 2 && x < 0) ? -1.0 : 1.0);
    ctab[k] = std::cos(2.0 * M_PI * (double)k / (double)m);
  }
  for (int64_t j = 0; j < m; ++j) {          // Re IDFT: (1/M) sum_k t[k] cos(2 pi k j / M)
    double acc = 0.0;
    int64_t idx = 0;
    for (int64_t k = 0; k < m; ++k) { acc += t[k] * ctab[idx]; idx += j; if (idx >= m) idx -= m; }
    w[j] = acc / (double)m;
  }
  double mx = -1e300;
  for (int64_t i = 0; i < m; ++i) {
    int64_t k = ((i - (m - 1) / 2) % m + m) % m;
    out[i] = w[k];
    if (out[i] > mx) mx = out[i];
  }
  for (auto& v : out) v /= mx;
  return out;
}

static std::vector<double> prewindow(const rsft_params& P, int64_t n) {
  if (P.prewin == RSFT_WIN_HANN) return hann(n);
  if (P.prewin == RSFT_WIN_CHEB) {
    auto w = dolph_chebyshev(n + 1, P.prewin_param);   // periodic: N+1 points, drop the last
    w.resize(n);
    return w;
  }
  return std::vector<double>(n, 1.0);
}

// Real even cyclic flat-window prototype (readings L1, L2, L13):
// g[t] = sinc(t_c / B) * Cheb_{W+1}(t_c) for |t_c| <= W/2, else 0; B == N -> g = 1.
static std::vector<double> flat_proto(int64_t n, int64_t b, int64_t w, double atten) {
  std::vector<double> g(n, 0.0);
  if (b == n) { for (auto& v : g) v = 1.0; return g; }
  if (w == 0) w = n;
  auto taper = dolph_chebyshev(w + 1, atten);
  for (int64_t t = 0; t < n; ++t) {
    int64_t tc = t < n / 2 ? t : t - n;
    if (std::llabs(tc) > w / 2) continue;
    double u = (double)tc / (double)b;
    double s = (tc == 0) ? 1.0 : std::sin(M_PI * u) / (M_PI * u);
    g[t] = s * taper[tc + w / 2];
  }
  return g;
}

// Factored fold weights (identity I3): for loop l and dimension d,
//   h_{l,d}[s] = w_d[s] * g_d[t] * (-1)^{floor(t / B_d)},  t = sigma^{-1} (s - tau) mod N_d,
// so that f_l[b] = e^{-j pi b/B} sum_{s : s = r (mod B)} x[s] prod_d h_{l,d}[s_d] with
// b_d = sigma^{-1}(r_d - tau_d) mod B_d (Def. 1-2 + the half-bucket shift of L1).
rsft_status rebuild_tables(rsft_plan_s* p) {
  const int D = p->D, L = p->L;
  p->beta.assign(L, 1.0);
  p->gamma.assign(L, 0.0);
  for (int d = 0; d < D; ++d) {
    const int64_t n = p->n[d], b = p->b[d];
    p->hd[d].assign((size_t)L * n, 0.0);
    p->hf[d].assign((size_t)L * n, 0.0f);
    for (int l = 0; l < L; ++l) {
      const int64_t si = p->sinv[l * D + d], ta = p->tau[l * D + d];
      double ss = 0.0;
      for (int64_t s = 0; s < n; ++s) {
        int64_t t = (int64_t)(((__int128)si * (((s - ta) % n + n) % n)) % n);
        double sign = (b < n && ((t / b) & 1)) ? -1.0 : 1.0;
        double h = p->prewin[d][s] * p->flatg[d][t] * sign;
        p->hd[d][(size_t)l * n + s] = h;
        p->hf[d][(size_t)l * n + s] = (float)h;
        ss += h * h;
      }
      p->beta[l] *= ss;              // beta = ||Wbar P_sigma w||^2 (Eq. alpha_beta)
    }
  }
  // Vote expansion masks (identity I1, Def. 3): bit j of X[l][k][w] is set iff location
  // i = 32 w + j of the last dimension maps to bucket k = floor(B [sigma i]_N / N).
  {
    const int ld = D - 1;
    const int64_t n = p->n[ld], b = p->b[ld], W = n / 32;
    const size_t bytes = (size_t)L * b * W * 4;
    p->xmask.clear();
    if (bytes <= kMaxXmaskBytes && b <= kMaxB) {
      p->xmask.assign((size_t)L * b * W, 0u);
      for (int l = 0; l < L; ++l) {
        const int64_t s = p->sigma[l * D + ld];
        for (int64_t i = 0; i < n; ++i) {
          const int64_t k = (int64_t)(((__int128)s * i) % n) * b / n;
          p->xmask[((size_t)l * b + k) * W + (i >> 5)] |= 1u << (i & 31);
        }
      }
    }
    // nibble tables NT[l][g][m][w] = OR of X[l][4 g + q][w] over the set bits q of m (the vote
    // expands 4 buckets per lookup); plan-constant, copied into shared memory by k_vote
    p->ntab.clear();
    if (!p->xmask.empty() && b >= 4 && 16 * p->xmask.size() <= kMaxNibbleBytes) {
      const int64_t ng = b / 4;
      p->ntab.assign((size_t)L * ng * 16 * W, 0u);
      for (int l = 0; l < L; ++l)
        for (int64_t g = 0; g < ng; ++g)
          for (int m = 0; m < 16; ++m)
            for (int64_t w = 0; w < W; ++w) {
              uint32_t e = 0;
              for (int q = 0; q < 4; ++q)
                if ((m >> q) & 1) e |= p->xmask[((size_t)l * b + 4 * g + q) * W + w];
              p->ntab[(((size_t)l * ng + g) * 16 + m) * W + w] = e;
            }
    }
  }
  for (int l = 0; l < L; ++l)        // Eq. tpd with P~_fa = P_fa per loop (L8)
    p->gamma[l] = p->P.gamma_override > 0 ? p->P.gamma_override
                                          : p->P.noise_var * p->beta[l] * std::log(1.0 / p->P.p_fa);
  p->bound = false;
  return RSFT_OK;
}

int loop_pad(int nl) {
  static const int pads[] = {2, 4, 6, 8, 12, 16, 24, 32};
  for (int v : pads) if (nl <= v) return v;
  return -1;
}

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

void layout_workspace(rsft_plan_s* p) {
  Workspace& w = p->ws;
  size_t off = 0;
  w.loops_off = off; off = align256(off + sizeof(LoopDev) * p->L);
  for (int d = 0; d < 3; ++d) {
    w.h_off[d] = off;
    if (d < p->D) off = align256(off + sizeof(float) * (size_t)p->L * p->n[d]);
  }
  for (int d = 0; d < 3; ++d) {                    // class-major copies for the split fold
    w.ht_off[d] = off;
    if (d + 1 < p->D) off = align256(off + sizeof(float) * (size_t)p->L * p->n[d]);
  }
  // split mode: folded spectra per dim-0 chunk, sized for the largest batch x chunks product
  // the launcher can choose (batch <= max_batch; chunks from split_lg_chunks)
  w.fbuf_off = off;
  w.fbuf_bytes = 0;
  if (p->D >= 2) {
    const int64_t warps = (int64_t)kSizingSms * (kThreadsSplit / 32) * kCtasSplit;   // rsft.h: 148-SM sizing
    int64_t best = p->P.max_batch;
    for (int64_t b = 1; b <= std::min<int64_t>(p->P.max_batch, 64); b *= 2)
      best = std::max(best, b << split_lg_chunks(p, b, p->L, p->a[0], warps));
    w.fbuf_bytes = (size_t)best * p->L * p->btot * 8;
    off = align256(off + w.fbuf_bytes);
  }

  int64_t dw = (p->ntot + 31) / 32;
  int64_t chunks = (p->P.max_batch * dw + kChunkWords - 1) / kChunkWords;
  w.chunk_capacity = chunks;
  w.chunk_off = off; off = align256(off + sizeof(long long) * (size_t)(chunks + 2));
  {
    const int64_t n = p->n[p->D - 1], b = p->b[p->D - 1];
    w.xmask_bytes = (size_t)p->L * b * (n / 32) * 4;
    if (w.xmask_bytes > kMaxXmaskBytes || b > kMaxB) w.xmask_bytes = 0;   // the vote's mask forms: B_last <= 64
  }
  w.xmask_off = off; off = align256(off + w.xmask_bytes);
  w.ntab_bytes = (w.xmask_bytes && p->b[p->D - 1] >= 4 && 4 * w.xmask_bytes <= kMaxNibbleBytes) ? 4 * w.xmask_bytes : 0;
  w.ntab_off = off; off = align256(off + w.ntab_bytes);
  w.region_capacity = p->P.max_batch * (p->D == 3 ? p->n[0] : 1) + 2;
  w.region_off = off; off = align256(off + 8 * (size_t)w.region_capacity);
  w.slots_off = off;                               // vote index lists (list_cap per region)
  {
    int64_t cap = kListCapMax;
    while (cap > kListCapMin && (size_t)w.region_capacity * cap * 4 > kListSlotsBytes) cap >>= 1;
    w.list_cap = cap;
  }
  w.slots_bytes = (size_t)w.region_capacity * w.list_cap * 4;
  off = align256(off + w.slots_bytes);
  w.etab_off = off;                                // D == 3 vote: E words for every dim-0 bucket
  w.etab_bytes = 0;
  if (p->D == 3 && w.xmask_bytes) {
    const size_t per = (size_t)p->L * p->b[0] * p->b[1] * (p->n[2] / 32) * 4;
    size_t fr = (size_t)p->P.max_batch;
    while (fr > 1 && fr * per > kMaxEtabBytes) fr >>= 1;
    if (fr * per <= kMaxEtabBytes) w.etab_bytes = fr * per;
    off = align256(off + w.etab_bytes);
  }
  for (int d = 0; d < 3; ++d) {                    // Bartlett baseline tables
    w.bwin_off[d] = off;
    if (d < p->D) off = align256(off + 4 * (size_t)p->n[d]);
  }
  w.bone_off = off; off = align256(off + 4);
  w.btw_off = off; off = align256(off + 8 * 2048);
  w.total = off;
}

// Shared-memory footprints (must match the carve-up at the top of k_fused / k_split_fold).
size_t fused_smem_bytes(const rsft_plan_s* p, int nl, int lpad, int stages) {
  FusedCfg fc = fused_cfg(p->D);
  if (stages > 0) fc.stages = stages;
  const int nwarps = fc.threads / 32;
  int64_t blast = p->b[p->D - 1], nlast = p->n[p->D - 1];
  int64_t bouter = p->btot / blast;
  int64_t nseg = nlast / 64;
  int64_t groups = p->D == 1 ? (nseg < 8 ? nseg : 8) : 1;
  int64_t n0 = p->D == 2 ? p->n[0] : 1;
  size_t ring = (size_t)nwarps * fc.stages * fc.u * 512 + (size_t)nwarps * fc.stages * 8;
  size_t fbytes = (((size_t)groups * nl * bouter * (blast + 1) + 1) & ~size_t(1)) * 8 + 128 * 8;
  return ring + fbytes + (size_t)(n0 + 1) * lpad * 4;
}

size_t split_smem_bytes(const rsft_plan_s* p, int nl, int lpad, int64_t a0c, int seg_L) {
  const int D = p->D;
  const int64_t nlast = p->n[D - 1];
  const int nseg = nlast >= 64 ? (int)(nlast / 64) : 1;
  SplitWarpLayout w = split_warp_layout(D, lpad, nl, (int)a0c, D == 3 ? (int)p->a[1] : 1, (int)p->b[D - 1], nseg,
                                        nlast >= 64 ? 1 : (int)(64 / nlast));
  const size_t hl = (size_t)(seg_L > 0 ? seg_L + lpad : lpad) * nlast * 4;     // segment mode: all loops
  const size_t dft = (size_t)(seg_L > 0 ? seg_L : lpad) * p->b[D - 1] * p->b[D - 1] * 16;
  return (size_t)(kThreadsSplit / 32) * w.total + (hl <= (size_t)kSplitHlastBytes ? hl : 0) + 128 * 8 +
         (dft <= (size_t)kSplitDftBytes ? dft : 0);
}

// Split-mode work units are (frame, outer residue class, dim-0 chunk) per WARP.  Chunk the
// dim-0 rows (2^lg chunks) until there are >= kSplitUnitsPerWarp units per resident warp
// with < 5 % tail loss, keeping >= 32 rows per unit (D == 2: a chunk holds >= 1 TMA box).
int split_lg_chunks(const rsft_plan_s* p, int64_t batch, int nl, int64_t a0_count, int64_t warps_total) {
  const int D = p->D;
  const int64_t nlast = p->n[D - 1];
  const int64_t bouter = p->btot / p->b[D - 1];
  const int64_t a1 = D == 3 ? p->a[1] : 1;
  const int64_t nseg = nlast >= 64 ? nlast / 64 : 1;
  const int64_t rpw = nlast >= 64 ? 1 : 64 / nlast;
  const int64_t amin = D == 3 ? 1 : kUSplit * rpw;
  int best = 0;
  double best_eff = -1.0;
  for (int lg = 0; (a0_count >> lg) >= 1; ++lg) {
    const int64_t a0c = a0_count >> lg;
    if (lg > 0 && (a0c < amin || a0c * a1 * nseg * (nlast >= 64 ? 1 : 1) < 32)) break;
    if (lg > 0 && (a0c << lg) != a0_count) break;
    const double n = (double)(batch * bouter << lg) / (double)warps_total;
    const double eff = n / std::ceil(n);
    if (n >= kSplitUnitsPerWarp && eff >= 0.95) return lg;
    if (eff > best_eff + 0.02) { best_eff = eff; best = lg; }
  }
  (void)nl;
  return best;
}

// D == 1 gather-form fold (k_gather1d): eligible when a loop's W taps fit the registers
// (W <= 1024) and a whole frame fits a shared-memory ring slot; returns the per-lane tap
// count the kernel is instantiated for, or 0.
int gather1d_taps(const rsft_plan_s* p) {
  const int64_t W = p->b[0] < p->n[0] ? p->W[0] : p->n[0];
  if (p->D != 1 || W % 32 != 0 || W > 1024 || p->n[0] * 8 > 64 * 1024) return 0;
  const int t = (int)(W / 32);
  return t <= 4 ? 4 : t <= 8 ? 8 : t <= 16 ? 16 : 32;
}

int resolve_mode(const rsft_plan_s* p, int64_t batch) {
  const int64_t nlast = p->n[p->D - 1];
  const int Lf = std::min(p->L, kMaxLaunchLoops);   // loops per fold launch
  const int lp = loop_pad(Lf);
  bool fused_ok = p->D <= 2 && nlast >= 64 && p->btot <= 8 * kThreads &&
                  (fused_smem_bytes(p, Lf, lp) <= (fused_cfg(p->D).ctas == 1 ? 220 : 110) * 1024 ||
                   gather1d_taps(p) > 0);
  // split mode chunks dim 0 as far as needed to fit the per-warp tables (launch_split_fold_t)
  const int64_t amin = p->D == 3 ? 1 : std::min<int64_t>(p->a[0], (int64_t)kUSplit * (nlast >= 64 ? 1 : 64 / nlast));
  bool split_ok = p->D >= 2 && split_smem_bytes(p, Lf, lp, amin) <= 220 * 1024;
  int m = p->P.mode;
  if (m == RSFT_MODE_FUSED) return fused_ok ? RSFT_MODE_FUSED : -1;
  if (m == RSFT_MODE_SPLIT) return split_ok ? RSFT_MODE_SPLIT : -1;
  if (fused_ok && (p->D == 1 || batch >= 64)) return RSFT_MODE_FUSED;
  if (split_ok) return RSFT_MODE_SPLIT;
  return fused_ok ? RSFT_MODE_FUSED : -1;
}

}  // namespace rsft

using namespace rsft;

extern "C" {

void rsft_default_params(rsft_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->ndim = 1;
  for (int d = 0; d < 3; ++d) { p->n[d] = 1; p->b[d] = 1; p->support[d] = 0; }
  p->loops = 1;
  p->prewin = RSFT_WIN_HANN;
  p->prewin_param = 60.0;
  p->flat_atten_db = 60.0;
  p->p_fa = 1e-6;
  p->noise_var = 1.0;
  p->gamma_override = 0.0;
  p->mu = 0;
  p->random_tau = 0;
  p->seed = 0;
  p->max_batch = 1;
  p->mode = RSFT_MODE_AUTO;
}

rsft_status rsft_plan_create(const rsft_params* params, rsft_plan_t* out) {
  if (!out) return RSFT_E_ARG;
  *out = nullptr;
  if (!params) return RSFT_E_ARG;
  const rsft_params& P = *params;
  if (P.ndim < 1) return RSFT_E_ARG;
  if (P.ndim > 3) return RSFT_E_UNSUPPORTED;
  if (P.loops < 1) return RSFT_E_ARG;
  if (P.loops > kMaxLoops - 1) return RSFT_E_UNSUPPORTED;
  int mu = P.mu == 0 ? P.loops : P.mu;
  if (mu < 1 || mu > P.loops) return RSFT_E_ARG;
  if (!(P.p_fa > 0.0 && P.p_fa < 1.0)) return RSFT_E_ARG;
  if (!(P.noise_var > 0.0) && !(P.gamma_override > 0.0)) return RSFT_E_ARG;
  if (P.max_batch < 1) return RSFT_E_ARG;
  if (P.prewin < RSFT_WIN_RECT || P.prewin > RSFT_WIN_CHEB) return RSFT_E_ARG;
  if (P.mode < RSFT_MODE_AUTO || P.mode > RSFT_MODE_SPLIT) return RSFT_E_ARG;
  for (int d = 0; d < P.ndim; ++d) {
    int64_t n = P.n[d], b = P.b[d], w = P.support[d];
    if (!is_pow2(n) || !is_pow2(b) || b > n) return RSFT_E_SHAPE;
    if (n > (int64_t(1) << 30)) return RSFT_E_UNSUPPORTED;
    if (b > (P.ndim == 1 ? kMaxB1d : kMaxB)) return RSFT_E_UNSUPPORTED;
    if (b < n) {
      if (w == 0) w = n;
      if (w < 0 || w > n || w % 2 || (w / 2) % b) return RSFT_E_SHAPE;
    }
  }
  if (P.n[P.ndim - 1] < 32) return RSFT_E_UNSUPPORTED;

  rsft_plan_s* p = new (std::nothrow) rsft_plan_s();
  if (!p) return RSFT_E_ARG;
  p->P = P;
  p->P.mu = mu;
  p->D = P.ndim;
  p->L = P.loops;
  p->mu = mu;
  for (int d = 0; d < p->D; ++d) {
    p->n[d] = P.n[d]; p->b[d] = P.b[d]; p->a[d] = P.n[d] / P.b[d];
    p->W[d] = P.support[d] == 0 ? P.n[d] : P.support[d];
    p->ntot *= p->n[d]; p->btot *= p->b[d];
  }
  // Schedule (reading L5): sigma odd uniform in [N_d], tau uniform in [N_d] or 0.
  p->sigma.assign((size_t)p->L * p->D, 1);
  p->sinv.assign((size_t)p->L * p->D, 0);
  p->tau.assign((size_t)p->L * p->D, 0);
  for (int l = 0; l < p->L; ++l)
    for (int d = 0; d < p->D; ++d) {
      const int64_t n = p->n[d];
      const uint64_t ctr = 2ull * (uint64_t)(l * p->D + d);
      int64_t s = n >= 2 ? 2 * (int64_t)(splitmix64(P.seed, ctr) & (uint64_t)(n / 2 - 1)) + 1 : 1;
      int64_t t = (P.random_tau && n > 1) ? (int64_t)(splitmix64(P.seed, ctr + 1) & (uint64_t)(n - 1)) : 0;
      p->sigma[l * p->D + d] = s;
      p->sinv[l * p->D + d] = inv_mod_pow2(s, n);
      p->tau[l * p->D + d] = t;
    }
  for (int d = 0; d < p->D; ++d) {
    p->prewin[d] = prewindow(P, p->n[d]);
    p->flatg[d] = flat_proto(p->n[d], p->b[d], p->W[d], P.flat_atten_db);
  }
  // D = 1 with B > 64: only the gather-form fold (k_gather1d, support W <= 1024) folds it
  if (p->D == 1 && p->b[0] > kMaxB && !gather1d_taps(p)) { delete p; return RSFT_E_UNSUPPORTED; }
  rebuild_tables(p);
  layout_workspace(p);
  if (resolve_mode(p, P.max_batch) < 0) { delete p; return RSFT_E_UNSUPPORTED; }
  *out = p;
  return RSFT_OK;
}

void rsft_plan_destroy(rsft_plan_t plan) { delete plan; }

rsft_status rsft_plan(const rsft_params* params, int32_t device, rsft_plan_t* out) {
  if (device < -1) return RSFT_E_ARG;
  rsft_status s = rsft_plan_create(params, out);
  if (s == RSFT_OK) (*out)->want_device = device;
  return s;
}

void rsft_destroy(rsft_plan_t plan) { rsft_plan_destroy(plan); }

rsft_status rsft_set_schedule(rsft_plan_t p, const int64_t* sigma, const int64_t* tau) {
  if (!p || !sigma) return RSFT_E_ARG;
  for (int l = 0; l < p->L; ++l)
    for (int d = 0; d < p->D; ++d) {
      int64_t s = sigma[l * p->D + d], n = p->n[d];
      if (s < 0 || s >= n && n > 1) return RSFT_E_ARG;
      if (n > 1 && (s % 2) == 0) return RSFT_E_SIGMA;
      if (tau && (tau[l * p->D + d] < 0 || tau[l * p->D + d] >= n)) return RSFT_E_ARG;
    }
  for (int l = 0; l < p->L; ++l)
    for (int d = 0; d < p->D; ++d) {
      int64_t s = p->n[d] > 1 ? sigma[l * p->D + d] : 1;
      p->sigma[l * p->D + d] = s;
      p->sinv[l * p->D + d] = inv_mod_pow2(s, p->n[d]);
      p->tau[l * p->D + d] = tau ? tau[l * p->D + d] : 0;
    }
  return rebuild_tables(p);
}

rsft_status rsft_get_schedule(rsft_plan_t p, int64_t* sigma, int64_t* sigma_inv, int64_t* tau) {
  if (!p) return RSFT_E_ARG;
  size_t k = (size_t)p->L * p->D;
  for (size_t i = 0; i < k; ++i) {
    if (sigma) sigma[i] = p->sigma[i];
    if (sigma_inv) sigma_inv[i] = p->sinv[i];
    if (tau) tau[i] = p->tau[i];
  }
  return RSFT_OK;
}

rsft_status rsft_get_thresholds(rsft_plan_t p, double* beta, double* gamma) {
  if (!p) return RSFT_E_ARG;
  for (int l = 0; l < p->L; ++l) {
    if (beta) beta[l] = p->beta[l];
    if (gamma) gamma[l] = p->gamma[l];
  }
  return RSFT_OK;
}

rsft_status rsft_get_window(rsft_plan_t p, int32_t d, int32_t which, double* out) {
  if (!p || !out || d < 0 || d >= p->D) return RSFT_E_ARG;
  if (which == 0) { for (int64_t i = 0; i < p->n[d]; ++i) out[i] = p->prewin[d][i]; return RSFT_OK; }
  if (which == 1) { for (int64_t i = 0; i < p->n[d]; ++i) out[i] = p->flatg[d][i]; return RSFT_OK; }
  if (which == 2) {
    for (size_t i = 0; i < p->hf[d].size(); ++i) out[i] = (double)p->hf[d][i];
    return RSFT_OK;
  }
  return RSFT_E_ARG;
}

rsft_status rsft_get_info(rsft_plan_t p, rsft_info* info) {
  if (!p || !info) return RSFT_E_ARG;
  info->ntot = p->ntot;
  info->btot = p->btot;
  info->bitmap_words = (p->btot + 31) / 32;
  info->detect_words = (p->ntot + 31) / 32;
  info->mode = resolve_mode(p, p->P.max_batch);
  info->lpad = loop_pad(std::min(p->L, kMaxLaunchLoops));
  info->workspace_bytes = p->ws.total;
  return RSFT_OK;
}

size_t rsft_workspace_bytes(rsft_plan_t p) { return p ? p->ws.total : 0; }

int32_t rsft_last_launch_count(rsft_plan_t p) { return p ? p->last_launches : 0; }

const char* rsft_status_string(rsft_status s) {
  switch (s) {
    case RSFT_OK: return "RSFT_OK";
    case RSFT_E_ARG: return "RSFT_E_ARG";
    case RSFT_E_SHAPE: return "RSFT_E_SHAPE";
    case RSFT_E_SIGMA: return "RSFT_E_SIGMA";
    case RSFT_E_UNSUPPORTED: return "RSFT_E_UNSUPPORTED";
    case RSFT_E_WORKSPACE: return "RSFT_E_WORKSPACE";
    case RSFT_E_CUDA: return "RSFT_E_CUDA";
    case RSFT_E_STATE: return "RSFT_E_STATE";
  }
  return "RSFT_E_UNKNOWN";
}

const char* rsft_last_error(void) { return g_err.c_str(); }

}  // extern "C"
