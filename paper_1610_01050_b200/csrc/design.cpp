// Optimal threshold design: Eq. opt on the host, fp64.
//
// First stage, Eqs. tpd / bpd: Pd_bar = Pfa_bar^(beta_bar / (alpha_bar SNR + beta_bar)).
// Second stage, Claims 2-3: the accumulated votes are asymptotically Normal,
//   H1: N(T Pd_bar, T Pd_bar (1 - Pd_bar)),
//   H0: N(F rate + (T - F) Pfa_bar, F rate (1 - rate) + (T - F) Pfa_bar (1 - Pfa_bar)),
//   F = T K eta_m / B, rate = eta_p Pd_bar (co-existing sinusoids).
// Eq. opt: for every mu in [T] solve P_d = int_mu^inf g_a1 for Pd_bar and P_fa =
// int_mu^inf g_a0 for Pfa_bar, invert Eq. bpd for SNR_min, keep the smallest; then
// gamma* = sigma_n^2 beta_bar ln(1 / Pfa_bar).
// alpha_bar, beta_bar: the permutation averages (Eq. bpd) of Eq. alpha_beta
// for this plan's windows, alpha at the Claim 1 peak bucket (Eq. lemma13), over every
// odd sigma_d (tau = 0); separable over dimensions (compound windows).
// Independent of the oracle (oracle/thresholds.py), which computes the same quantities by
// running its literal first stage.
#include <cmath>
#include <complex>
#include <vector>

#include "rsft_internal.h"

using cd = std::complex<double>;

namespace {

double normal_tail(double mu, double mean, double var) {
  if (var <= 0.0) return mean >= mu ? 1.0 : 0.0;
  return 0.5 * std::erfc((mu - mean) / std::sqrt(2.0 * var));
}

template <class F>
double bisect_increasing(F f, double target) {
  double lo = 0.0, hi = 1.0;
  for (int i = 0; i < 200; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (f(mid) < target) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

// 6.0-dB main-lobe width in bins of window w (|W(f)| >= |W(0)| / 2 around DC), by bisection
// on the DTFT magnitude (SPEC S:114-122 measures the same on a zero-padded DFT).
double eta_6db(const std::vector<double>& w) {
  const int64_t n = (int64_t)w.size();
  auto mag = [&](double f) {
    cd acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += w[i] * std::polar(1.0, -2.0 * M_PI * f * (double)i / (double)n);
    return std::abs(acc);
  };
  const double half = mag(0.0) / 2.0;
  double hi = 0.0;
  while (mag(hi + 0.25) >= half) hi += 0.25;          // walk to the first sample below half
  double lo = hi;
  hi += 0.25;
  for (int i = 0; i < 60; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (mag(mid) >= half) lo = mid; else hi = mid;
  }
  return 2.0 * 0.5 * (lo + hi);
}

}  // namespace

extern "C" {

void rsft_default_design_params(rsft_design_params* d) {
  *d = rsft_design_params{};
  d->K = 1;
  d->p_d = 0.9;
  d->p_fa = 1e-6;
  d->eta_m = 0.0;
  d->eta_p = 1.0;
  d->loops = 0;
  for (int i = 0; i < 3; ++i) d->omega[i] = 0.5;
}

rsft_status rsft_design_thresholds(rsft_plan_t p, const rsft_design_params* dp, rsft_design_result* out) {
  if (!p || !dp || !out) return RSFT_E_ARG;
  const int D = p->D;
  const int T = dp->loops > 0 ? dp->loops : p->L;
  if (dp->K < 0 || !(dp->p_d > 0.0 && dp->p_d < 1.0) || !(dp->p_fa > 0.0 && dp->p_fa < 1.0) || dp->eta_p < 0.0)
    return RSFT_E_ARG;
  for (int d = 0; d < D; ++d)
    if (!(dp->omega[d] >= 0.0 && dp->omega[d] < (double)p->n[d])) return RSFT_E_ARG;
  double alpha_bar = 1.0, beta_bar = 1.0, eta_m = 1.0;
  for (int d = 0; d < D; ++d) {
    const int64_t n = p->n[d], b = p->b[d];
    const std::vector<double>& w = p->prewin[d];
    const std::vector<double>& g = p->flatg[d];
    const bool shift = b < n;
    const double om = dp->omega[d];
    const int64_t k0 = (int64_t)std::floor(om);
    double asum = 0.0, bsum = 0.0;
    int64_t cnt = 0;
    for (int64_t s = 1; s < n; s += 2) {                 // every odd sigma (uniform)
      const int64_t pk = (int64_t)(((__int128)b * (((__int128)s * k0) % n)) / n);   // Eq. lemma13
      cd acc = 0.0;
      double bb = 0.0;
      for (int64_t t = 0; t < n; ++t) {
        const int64_t src = (int64_t)(((__int128)s * t) % n);          // p[t] = y[sigma t] (tau = 0)
        const cd gbar = shift ? std::polar(g[t], -M_PI * (double)t / (double)b) : cd(g[t], 0.0);
        const cd v = std::polar(1.0, 2.0 * M_PI * om * (double)src / (double)n);
        // fold + B-point DFT at bucket pk: sum_t z[t] e^{-j 2 pi pk t / B}  (Eqs. l, f)
        acc += gbar * w[src] * v * std::polar(1.0, -2.0 * M_PI * (double)((pk * t) % b) / (double)b);
        bb += g[t] * g[t] * w[src] * w[src];
      }
      asum += std::norm(acc);
      bsum += bb;
      ++cnt;
    }
    alpha_bar *= asum / (double)cnt;
    beta_bar *= bsum / (double)cnt;
    eta_m *= eta_6db(w);
  }
  if (dp->eta_m > 0.0) eta_m = dp->eta_m;
  const double B = (double)p->btot;
  const double F = (double)T * dp->K * eta_m / B;        // Claim 3
  *out = rsft_design_result{};
  out->alpha_bar = alpha_bar;
  out->beta_bar = beta_bar;
  out->eta_m = eta_m;
  out->F = F;
  if (F >= (double)T) { rsft::set_error("infeasible: K eta_m >= B (Remark 2, P:517)"); return RSFT_E_ARG; }
  int best_mu = 0;
  double best = 0.0, best_pd = 0.0, best_pfa = 0.0;
  for (int mu = 1; mu <= T; ++mu) {
    const double pd = bisect_increasing([&](double q) { return normal_tail(mu, T * q, T * q * (1.0 - q)); }, dp->p_d);
    double rate = dp->eta_p > 0.0 ? dp->eta_p * pd : 1.0;   // eta_p = 0: upper bound (Remark 3)
    if (rate > 1.0) rate = 1.0;
    auto tail0 = [&](double q) {
      return normal_tail(mu, F * rate + (T - F) * q, F * rate * (1.0 - rate) + (T - F) * q * (1.0 - q));
    };
    if (tail0(0.0) > dp->p_fa) continue;
    const double pfa = bisect_increasing(tail0, dp->p_fa);
    if (!(pfa > 0.0 && pfa < pd && pd < 1.0)) continue;
    const double snr = beta_bar / alpha_bar * (std::log(pfa) / std::log(pd) - 1.0);   // Eq. bpd inverted
    if (best_mu == 0 || snr < best) { best_mu = mu; best = snr; best_pd = pd; best_pfa = pfa; }
  }
  if (best_mu == 0) { rsft::set_error("no feasible second-stage threshold"); return RSFT_E_ARG; }
  out->mu = best_mu;
  out->snr_min = best;
  out->snr_min_db = 10.0 * std::log10(best);
  out->pd_bar = best_pd;
  out->pfa_bar = best_pfa;
  out->gamma = p->P.noise_var * beta_bar * std::log(1.0 / best_pfa);   // Eq. bpd
  return RSFT_OK;
}

}  // extern "C"
