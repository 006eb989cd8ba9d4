// host_params.h -- host-side derivation of per-option lattice / grid records.
//
// Every formula follows the reference operation order with the same libm
// calls Python's `math` module makes (log, exp, sqrt, expm1, pow, rint), so the
// derived constants, k*, terminal/junction boundaries and dispatch decisions
// are bit-identical to the reference:
//   validate_spec          model.py:145-175
//   derive_binomial_params model.py:211-248
//   discretize_bsm         bsm.py:150-229
//   top_row_state          american.py:260-295
//   _junction_row          american.py:366-425 (boundary search only; values on device)
//   fast_* dispatch        binomial.py:161, american.py:428-470, bsm.py:585-625
#pragma once

#include <cmath>
#include <cstdint>

#include "fl_status.h"

// The same derivation also runs on the device for the device-pointer entry
// points (fl_price_batch_dev: caller-owned device buffers, no host round trip).
// There the CUDA libm (exp/log within 1 ulp) and the compiler's FMA
// contraction replace glibc's bits, so device-derived constants may differ
// from the reference's in the last place; prices stay within the parity
// tolerance and the host path stays bit-identical.
#ifdef __CUDACC__
#define FL_HD __host__ __device__
#else
#define FL_HD
#endif

namespace fl {

enum : int32_t {
  MODE_ERROR = -1,
  MODE_FAST = 0,      // device divide-and-conquer
  MODE_BASELINE = 1,  // device O(T^2) sweep (reference dispatch T <= cutoff)
  MODE_INTRINSIC = 2, // closed price decided on host (k* <= -T; all-exercise junction)
  MODE_EURO = 3,      // American call that the reference prices as European
};

struct SpecIn {
  double S, K, R, Y, V, E;
  int64_t T;
};

struct PutParams {
  double S, K;
  double cd, cm, cu, ds;
  int64_t n, ks;
  int32_t cutoff, mode;
  double price;  // host-decided price (MODE_INTRINSIC)
  int32_t slide;  // 1: exercise cells provably stay exercise (sliding-frame leaf strips)
  int32_t pad;
};

struct CallParams {
  double S, K;
  double wd, wu, lu;
  int64_t n;
  int64_t top_b;   // last red column of the terminal row
  int64_t junc_j;  // last red column of row T-1
  int32_t cutoff, mode;
  double price;    // MODE_INTRINSIC
};

struct EuroParams {
  double S, K;
  double wd, wu;   // one-step weights (baseline_european)
  double bg;       // gauged up weight wu e^{2 lu}; kernel [wd, bg] (binomial.py:181-186)
  double lu;
  int64_t n;
  int32_t mode, pad;
};

constexpr double DAYS_PER_YEAR = 365.0;

FL_HD inline int32_t validate_spec(const SpecIn& s) {
  if (!(s.S > 0.0 && std::isfinite(s.S))) return FL_E_VALIDATION | FL_F_SPOT;
  if (!(s.K >= 0.0 && std::isfinite(s.K))) return FL_E_VALIDATION | FL_F_STRIKE;
  if (!(s.R >= 0.0 && std::isfinite(s.R))) return FL_E_VALIDATION | FL_F_RATE;
  if (!(s.Y >= 0.0 && std::isfinite(s.Y))) return FL_E_VALIDATION | FL_F_YIELD;
  if (!(s.V > 0.0 && std::isfinite(s.V))) return FL_E_VALIDATION | FL_F_VOL;
  if (!(s.E > 0.0 && std::isfinite(s.E))) return FL_E_VALIDATION | FL_F_DAYS;
  if (!(s.T >= 1)) return FL_E_VALIDATION | FL_F_STEPS;
  return FL_OK;
}

struct Binom {
  double dt, up, down, p, disc, wd, wu, lu;
};

FL_HD inline int32_t derive_binomial(const SpecIn& s, Binom& b) {
  int32_t st = validate_spec(s);
  if (st) return st;
  b.dt = s.E / (DAYS_PER_YEAR * (double)s.T);
  b.lu = s.V * std::sqrt(b.dt);
  b.up = std::exp(b.lu);
  b.down = 1.0 / b.up;
  double growth = std::exp((s.R - s.Y) * b.dt);
  b.p = (growth - b.down) / (b.up - b.down);
  if (!(0.0 < b.p && b.p < 1.0)) return FL_E_VALIDATION | FL_F_PROB_UP;
  b.disc = std::exp(-s.R * b.dt);
  b.wd = b.disc * (1.0 - b.p);
  b.wu = b.disc * b.p;
  return FL_OK;
}

FL_HD inline double green_call(const SpecIn& s, const Binom& b, int64_t i, int64_t j) {
  return s.S * std::exp((double)(2 * j - i) * b.lu) - s.K;
}

// american.py:260-295
FL_HD inline int64_t call_top_boundary(const SpecIn& s, const Binom& b) {
  const int64_t n = s.T;
  if (s.K <= 0.0) return -1;
  double g = std::floor(0.5 * (double)n + std::log(s.K / s.S) / (2.0 * b.lu));
  if (g < -1.0) g = -1.0;
  if (g > (double)n) g = (double)n;
  int64_t bnd = (int64_t)g;
  while (bnd < n && green_call(s, b, n, bnd + 1) <= 0.0) ++bnd;
  while (bnd >= 0 && green_call(s, b, n, bnd) > 0.0) --bnd;
  return bnd;
}

// american.py:366-425, boundary part; returns status (ValueError on log domain)
FL_HD inline int32_t call_junction_boundary(const SpecIn& s, const Binom& b, int64_t top_b, int64_t& j_out) {
  const int64_t n = s.T;
  const int64_t i = n - 1;
  auto red = [&](int64_t j) {
    double vd = green_call(s, b, n, j);
    double vu = green_call(s, b, n, j + 1);
    double lin = b.wd * (vd > 0.0 ? vd : 0.0) + b.wu * (vu > 0.0 ? vu : 0.0);
    return lin >= green_call(s, b, i, j);
  };
  double rdt = s.R * b.dt;
  double ydt = s.Y * b.dt;
  int64_t guess = top_b;
  if (rdt > 0.0 && ydt > 0.0) {
    double q1 = s.K / s.S;
    double q2 = std::expm1(rdt) / std::expm1(ydt);
    if (!(q1 > 0.0) || !(q2 > 0.0)) return FL_E_VALUE;  // Python math.log raises
    double shift = std::log(q1) + std::log(q2) - (rdt - ydt);
    double e = std::ceil(0.5 * (double)i + shift / (2.0 * b.lu)) - 1.0;
    if (e > 9.0e18) e = 9.0e18;
    if (e < -9.0e18) e = -9.0e18;
    int64_t est = (int64_t)e;
    if (est > guess) guess = est;
  }
  int64_t j = guess;
  if (j < -1) j = -1;
  if (j > i) j = i;
  while (j < i && red(j + 1)) ++j;
  while (j >= 0 && !red(j)) --j;
  j_out = j;
  return FL_OK;
}

// Caller-supplied lattice constants (the reference pricers' `params=`
// argument, binomial.py:161 / american.py:428): used instead of the derived
// ones; the spec is still validated.
FL_HD inline int32_t binomial_or_override(const SpecIn& s, const Binom* ovr, Binom& b) {
  if (!ovr) return derive_binomial(s, b);
  const int32_t st = validate_spec(s);
  if (st) return st;
  b = *ovr;
  return FL_OK;
}

FL_HD inline int32_t prep_euro(const SpecIn& s, EuroParams& e, const Binom* ovr = nullptr) {
  Binom b;
  int32_t st = binomial_or_override(s, ovr, b);
  e.S = s.S; e.K = s.K; e.n = s.T; e.lu = b.lu;
  e.mode = st ? MODE_ERROR : MODE_FAST;
  e.pad = 0;
  if (st) return st;
  e.wd = b.wd;
  e.wu = b.wu;
  e.bg = b.wu * std::exp(2.0 * b.lu);
  return FL_OK;
}

// american.py:428-470 dispatch
FL_HD inline int32_t prep_call(const SpecIn& s, int64_t cutoff, CallParams& c, EuroParams& e,
                               const Binom* ovr = nullptr) {
  Binom b;
  c.S = s.S; c.K = s.K; c.n = s.T; c.cutoff = (int32_t)cutoff; c.price = 0.0;
  c.top_b = -1; c.junc_j = -1;
  int32_t st = binomial_or_override(s, ovr, b);
  if (st) { c.mode = MODE_ERROR; return st; }
  c.wd = b.wd; c.wu = b.wu; c.lu = b.lu;
  prep_euro(s, e, ovr);
  const int64_t n = s.T;
  if (s.Y == 0.0) {
    c.top_b = call_top_boundary(s, b);
    c.mode = MODE_EURO;
    return FL_OK;
  }
  if (n <= cutoff) { c.mode = MODE_BASELINE; return FL_OK; }
  c.top_b = call_top_boundary(s, b);
  if (c.top_b == n) { c.mode = MODE_EURO; return FL_OK; }
  int64_t j;
  st = call_junction_boundary(s, b, c.top_b, j);
  if (st) { c.mode = MODE_ERROR; return st; }
  c.junc_j = j;
  // all-exercise row T-1: the reference builds BoundarySeries(times=[T, T-1])
  // here (american.py:478-486), which its constructor rejects -> it raises
  // ValidationError('times'); mirrored (the price would be S - K)
  if (j < 0) { c.mode = MODE_ERROR; c.price = s.S - s.K; return FL_E_VALIDATION | FL_F_TIMES; }
  c.mode = MODE_FAST;
  return FL_OK;
}

// European normal-limit approximations (binomial.py:197-296)
struct EuroApprox {
  double S, K, lu, mu, sigma, disc;  // disc = exp(-R * years)
  int64_t n, lo, hi, x0;             // Gaussian window [lo, hi]; closed-form threshold x0
  int32_t method, pad;               // 2: Gaussian window sum, 3: closed form
};

inline int32_t prep_euro_approx(const SpecIn& s, int method, EuroApprox& a) {
  Binom b;
  int32_t st = derive_binomial(s, b);
  a.S = s.S; a.K = s.K; a.n = s.T; a.method = method; a.pad = 0;
  a.lo = a.hi = a.x0 = 0;
  if (st) return st;
  const int64_t n = s.T;
  a.lu = b.lu;
  a.mu = -b.p * (double)n;
  a.sigma = b.p * (1.0 - b.p) * (double)n;
  a.disc = std::exp(-s.R * (s.E / DAYS_PER_YEAR));
  if (method == 2) {  // _gaussian_window (binomial.py:197-215)
    const double center = -a.mu;
    const double lo = std::ceil(center - 6.0 * std::sqrt(a.sigma));
    const double hi = std::floor(center + 6.0 * std::sqrt(a.sigma));
    a.lo = lo > 0.0 ? (int64_t)lo : 0;
    a.hi = hi < (double)(n - 1) ? (int64_t)hi : n - 1;
    if (a.lo > a.hi) return FL_E_DOMAIN | FL_D_WINDOW;
  } else {  // closed_form_european (binomial.py:243-296)
    if (s.K <= 0.0) return FL_E_DOMAIN | FL_D_CF_STRIKE;
    const double threshold = 0.5 * (double)n + std::log(s.K / s.S) / (2.0 * b.lu);
    const double x0 = std::ceil(threshold);
    a.x0 = x0 > (double)n ? n + 1 : (x0 < 0.0 ? 0 : (int64_t)x0);
  }
  return FL_OK;
}

struct PutDisc {
  int64_t n, ks;
  double omega, tau_max, d_tau, d_s, cd, cm, cu;
};

// bsm.py:150-229
FL_HD inline int32_t discretize_put(const SpecIn& s, double lam, PutDisc& d) {
  int32_t st = validate_spec(s);
  if (st) return st;
  const int64_t n = s.T;
  if (!(std::isfinite(lam) && lam > 0.0)) return FL_E_VALIDATION | FL_F_LAM;
  if (s.K <= 0.0) return FL_E_DOMAIN | FL_D_STRIKE;
  double years = s.E / DAYS_PER_YEAR;
  double omega = 2.0 * s.R / std::pow(s.V, 2.0);
  double tau_max = 0.5 * std::pow(s.V, 2.0) * years;
  double d_tau = tau_max / (double)n;
  double d_s = std::sqrt(d_tau / lam);
  double lm = std::log(s.S / s.K);
  double kr = std::rint(lm / d_s);  // round-half-even, like Python round()
  if (!(std::fabs(kr) <= 8.0 * (double)n)) return FL_E_DOMAIN | FL_D_GRID_NODES;
  int64_t ks = (int64_t)kr;
  if (ks != 0) d_s = lm / (double)ks;
  double lam_eff = d_tau / (d_s * d_s);
  double drift = (omega - 1.0) * d_tau / (2.0 * d_s);
  double cu = lam_eff + drift;
  double cd = lam_eff - drift;
  double cm = 1.0 - omega * d_tau - 2.0 * lam_eff;
  if (cm < 0.0) return FL_E_STABILITY | FL_W_MID;
  if (cu < 0.0) return FL_E_STABILITY | FL_W_UP;
  if (cd < 0.0) return FL_E_STABILITY | FL_W_DOWN;
  d.n = n; d.ks = ks; d.omega = omega; d.tau_max = tau_max; d.d_tau = d_tau;
  d.d_s = d_s; d.cd = cd; d.cm = cm; d.cu = cu;
  return FL_OK;
}

// bsm.py:585-625 dispatch
FL_HD inline int32_t prep_put(const SpecIn& s, double lam, int64_t cutoff, PutParams& p) {
  PutDisc d;
  p.S = s.S; p.K = s.K; p.n = s.T; p.cutoff = (int32_t)cutoff; p.price = 0.0;
  p.cd = p.cm = p.cu = p.ds = 0.0; p.ks = 0; p.slide = 0; p.pad = 0;
  int32_t st = discretize_put(s, lam, d);
  if (st) { p.mode = MODE_ERROR; return st; }
  p.cd = d.cd; p.cm = d.cm; p.cu = d.cu; p.ds = d.d_s; p.ks = d.ks;
  // A cell whose three parents hold the payoff g(x) = 1 - e^x (x = col ds <= 0,
  // the exercise side of the strike node) gets lin - g = -omega dtau +
  // e^x (1 - A), A = cd e^-ds + cm + cu e^ds (cd + cm + cu = 1 - omega dtau).
  // When that is negative for every x <= 0 with a margin far above the
  // rounding of lin (~1e-15), exercise cells stay exercise cells and the
  // boundary drops by at most one column per row: the leaf strips may then
  // skip every column left of the moving boundary (put_strip_slide).
  {
    const double A = d.cd * std::exp(-d.d_s) + d.cm + d.cu * std::exp(d.d_s);
    const double rise = 1.0 - A > 0.0 ? 1.0 - A : 0.0;
    p.slide = (d.omega * d.d_tau - rise > 1e-12) ? 1 : 0;
  }
  if (cutoff < 1) { p.mode = MODE_ERROR; return FL_E_VALIDATION | FL_F_CUTOFF; }
  if (d.ks <= -d.n) { p.mode = MODE_INTRINSIC; p.price = s.K - s.S; return FL_OK; }
  if (d.n <= 2 * cutoff) { p.mode = MODE_BASELINE; return FL_OK; }
  p.mode = MODE_FAST;
  return FL_OK;
}

}  // namespace fl
