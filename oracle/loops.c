/*
 * oracle/loops.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product path).  Plain-C restatement of the five explicit inner loops of the
 * reference `fftlattice` package (pkg/src/fftlattice/_accel.py).  Compiled with
 * -ffp-contract=off so every multiply and add rounds separately, in the same
 * left-to-right order as the reference's numba loops (which LLVM does not
 * contract), which makes these loops bit-identical to the reference.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.
 */
#include <math.h>
#include <stdint.h>

#define ORC_NONE_SEEN (-(((int64_t)1) << 60)) /* _accel.py:46 */

/* _accel.py:49-59: plain backward induction of a leaf row, in place. */
double orc_european_backward(double *v, int64_t len, double wd, double wu) {
  int64_t n = len - 1;
  for (int64_t i = n; i > 0; --i)
    for (int64_t j = 0; j < i; ++j) v[j] = wd * v[j] + wu * v[j + 1];
  return v[0];
}

/* _accel.py:62-102: projected backward induction for the American call,
 * recording the first exercise column of every row (ties -> continuation). */
double orc_american_call_backward(double *v, int64_t len, const double *u2,
                                  int64_t *first_green, double spot,
                                  double strike, double wd, double wu,
                                  double log_up) {
  int64_t n = len - 1;
  int64_t fg = ORC_NONE_SEEN;
  for (int64_t j = 0; j <= n; ++j) {
    if (spot * u2[j] - strike > 0.0) { fg = j; break; }
  }
  first_green[n] = fg;
  for (int64_t i = n - 1; i >= 0; --i) {
    double scale = spot * exp((double)(n - i) * log_up);
    fg = ORC_NONE_SEEN;
    for (int64_t j = 0; j <= i; ++j) {
      double lin = wd * v[j] + wu * v[j + 1];
      double grn = scale * u2[j] - strike;
      if (lin >= grn) {
        v[j] = lin;
      } else {
        v[j] = grn;
        if (fg == ORC_NONE_SEEN) fg = j;
      }
    }
    first_green[i] = fg;
  }
  return v[0];
}

/* _accel.py:105-160: explicit projected sweeps on a boundary-hugging strip of
 * the call lattice; returns the last continuation column after `height` rows. */
int64_t orc_binomial_strip_sweep(double *v, const double *e2, int64_t lo,
                                 int64_t top_row, int64_t boundary,
                                 int64_t height, double spot, double strike,
                                 double wd, double wu, double log_up) {
  int64_t j = boundary;
  for (int64_t s = 0; s < height; ++s) {
    int64_t parent = top_row - s;
    int64_t child = parent - 1;
    if (j < lo) break;
    int64_t top = j < child ? j : child;
    double bc = spot * exp((double)(2 * lo - child) * log_up);
    double bp = spot * exp((double)(2 * lo - parent) * log_up);
    int64_t fg = ORC_NONE_SEEN;
    for (int64_t c = lo; c <= top; ++c) {
      double vr = (c + 1 <= j) ? v[c + 1 - lo] : bp * e2[c + 1 - lo] - strike;
      double lin = wd * v[c - lo] + wu * vr;
      double grn = bc * e2[c - lo] - strike;
      if (lin >= grn) {
        v[c - lo] = lin;
      } else {
        v[c - lo] = grn;
        if (fg == ORC_NONE_SEEN) fg = c;
      }
    }
    j = (fg == ORC_NONE_SEEN) ? top : fg - 1;
  }
  return j;
}

/* _accel.py:163-200: projected marching of the put over its shrinking
 * dependency window; last_green[n] = largest exercise offset (ties -> exercise). */
double orc_put_march_window(double *v, int64_t len, const double *payoff,
                            int64_t start_step, int64_t end_step, double cd,
                            double cm, double cu, int64_t *last_green) {
  int64_t two_t = len - 1;
  for (int64_t n = start_step + 1; n <= end_step; ++n) {
    double left = v[n - 1];
    int64_t lg = ORC_NONE_SEEN;
    for (int64_t k = n; k <= two_t - n; ++k) {
      double cur = v[k];
      double lin = cm * cur + cu * v[k + 1] + cd * left;
      left = cur;
      double pay = payoff[k];
      if (lin > pay) {
        v[k] = lin;
      } else {
        v[k] = pay;
        lg = k;
      }
    }
    last_green[n] = lg;
  }
  return v[two_t / 2];
}

/* _accel.py:203-242: explicit put sweeps on a strip straddling the boundary;
 * returns the largest exercise column of the final row (or NONE_SEEN). */
int64_t orc_bsm_strip_sweep(double *v, int64_t len, const double *payoff,
                            int64_t lo, int64_t height, double cd, double cm,
                            double cu) {
  int64_t hi = lo + len - 1;
  int64_t lg = ORC_NONE_SEEN;
  for (int64_t s = 1; s <= height; ++s) {
    double left = v[s - 1];
    lg = ORC_NONE_SEEN;
    for (int64_t k = lo + s; k <= hi - s; ++k) {
      double cur = v[k - lo];
      double lin = cm * cur + cu * v[k - lo + 1] + cd * left;
      left = cur;
      double pay = payoff[k - lo];
      if (lin > pay) {
        v[k - lo] = lin;
      } else {
        v[k - lo] = pay;
        lg = k;
      }
    }
  }
  return lg;
}
