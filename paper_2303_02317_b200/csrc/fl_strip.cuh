// fl_strip.cuh -- warp-level explicit projected sweeps of the put (the
// nonlinear base cases of the boundary recursion).
//
// put_strip_fixed / put_strip_pipe replace _accel.bsm_strip_sweep
// (_accel.py:203-242) as driven by bsm._strip_advance (bsm.py:402-440).  The
// call's strips are in fl_callstrip.cuh.
//
// One warp owns the whole strip; lanes hold consecutive columns in registers,
// neighbours move by warp shuffles, and the boundary (the last exercise
// column) comes from one warp-wide max after the last row instead of a scalar
// scan.  Tie rule as the reference: a cell is continuation iff lin > payoff.
// (Variants measured and not used -- the plain full frame, the 3h+2 frame,
// the sliding frame without the ghost lane, two rows per exchange, time-tiled
// full frames -- live in tools/strip_variants.cuh with their A/B tools;
// profiles/r01_experiments.md and r02_experiments.md.)
#pragma once

#include "fl_common.cuh"

namespace fl {

constexpr int64_t NONE_SEEN = -(((int64_t)1) << 60);  // _accel.py:46

// Full-frame put strip over columns [lo, hi] (lo = f-2h-1, hi = f+2h, the
// reference's 4h+2 frame), `height` forward rows: cells <= f hold the payoff,
// cells f+1..hi come from in_org[col].  Writes the continuation values of cols
// kb+1 .. hi-height of the final row to out_org[col] and returns kb, the
// largest exercise column of the final row within its valid range (NONE_SEEN
// if none).  Every lane of the warp calls; lane l holds CPL consecutive
// columns.  The neighbour exchange is software-pipelined: the per-row
// loop-carried cycle is shuffle -> DFMA -> DSETP/FSEL -> shuffle, and the warp
// issues in order, so the two edge cells of each row are finished FIRST and
// their shuffles for the next row issued before the interior cells, whose
// FP64 issue then overlaps the shuffle latency.  Used for options without the
// exercise margin the sliding frame needs (PutParams::slide == 0).
template <int CPL>
__device__ int64_t put_strip_pipe(const double* __restrict__ in_org, double* __restrict__ out_org,
                                  const double* __restrict__ pay_org, int64_t lo, int64_t hi, int64_t f,
                                  int height, double cd, double cm, double cu, long long* tm = nullptr) {
  static_assert(CPL >= 3, "edge / interior split");
  const int lane = threadIdx.x & 31;
  double v[CPL], p[CPL];
  const int64_t c0 = lo + (int64_t)lane * CPL;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int64_t col = c0 + c;
    if (col <= hi) {
      p[c] = pay_org[col];
      v[c] = (col <= f) ? p[c] : in_org[col];
    } else {
      p[c] = 0.0;
      v[c] = 0.0;
    }
  }
  long long ta = 0;
  __syncwarp();
  if (tm) { ta = clock64() + (long long)(v[0] + p[0] == 12345.678 ? 1 : 0); }
  double L = __shfl_up_sync(FULL, v[CPL - 1], 1);
  double R = __shfl_down_sync(FULL, v[0], 1);
  unsigned green = 0;
  for (int s = 1; s <= height; ++s) {
    // off-path partial sums of every cell (previous row only)
    double a[CPL];
    a[0] = fma(cu, v[1], cm * v[0]);
#pragma unroll
    for (int c = 1; c < CPL - 1; ++c) a[c] = fma(cu, v[c + 1], cm * v[c]);
    a[CPL - 1] = fma(cd, v[CPL - 2], cm * v[CPL - 1]);
    // edges (the shuffled neighbour enters last), then next row's exchange
    const double lin0 = fma(cd, L, a[0]);
    const double linE = fma(cu, R, a[CPL - 1]);
    const bool red0 = lin0 > p[0], redE = linE > p[CPL - 1];
    const double n0 = red0 ? lin0 : p[0];
    const double nE = redE ? linE : p[CPL - 1];
    L = __shfl_up_sync(FULL, nE, 1);
    R = __shfl_down_sync(FULL, n0, 1);
    green = (red0 ? 0u : 1u) | ((redE ? 0u : 1u) << (CPL - 1));
    double nv[CPL];
#pragma unroll
    for (int c = 1; c < CPL - 1; ++c) {
      const double lin = fma(cd, v[c - 1], a[c]);
      const bool red = lin > p[c];
      nv[c] = red ? lin : p[c];
      green |= (red ? 0u : 1u) << c;
    }
    nv[0] = n0;
    nv[CPL - 1] = nE;
#pragma unroll
    for (int c = 0; c < CPL; ++c) v[c] = nv[c];
  }
  if (tm) { tm[0] += ta; tm[1] += clock64() + (long long)(v[0] == 12345.678 ? 1 : 0) - ta; }
  const int64_t vlo = lo + height, vhi = hi - height;
  int best = -1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int64_t col = c0 + c;
    if (((green >> c) & 1u) && col >= vlo && col <= vhi) best = (int)(col - lo);
  }
  best = warp_max_i32(best);
  const int64_t kb = (best < 0) ? NONE_SEEN : lo + best;
  const int64_t wlo = (best < 0) ? vhi + 1 : kb + 1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int64_t col = c0 + c;
    if (col >= wlo && col <= vhi) out_org[col] = v[c];
  }
  return kb;
}

// Projection max(lin, pay) with the reference's tie rule (lin > pay ? lin : pay).
__device__ __forceinline__ double proj_max(double lin, double pay) {
  return lin > pay ? lin : pay;
}

#ifndef FL_FIXED_MARGIN_CAP  // test builds only (tools/test_fixed_miss.sh): a tiny margin forces FIXED_MISS
#define FL_FIXED_MARGIN_CAP 1000000
#endif
#ifndef FL_FIXED_UNROLL
#define FL_FIXED_UNROLL 2  // measured: 1 is -0.5..-2 % at the headline (two chains per SM) but +7 % at C4 (one per SM); 4 slower
#endif
constexpr int FIXED_UNROLL = FL_FIXED_UNROLL;
constexpr int64_t FIXED_MISS = NONE_SEEN - 1;  // put_strip_fixed: left edge not exercise, nothing written

// Fixed-column put strip with a ghost lane (production leaf).  Same contract as
// the sliding-frame put_strip_ghost (round 1-2 production leaf, now in
// tools/strip_variants.cuh), but the frame does not slide: lanes 1..31 hold the columns
// base .. f+2h (cell j = column base + j, CPL consecutive cells per lane,
// base = f - M with M = min(31 CPL - 2h - 1, 2h) exercise columns left of f;
// 2h + 2 <= 31 CPL),
// so a cell keeps its payoff in a register for the whole strip: no payoff
// shift and no payoff load per row (the sliding frame spends ~10 register
// moves and a shared load per row on them -- in the kernel two chain warps
// share one SMSP and the strip is issue-bound, ncu source view round 3).
// Per row a lane exchanges one cell with each neighbour (two shuffle
// directions, the same four 32-bit shuffles as the sliding frame).
//   * right side: as in the sliding frame, garbage enters at column f+2h+1 and
//     moves left one column per row, never reaching the valid range
//     [f-h-1, f+h] of the last row (_accel.py:203-242);
//   * left side: every column < base is an exercise cell at every row as long
//     as column base is (a cell whose three parents are exercise cells stays
//     exercise, PutParams::slide margin, see put_strip_ghost).  Lane 0 is the
//     ghost lane (cols base-CPL .. base-1, values exactly their payoffs, its
//     shuffled-in left inputs come from its own lower-payoff cells).  Column
//     base is checked on every row; if it ever turns continuation the strip
//     writes nothing and returns FIXED_MISS (the caller reruns the full frame).
// Per-cell arithmetic is put_strip_ghost's (bit-identical results).
// pay_org must cover cols f-2h-1 .. f+2h (the reference strip's frame).
template <int CPL>
__device__ int64_t put_strip_fixed(const double* __restrict__ in_org, double* __restrict__ out_org,
                                   const double* __restrict__ pay_org, int64_t f, int height, double cd, double cm,
                                   double cu, long long* tm = nullptr) {
  const int lane = threadIdx.x & 31;
  const int h = height;
  // margin: what the frame's 31 CPL cells leave, at most 2h (column base-1
  // stays inside the reference frame [f-2h-1, f+2h])
  const int Mx = 31 * CPL - 2 * h - 1;
  int M = Mx < 2 * h ? Mx : 2 * h;
  if (M > FL_FIXED_MARGIN_CAP) M = FL_FIXED_MARGIN_CAP;  // test builds: force the full-frame re-run path
  const int64_t base = f - M;
  const int W = M + 2 * h + 1;      // frame cells base .. f+2h
  const int j0 = (lane - 1) * CPL;  // lane 0: cells -CPL .. -1
  double v[CPL], p[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int j = (j0 + c < W) ? j0 + c : W - 1;
    int64_t col = base + j;
    // ghost cells left of the reference frame read its first column: a lower
    // payoff only lowers the ghost lane's lin, and the ghost cell next to the
    // frame (column base-1 >= f-2h-1) is exact
    col = col < f - 2 * h - 1 ? f - 2 * h - 1 : col;
    p[c] = pay_org[col];
    v[c] = (col <= f) ? p[c] : in_org[col];
  }
  __syncwarp();
  long long ta = 0;
  if (tm) { ta = clock64() + (long long)(v[0] + p[0] == 12345.678 ? 1 : 0); }
  bool cont0 = false;  // lane 1: column base turned continuation on some row
#pragma unroll FIXED_UNROLL
  for (int s = 0; s < h; ++s) {
    const double L = __shfl_up_sync(FULL, v[CPL - 1], 1);
    const double R = __shfl_down_sync(FULL, v[0], 1);
    double nv[CPL];
    {
      const double lin = fma(cd, L, fma(cu, v[1], cm * v[0]));
      cont0 |= lin > p[0];
      nv[0] = proj_max(lin, p[0]);
    }
#pragma unroll
    for (int c = 1; c < CPL - 1; ++c) {
      const double lin = fma(cd, v[c - 1], fma(cu, v[c + 1], cm * v[c]));
      nv[c] = proj_max(lin, p[c]);
    }
    {
      const double lin = fma(cd, v[CPL - 2], fma(cu, R, cm * v[CPL - 1]));
      nv[CPL - 1] = proj_max(lin, p[CPL - 1]);
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) v[c] = nv[c];
  }
  if (tm) { tm[0] += ta; tm[1] += clock64() + (long long)(v[0] == 12345.678 ? 1 : 0) - ta; }
  if (__shfl_sync(FULL, cont0 ? 1 : 0, 1)) return FIXED_MISS;
  // last exercise column of the final row within the valid range (cols <= f+h)
  int best = -1;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (v[c] == p[c] && j0 + c >= 0 && j0 + c <= M + h) best = j0 + c;
  best = warp_max_i32(best);
  const int64_t kb = (best < 0) ? NONE_SEEN : base + best;
  const int jlo = (best < 0) ? W : best + 1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int j = j0 + c;
    if (j >= jlo && j <= M + h) out_org[base + j] = v[c];
  }
  __syncwarp();
  return kb;
}

}  // namespace fl
