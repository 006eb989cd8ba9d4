// fl_strip.cuh -- warp-level explicit projected sweeps (the nonlinear base cases).
//
// put_strip_warp  replaces _accel.bsm_strip_sweep        (_accel.py:203-242)
//                 as driven by bsm._strip_advance          (bsm.py:402-440)
// call_strip_warp replaces _accel.binomial_strip_sweep   (_accel.py:105-160)
//
// One warp owns the whole strip; lane l holds CPL consecutive columns in
// registers, neighbours move by warp shuffles, and the boundary (last green
// for the put, first green for the call) comes from warp-wide min/max
// reductions instead of a scalar scan.  Tie rules follow the reference:
// put cells are continuation iff lin > payoff (ties exercise); call cells are
// continuation iff lin >= green (ties continuation).
#pragma once

#include "fl_common.cuh"

namespace fl {

constexpr int64_t NONE_SEEN = -(((int64_t)1) << 60);  // _accel.py:46
#ifndef FL_GHOST_UNROLL  // rows per unrolled step of the ghost-lane strip loop
#define FL_GHOST_UNROLL 2
#endif
#ifndef FL_PIPE_NOINLINE  // 1: the full-frame fallback strip is a real call (measured slower: spills)
#define FL_PIPE_NOINLINE 0
#endif
#ifndef FL_STRIP_ORDER
#define FL_STRIP_ORDER 1
#endif

// Put strip over columns [lo, hi], `height` forward rows.  Cells <= f hold the
// payoff, cells f+1..hi come from in_org[col].  Writes the continuation values
// of cols kb+1 .. hi-height of the final row to out_org[col] and returns kb, the
// largest exercise column of the final row within its valid range (NONE_SEEN
// if none).  Every lane of the warp must call.
template <int CPL>
__device__ int64_t put_strip_warp(const double* __restrict__ in_org, double* __restrict__ out_org,
                                  const double* __restrict__ pay_org, int64_t lo, int64_t hi, int64_t f,
                                  int height, double cd, double cm, double cu, long long* tm = nullptr) {
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
  unsigned green = 0;
  long long ta = 0;
  __syncwarp();
  if (tm) { ta = clock64() + (long long)(v[0] + p[0] == 12345.678 ? 1 : 0); }
  for (int s = 1; s <= height; ++s) {
    const double left = __shfl_up_sync(FULL, v[CPL - 1], 1);
    const double right = __shfl_down_sync(FULL, v[0], 1);
    double nv[CPL];
    green = 0;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const double l = (c == 0) ? left : v[c - 1];
      const double r = (c == CPL - 1) ? right : v[c + 1];
      // the shuffled neighbour enters last: one DFMA between a shuffle and the
      // next row's shuffle on the warp's critical path
#if FL_STRIP_ORDER
      const double lin = (c == CPL - 1) ? fma(cu, r, fma(cd, l, cm * v[c])) : fma(cd, l, fma(cu, r, cm * v[c]));
#else
      const double lin = fma(cd, l, fma(cu, r, cm * v[c]));
#endif
      const bool red = lin > p[c];
      nv[c] = red ? lin : p[c];
      green |= (red ? 0u : 1u) << c;
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) v[c] = nv[c];
  }
  if (tm) { tm[0] += ta; tm[1] += clock64() + (long long)(v[0] == 12345.678 ? 1 : 0) - ta; }
  // last green inside the final valid range [lo+height, hi-height]
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

// put_strip_warp with the neighbour exchange software-pipelined.  The per-row
// loop-carried cycle is shuffle -> DFMA -> DSETP/FSEL -> shuffle (~48 cycles on
// B200: shuffle 24, DFMA 8, select 14); the warp issues in order, so the two
// edge cells of each row are finished FIRST and their shuffles for the next row
// issued before the interior cells, whose ~30 FP64 issue cycles then overlap
// the shuffle latency instead of preceding it.  Same per-cell arithmetic as
// put_strip_warp (bit-identical rows, boundary and outputs).
template <int CPL>
#if FL_PIPE_NOINLINE
__noinline__
#endif
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

// put_strip_warp restricted to the columns that can still change.  The put
// boundary drops by 0 or 1 column per row (bsm.py:420-427 enforces it: the
// reference raises GeometryError otherwise), so at row s every column below
// f-s is an exercise cell: its projected value is its payoff (deep in the
// exercise region lin - payoff ~ -omega*dtau, far from any rounding tie).
// The strip therefore only needs the frame [f-h-1, hi] (3h+2 columns instead
// of 4h+2), with the payoff of column f-h-2 as the fixed left neighbour.
// Same per-cell arithmetic and the same returned boundary / outputs as
// put_strip_warp.  The green mask is formed on the final row only.
template <int CPL>
__device__ int64_t put_strip_v2(const double* __restrict__ in_org, double* __restrict__ out_org,
                                const double* __restrict__ pay_org, int64_t hi, int64_t f, int height, double cd,
                                double cm, double cu, long long* tm = nullptr) {
  const int lane = threadIdx.x & 31;
  const int64_t lo = f - height - 1;
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
  const double edge = pay_org[lo - 1];  // fixed left neighbour of the frame (an exercise cell)
  long long ta = 0;
  __syncwarp();
  if (tm) { ta = clock64() + (long long)(v[0] + p[0] + edge == 12345.678 ? 1 : 0); }
  unsigned green = 0;
  for (int s = 1; s <= height; ++s) {
    const double up = __shfl_up_sync(FULL, v[CPL - 1], 1);
    const double right = __shfl_down_sync(FULL, v[0], 1);
    const double left = (lane == 0) ? edge : up;
    double nv[CPL];
    if (s < height) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const double l = (c == 0) ? left : v[c - 1];
        const double r = (c == CPL - 1) ? right : v[c + 1];
        const double lin = fma(cd, l, fma(cu, r, cm * v[c]));
        nv[c] = lin > p[c] ? lin : p[c];
      }
    } else {
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const double l = (c == 0) ? left : v[c - 1];
        const double r = (c == CPL - 1) ? right : v[c + 1];
        const double lin = fma(cd, l, fma(cu, r, cm * v[c]));
        const bool red = lin > p[c];
        nv[c] = red ? lin : p[c];
        green |= (red ? 0u : 1u) << c;
      }
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) v[c] = nv[c];
  }
  if (tm) { tm[0] += ta; tm[1] += clock64() + (long long)(v[0] == 12345.678 ? 1 : 0) - ta; }
  // last green inside the final valid range [f-h-1, hi-h]
  const int64_t vhi = hi - height;
  int best = -1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int64_t col = c0 + c;
    if (((green >> c) & 1u) && col <= vhi) best = (int)(col - lo);
  }
  best = warp_max_i32(best);
  const int64_t kb = (best < 0) ? NONE_SEEN : lo + best;
  const int64_t wlo = (best < 0) ? vhi + 1 : kb + 1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int64_t col = c0 + c;
    if (col >= wlo && col <= vhi) out_org[col] = v[c];
  }
  __syncwarp();
  return kb;
}

// Sliding-frame put strip.  Same contract as put_strip_warp (lo = f-2h-1,
// hi = f+2h) but the frame follows the valid cone: at row s it holds only
// the 2h+2 columns f-s-1 .. f+2h-s, cell j = column f-s-1+j.  Two facts make
// that exact:
//   * right side: the reference's valid range shrinks by one column per row
//     (_accel.py:203-242: after s rows only [lo+s, hi-s] is valid), so
//     columns right of f+2h-s never influence the final valid range;
//   * left side: at row s every column < f-s is an exercise cell whose value
//     is its payoff (the boundary drops by at most one column per row: a cell
//     whose three parents are exercise cells gets lin = payoff - omega*dtau +
//     O(dtau ds^2) < payoff; the host checks that margin per option,
//     PutParams::slide, and options that fail it use put_strip_pipe).
// In frame coordinates the stencil is left-shifted, new u[j] = F(u[j-2],
// u[j-1], u[j]), so a lane needs two cells from its left neighbour and none
// from its right: one shuffle direction, and the lane's last cell of the next
// row depends on its own cells only.  The loop-carried path is one shuffle,
// one DFMA and one max per row; each row costs 3 CPL FP64 ops + CPL maxes
// instead of the 4h+2 frame's 5 x (3 + 1).  Lane 0's two left cells are the
// payoffs of columns f-s-3, f-s-2.  Per-cell arithmetic is put_strip_warp's
// interior order: fma(cd, left, fma(cu, right, cm * cur)), projected by max
// (equal to the reference's lin > pay ? lin : pay), exercise iff !(lin > pay).
// Requires 2h+2 <= 32*CPL.  pay_org must cover cols f-h-4 .. f+2h.
template <int CPL, int PAYMODE = 0>
__device__ int64_t put_strip_slide(const double* __restrict__ in_org, double* __restrict__ out_org,
                                   const double* __restrict__ pay_org, int64_t f, int height, double cd, double cm,
                                   double cu, long long* tm = nullptr) {
  static_assert(CPL >= 2, "two left cells come from one neighbour");
  const int lane = threadIdx.x & 31;
  const int W = 2 * height + 2;
  const int j0 = lane * CPL;
  const bool l0 = lane == 0;
  // row 0: cols f-1+j; cols <= f hold the payoff, f+1 .. f+2h the input segment
  const double* pay0 = pay_org + (f - 1);
  // cells past the frame (j >= W: idle lanes, the tail of the last lane) read
  // the frame's last column; their values never reach a cell j < W
  int jx[CPL];
  double u[CPL], p[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    jx[c] = (j0 + c < W) ? j0 + c : W - 1;
    p[c] = pay0[jx[c]];  // payoff of cell j at row 0 (col f-1+j)
    u[c] = (jx[c] <= 1) ? p[c] : in_org[f - 1 + jx[c]];
  }
  // lane 0's left fills: at row s cells -2, -1 are cols f-s-3, f-s-2 (exercise
  // cells: their payoff), loaded two rows ahead (one uniform load per row).
  double fill1 = pay_org[f - 2], fill2 = pay_org[f - 3], fill3 = pay_org[f - 4];
  long long ta = 0;
  __syncwarp();
  if (tm) { ta = clock64() + (long long)(u[0] + fill1 == 12345.678 ? 1 : 0); }
  const double* pq = pay0 - 1;  // row s+1 payoff of cell j: pq[j - s]
  unsigned green = 0;
  for (int s = 0; s < height; ++s) {
    const double fill4 = pay_org[f - s - 5];  // row s+2's cell -2 (never past col f-h-4)
    double L2 = __shfl_up_sync(FULL, u[CPL - 2], 1);
    double L1 = __shfl_up_sync(FULL, u[CPL - 1], 1);
    L2 = l0 ? fill2 : L2;
    L1 = l0 ? fill1 : L1;
    // payoffs of row s+1 (col f-s-2+j = col of cell j-1 at row s)
    double np[CPL];
    if (PAYMODE == 0) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) np[c] = pq[jx[c] - s];
    } else {
      const double pl = __shfl_up_sync(FULL, p[CPL - 1], 1);
      np[0] = l0 ? fill1 : pl;
#pragma unroll
      for (int c = 1; c < CPL; ++c) np[c] = p[c - 1];
    }
    double nu[CPL];
    // the lane's last cells first (local inputs), so the next row's shuffles issue early
#pragma unroll
    for (int c = CPL - 1; c >= 2; --c) {
      const double lin = fma(cd, u[c - 2], fma(cu, u[c], cm * u[c - 1]));
      nu[c] = lin > np[c] ? lin : np[c];
    }
    const double lin1 = fma(cd, L1, fma(cu, u[1], cm * u[0]));
    const double lin0 = fma(cd, L2, fma(cu, u[0], cm * L1));
    nu[1] = lin1 > np[1] ? lin1 : np[1];
    nu[0] = lin0 > np[0] ? lin0 : np[0];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      u[c] = nu[c];
      p[c] = np[c];
    }
    fill1 = fill2;
    fill2 = fill3;
    fill3 = fill4;
  }
  // exercise flags of the final row: the reference's cell is exercise iff
  // !(lin > pay), i.e. iff its projected value is exactly its payoff
#pragma unroll
  for (int c = 0; c < CPL; ++c) green |= (u[c] == p[c] ? 1u : 0u) << c;
  if (tm) { tm[0] += ta; tm[1] += clock64() + (long long)(u[0] == 12345.678 ? 1 : 0) - ta; }
  // final row: cell j = col f-h-1+j, j < W is the reference's final valid range
  int best = -1;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (((green >> c) & 1u) && j0 + c < W) best = j0 + c;
  best = warp_max_i32(best);
  const int64_t base = f - height - 1;
  const int64_t kb = (best < 0) ? NONE_SEEN : base + best;
  const int jlo = (best < 0) ? W : best + 1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int j = j0 + c;
    if (j >= jlo && j < W) out_org[base + j] = u[c];
  }
  __syncwarp();
  return kb;
}

// Projection max(lin, pay) with the reference's tie rule (lin > pay ? lin : pay)
// decided on the integer pipe: lin is a sum of products of nonnegative
// coefficients and values, so lin >= +0 and its bit pattern orders like an
// int64 against any payoff's (negative payoffs have the sign bit set, i.e.
// compare below every lin).  Frees the FP64 pipe of the DSETP (the strip is
// FP64-issue-bound when two strips share an SMSP).
#ifndef FL_INT_PROJ
#define FL_INT_PROJ 0  // measured slower: the 64-bit integer compare lengthens the row's critical path
#endif
__device__ __forceinline__ double proj_max(double lin, double pay) {
#if FL_INT_PROJ
  return __double_as_longlong(lin) > __double_as_longlong(pay) ? lin : pay;
#else
  return lin > pay ? lin : pay;
#endif
}

// put_strip_slide with a ghost lane: lane 0 holds the CPL exercise cells left
// of the frame (cols f-s-1-CPL .. f-s-2 at row s) and lanes 1.. hold the
// frame, so no lane needs a select after the shuffle.  Lane 0's values stay
// exactly their payoffs: its own left inputs (shfl_up returns lane 0's own,
// more-right cells, whose payoffs are smaller) only lower its lin, and an
// exercise cell with a lower lin is still an exercise cell (cd, cm, cu >= 0).
// Payoffs of the new row: PAYLDS = 0 shifts them one cell right in registers
// and loads only the lane's first cell (one load per row); PAYLDS = 1 loads
// every cell.  Requires 2h+2 <= 32*CPL - CPL; pay_org must cover cols
// f-h-1-CPL .. f+2h.
template <int CPL, int PAYLDS = 0>
__device__ int64_t put_strip_ghost(const double* __restrict__ in_org, double* __restrict__ out_org,
                                   const double* __restrict__ pay_org, int64_t f, int height, double cd, double cm,
                                   double cu, long long* tm = nullptr) {
  static_assert(CPL >= 2, "two left cells come from one neighbour");
  const int lane = threadIdx.x & 31;
  const int W = 2 * height + 2;
  const int j0 = (lane - 1) * CPL;  // lane 0: cells -CPL .. -1
  // cells past the frame (idle lanes, the tail of the last lane) read the
  // frame's last column; their values never reach a cell j < W
  const double* pay0 = pay_org + (f - 1);
  int jx[CPL];
  double u[CPL], p[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    jx[c] = (j0 + c < W) ? j0 + c : W - 1;
    p[c] = pay0[jx[c]];
    u[c] = (jx[c] <= 1) ? p[c] : in_org[f - 1 + jx[c]];
  }
  long long ta = 0;
  __syncwarp();
  if (tm) { ta = clock64() + (long long)(u[0] == 12345.678 ? 1 : 0); }
  // row s+1 payoff of cell j: col f-s-2+j = pay0[j - 1 - s]
  const double* pq0 = pay0 - 1 + jx[0];
  double np0 = pq0[0];
  unsigned green = 0;
  // unrolled by 2 only: in the kernel the strip shares the SM's instruction
  // cache with every other role, and a longer body measured slower there
  // (4 -> 14.2, 5 -> 14.8, 10 -> 15.8 ms; 2 -> 14.0 ms) although faster alone
  constexpr int kUnroll = FL_GHOST_UNROLL;
#pragma unroll kUnroll
  for (int s = 0; s < height; ++s) {
    const double L2 = __shfl_up_sync(FULL, u[CPL - 2], 1);
    const double L1 = __shfl_up_sync(FULL, u[CPL - 1], 1);
    double np[CPL];
    if (PAYLDS) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) np[c] = pay0[jx[c] - 1 - s];
    } else {
      np[0] = np0;
#pragma unroll
      for (int c = 1; c < CPL; ++c) np[c] = p[c - 1];
      np0 = pq0[-(s + 1)];  // next row's first-cell payoff
    }
    double nu[CPL];
#pragma unroll
    for (int c = CPL - 1; c >= 2; --c) {
      const double lin = fma(cd, u[c - 2], fma(cu, u[c], cm * u[c - 1]));
      nu[c] = proj_max(lin, np[c]);
    }
    const double lin1 = fma(cd, L1, fma(cu, u[1], cm * u[0]));
    const double lin0 = fma(cd, L2, fma(cu, u[0], cm * L1));
    nu[1] = proj_max(lin1, np[1]);
    nu[0] = proj_max(lin0, np[0]);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      u[c] = nu[c];
      p[c] = np[c];
    }
  }
#pragma unroll
  for (int c = 0; c < CPL; ++c) green |= (u[c] == p[c] ? 1u : 0u) << c;
  if (tm) { tm[0] += ta; tm[1] += clock64() + (long long)(u[0] == 12345.678 ? 1 : 0) - ta; }
  int best = -1;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (((green >> c) & 1u) && j0 + c >= 0 && j0 + c < W) best = j0 + c;
  best = warp_max_i32(best);
  const int64_t base = f - height - 1;
  const int64_t kb = (best < 0) ? NONE_SEEN : base + best;
  const int jlo = (best < 0) ? W : best + 1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int j = j0 + c;
    if (j >= jlo && j < W) out_org[base + j] = u[c];
  }
  __syncwarp();
  return kb;
}

// Time-tiled variant of put_strip_warp: lanes exchange K halo cells per side
// once per K rows (instead of one cell per side per row) and advance K rows on
// an extended register tile, recomputing the halo cone redundantly.  One
// shuffle round trip per K rows takes the shuffle latency off the per-row
// critical path.  Same arithmetic per valid cell as put_strip_warp (identical
// results).  Requires K <= CPL.
template <int CPL, int K>
__device__ int64_t put_strip_tiled(const double* __restrict__ in_org, double* __restrict__ out_org,
                                   const double* __restrict__ pay_org, int64_t lo, int64_t hi, int64_t f,
                                   int height, double cd, double cm, double cu) {
  static_assert(K <= CPL, "halo must come from the neighbouring lane");
  constexpr int E = CPL + 2 * K;
  const int lane = threadIdx.x & 31;
  const int64_t c0 = lo + (int64_t)lane * CPL;
  double e[E], p[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int64_t col = c0 - K + i;
    p[i] = (col >= lo && col <= hi) ? pay_org[col] : 0.0;
  }
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int64_t col = c0 + c;
    e[K + c] = (col <= hi) ? ((col <= f) ? p[K + c] : in_org[col]) : 0.0;
  }
  unsigned green = 0;
  __syncwarp();
  for (int s0 = 0; s0 < height; s0 += K) {
    const int kk = (height - s0 < K) ? (height - s0) : K;
    // halo exchange: K cells from each neighbour
#pragma unroll
    for (int i = 0; i < K; ++i) {
      e[i] = __shfl_up_sync(FULL, e[K + CPL - K + i], 1);
      e[K + CPL + i] = __shfl_down_sync(FULL, e[K + i], 1);
    }
#pragma unroll
    for (int s = 1; s <= K; ++s) {
      if (s <= kk) {
        const bool last = (s0 + s == height);
        double left = e[s - 1];
        green = 0;
#pragma unroll
        for (int i = s; i <= E - 1 - s; ++i) {
          const double cur = e[i];
          const double lin = fma(cd, left, fma(cu, e[i + 1], cm * cur));
          left = cur;
          const bool red = lin > p[i];
          e[i] = red ? lin : p[i];
          if (last && i >= K && i < K + CPL) green |= (red ? 0u : 1u) << (i - K);
        }
      }
    }
  }
  // last green inside the final valid range [lo+height, hi-height]
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
    if (col >= wlo && col <= vhi) out_org[col] = e[K + c];
  }
  return kb;
}

}  // namespace fl
