// fl_callstrip.cuh -- warp-level leaf strips of the American call
// (binomial_strip_sweep, _accel.py:105-160, as driven by american._solve,
// american.py:201-225): one strip of height h <= 32 over the h columns
// lo .. j of the continuation run, on one warp.
#pragma once

#include "fl_common.cuh"
#include "host_params.h"

namespace fl {


// Leaf strip (binomial_strip_sweep with lo = j-h+1, height h <= 32) on the
// chain warp: lane l holds column lo+l; reads in_org[lo..j0], writes
// out_org[lo..jp], returns jp (the last continuation column of the final
// row).  The call boundary only moves left as rows descend
// (american.py:232-251 enforces it), so every column right of the row's
// boundary is an exercise cell for the rest of the strip: advancing all strip
// columns with the projected update max(wd v + wu v', green) reproduces the
// analytic exercise values there, and the boundary is needed only once, on
// the last row (first green by one warp min).  Cells beyond the lattice edge
// (col > child) are never read by valid cells.  The e2 factors come from a
// per-option shared table, the parent base of row s+1 is carried from row s
// (one broadcast shuffle per row), and every value that does not depend on
// the row's neighbour exchange (the green value, the out-of-strip right
// neighbour, wd v) is formed before the exchange lands.  Operation order as
// _accel.py:143-158 (unfused products and sums).
__device__ int64_t call_leaf_v3(const CallParams& P, const double* __restrict__ in_org, double* __restrict__ out_org,
                                int64_t lo, int64_t top_row, int64_t j0, int height, double* cells,
                                const double* __restrict__ e2) {
  const int lane = threadIdx.x & 31;
  const int W = (int)(j0 - lo + 1);
  const int64_t col = lo + lane;
  double v = (lane < W) ? in_org[col] : 0.0;
  const double e2_me = e2[lane], e2_nx = e2[lane + 1];
  const double Bl = __dmul_rn(P.S, exp((double)(2 * lo - (top_row - lane)) * P.lu));
  const double B32 = __dmul_rn(P.S, exp((double)(2 * lo - (top_row - 32)) * P.lu));
  const bool edge = (lane + 1 >= W);  // right neighbour outside the strip: exercise value
  double bp = __shfl_sync(FULL, Bl, 0);
  bool green = false;
  // unrolled by 2 only (instruction-cache footprint; C2 4.45 -> 4.30 ms, C5 630 -> 620 ms)
#pragma unroll 2
  for (int s = 0; s < height; ++s) {
    const double bc = (s + 1 < 32) ? __shfl_sync(FULL, Bl, s + 1) : B32;
    const double right = __shfl_down_sync(FULL, v, 1);
    const double ex_r = __dsub_rn(__dmul_rn(bp, e2_nx), P.K);
    const double grn = __dsub_rn(__dmul_rn(bc, e2_me), P.K);
    const double a = __dmul_rn(P.wd, v);
    const double vr = edge ? ex_r : right;
    const double lin = __dadd_rn(a, __dmul_rn(P.wu, vr));
    green = !(lin >= grn);
    v = green ? grn : lin;
    bp = bc;
  }
  const int64_t child = top_row - height;
  const int64_t top = (j0 < child) ? j0 : child;
  const int fg = warp_min_i32((green && lane < W && col <= top) ? lane : INT32_MAX);
  const int64_t jp = (fg == INT32_MAX) ? top : lo + fg - 1;
  *cells += (double)W * height;
  if (col <= jp && lane < W) out_org[col] = v;
  __syncwarp();
  return jp;
}

// call_leaf_v3 for strips of up to 64 rows and columns: lane l holds the CPL
// consecutive columns lo + l*CPL .. +CPL-1 (one exchange per row: the next
// lane's first column), the row bases of rows 0..64 come from two lane-indexed
// registers.  A taller leaf halves the recursion nodes above it (each costs
// a helper post, a wait and the walk); the row's critical path is unchanged
// (one neighbour shuffle, then the cells of the lane in parallel).  Same
// per-cell arithmetic as call_leaf_v3.  e2 must cover indices 0 .. 32*CPL.
template <int CPL>
__device__ int64_t call_leaf_v4(const CallParams& P, const double* __restrict__ in_org, double* __restrict__ out_org,
                                int64_t lo, int64_t top_row, int64_t j0, int height, double* cells,
                                const double* __restrict__ e2, double* __restrict__ bt = nullptr) {
  const int lane = threadIdx.x & 31;
  const int W = (int)(j0 - lo + 1);
  const int k0 = lane * CPL;
  double v[CPL], e2c[CPL + 1];
  bool edge[CPL], green[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    v[c] = (k0 + c < W) ? in_org[lo + k0 + c] : 0.0;
    edge[c] = (k0 + c + 1 >= W);  // right neighbour outside the strip: exercise value
    green[c] = false;
  }
#pragma unroll
  for (int c = 0; c <= CPL; ++c) e2c[c] = e2[k0 + c];
  // base(t) = S exp((2 lo - (top_row - t)) lu), t = 0..32*CPL: two lane-indexed
  // registers for CPL <= 2, a shared-memory table (broadcast loads) above
  double B0 = 0.0, B1 = 0.0, B64 = 0.0;
  if (CPL <= 2) {
    B0 = __dmul_rn(P.S, exp((double)(2 * lo - (top_row - lane)) * P.lu));
    B1 = __dmul_rn(P.S, exp((double)(2 * lo - (top_row - 32 - lane)) * P.lu));
    B64 = __dmul_rn(P.S, exp((double)(2 * lo - (top_row - 64)) * P.lu));
  } else {
    for (int t = lane; t <= 32 * CPL; t += 32) bt[t] = __dmul_rn(P.S, exp((double)(2 * lo - (top_row - t)) * P.lu));
    __syncwarp();
  }
  double bp = CPL <= 2 ? __shfl_sync(FULL, B0, 0) : bt[0];
  // the exercise value of the right neighbour column at the previous row,
  // bp e2[c+1] - K, IS that column's green value of the previous row: carried
  // in registers (same operations, bit-identical) instead of recomputed, except
  // for the lane's last column (its neighbour lives on the next lane)
  double gp[CPL];
#pragma unroll
  for (int c = 1; c < CPL; ++c) gp[c] = __dsub_rn(__dmul_rn(bp, e2c[c]), P.K);
#pragma unroll 2
  for (int s = 0; s < height; ++s) {
    const int t = s + 1;
    double bc;
    if (CPL <= 2) {
      const double b0 = __shfl_sync(FULL, B0, t & 31), b1 = __shfl_sync(FULL, B1, t & 31);
      bc = (t < 32) ? b0 : (t < 64) ? b1 : B64;
    } else {
      bc = bt[t];
    }
    const double right = __shfl_down_sync(FULL, v[0], 1);
    const double ex_last = __dsub_rn(__dmul_rn(bp, e2c[CPL]), P.K);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const double ex_r = (c + 1 < CPL) ? gp[c + 1] : ex_last;
      const double grn = __dsub_rn(__dmul_rn(bc, e2c[c]), P.K);
      const double a = __dmul_rn(P.wd, v[c]);
      const double vr = edge[c] ? ex_r : (c + 1 < CPL ? v[c + 1] : right);
      const double lin = __dadd_rn(a, __dmul_rn(P.wu, vr));
      green[c] = !(lin >= grn);
      v[c] = green[c] ? grn : lin;
      if (c > 0) gp[c] = grn;
    }
    bp = bc;
  }
  const int64_t child = top_row - height;
  const int64_t top = (j0 < child) ? j0 : child;
  int mine = INT32_MAX;
#pragma unroll
  for (int c = CPL - 1; c >= 0; --c)
    if (green[c] && k0 + c < W && lo + k0 + c <= top) mine = k0 + c;
  const int fg = warp_min_i32(mine);
  const int64_t jp = (fg == INT32_MAX) ? top : lo + fg - 1;
  *cells += (double)W * height;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (lo + k0 + c <= jp && k0 + c < W) out_org[lo + k0 + c] = v[c];
  __syncwarp();
  return jp;
}

}  // namespace fl
