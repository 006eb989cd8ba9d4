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


}  // namespace fl
