// tools/conv_variants.cuh -- helper-warp direct-correlation variants that were
// measured and NOT kept in the product (fl_sched.cuh: conv_direct_blk is the
// production one).  Used by the microbenchmarks in tools/ only; results in
// profiles/r01_experiments.md.
#pragma once

#include "../paper_2303_02317_b200/csrc/fl_sched.cuh"

namespace fl {

// y[k] = sum_{r<M} w[r] x[k+r], k < Lout, on the calling warp (x, w normally
// in shared memory).  Lane l produces outputs k0+l+32j (j < B) of a pass:
// consecutive lanes read consecutive x (bank-conflict free), w[r] is a
// broadcast, and every output keeps two partial sums (even / odd taps) to
// halve its dependent DFMA chain.  Reads x only inside [0, Lout+M-1).
template <int B>
__device__ __forceinline__ void conv_direct_pass(const double* __restrict__ x, double* __restrict__ y, int64_t k0,
                                                 int64_t Lout, const double* __restrict__ w, int M) {
  const int lane = lane_id();
  double ae[B], ao[B];
  const double* xp[B];
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const int64_t k = k0 + lane + 32 * j;
    xp[j] = x + (k < Lout ? k : Lout - 1);
    ae[j] = 0.0;
    ao[j] = 0.0;
  }
  int r = 0;
#pragma unroll 4
  for (; r + 1 < M; r += 2) {
    const double w0 = w[r], w1 = w[r + 1];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      ae[j] = fma(w0, xp[j][r], ae[j]);
      ao[j] = fma(w1, xp[j][r + 1], ao[j]);
    }
  }
  if (r < M) {
    const double w0 = w[r];
#pragma unroll
    for (int j = 0; j < B; ++j) ae[j] = fma(w0, xp[j][r], ae[j]);
  }
#pragma unroll
  for (int j = 0; j < B; ++j) {
    const int64_t k = k0 + lane + 32 * j;
    if (k < Lout) y[k] = ae[j] + ao[j];
  }
}

// Lout <= 64: lane l produces the two consecutive outputs 2l, 2l+1, sliding a
// 3-value window of x through registers (one new x per tap instead of two).
// Reads x[0 .. Lout+M-1] (one past the window when Lout is odd: callers keep
// slack behind x) and w[0 .. M-1].
__device__ __forceinline__ void conv_direct_pairs(const double* __restrict__ x, double* __restrict__ y, int Lout,
                                                  const double* __restrict__ w, int M) {
  const int k = 2 * lane_id();
  const double* xk = x + (k < Lout ? k : 0);
  double a0e = 0.0, a0o = 0.0, a1e = 0.0, a1o = 0.0;
  double xc = xk[0];
  int r = 0;
#pragma unroll 4
  for (; r + 1 < M; r += 2) {
    const double w0 = w[r], w1 = w[r + 1];
    const double x1 = xk[r + 1], x2 = xk[r + 2];
    a0e = fma(w0, xc, a0e);
    a1e = fma(w0, x1, a1e);
    a0o = fma(w1, x1, a0o);
    a1o = fma(w1, x2, a1o);
    xc = x2;
  }
  if (r < M) {
    const double w0 = w[r];
    a0e = fma(w0, xc, a0e);
    a1e = fma(w0, xk[r + 1], a1e);
  }
  if (k < Lout) y[k] = a0e + a0o;
  if (k + 1 < Lout) y[k + 1] = a1e + a1o;
}


// conv_direct_blk without shared-memory bank conflicts.  The helpers' x loads
// were the SM's largest source of conflict wavefronts (output groups 8 apart
// put lanes og and og+2 on one bank), and every queued wavefront delays the
// chain warps' shuffles.  Here the taps are shifted by 3 (three leading zero
// weights, M' = M + 3), lane (og, tg) takes the taps [tg Q + og%4, + Q) of the
// shifted kernel with Q = 4 (mod 16): within a half-warp the x addresses
// 8 og + og%4 + tg Q (+ step) and the weight addresses og%4 + tg Q (+ step)
// then fall on 16 distinct banks.  Rounding Q up adds zero taps (<= 15 per
// quarter).  Same outputs as conv_direct_blk up to the summation order.
__device__ __forceinline__ void conv_direct_blk_cf(const double* __restrict__ x, double* __restrict__ y, int Lout,
                                                   const double* __restrict__ w, int M) {
  const int lane = lane_id();
  const int tg = lane & 3, og = lane >> 2;
  const int Mp = M + 3;
  int Q = (Mp + 3) >> 2;
  Q += (20 - (Q & 15)) & 15;  // Q = 4 (mod 16)
  const int s = tg * Q + (og & 3);
  const int e = s + Q;
  const int xlen = Lout + M - 1;
  const int xb = 8 * og - 3;  // x index of output 8 og at shifted tap 0
  double acc[8], xw[12];
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    acc[b] = 0.0;
    const int i = xb + s + b;
    xw[b] = (i >= 0 && i < xlen) ? x[i] : 0.0;
  }
  for (int r = s; r < e; r += 4) {
    double wv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = xb + r + 8 + j;
      xw[8 + j] = (i >= 0 && i < xlen) ? x[i] : 0.0;
      const int t = r + j - 3;  // unshifted tap
      wv[j] = (t >= 0 && t < M) ? w[t] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[b] = fma(wv[j], xw[b + j], acc[b]);
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) xw[b] = xw[b + 4];
  }
  const bool b0 = tg & 1, b1 = (tg >> 1) & 1;
  double k4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = b0 ? acc[i] : acc[i + 4];
    const double keep = b0 ? acc[i + 4] : acc[i];
    k4[i] = keep + __shfl_xor_sync(FULL, send, 1);
  }
  double k2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = b1 ? k4[i] : k4[i + 2];
    const double keep = b1 ? k4[i + 2] : k4[i];
    k2[i] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  const int k = 8 * og + 4 * b0 + 2 * b1;
  if (k < Lout) y[k] = k2[0];
  if (k + 1 < Lout) y[k + 1] = k2[1];
}

}  // namespace fl
