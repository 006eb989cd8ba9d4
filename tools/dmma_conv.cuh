// tools/dmma_conv.cuh -- the tensor-core (mma.sync .f64) direct correlation
// measured in round 2 as an alternative to the FFT for the recursion nodes'
// mid-size jumps (tools/dmma_conv_bench.cu, profiles/r02_experiments.md): not
// kept in the product -- at these sizes the FP64 pipe DMMA shares with DFMA
// makes it no faster than the FFT in the kernel.
#pragma once

#include "../paper_2303_02317_b200/csrc/fl_conv.cuh"

namespace fl {

// ---------------------------------------------------------------------------
// FP64 tensor-core executor (DMMA) for mid-size jumps.  The valid-mode
// correlation y[k] = sum_r w[r] x[k+r] (r < M) is a dense contraction once
// the row is reshaped into rows of eight, Z[i][m] = x[8i+m]:
//     y[8i+j] = sum_q sum_{m<8} Z[i+q][m] * Wq[m][j],   Wq[m][j] = w[8q+m-j],
// i.e. for every q a (rows x 8) x (8 x 8) product: mma.sync m16n8k4 .f64
// (two k-steps per q) over 16-row tiles of 128 outputs, fp64 accumulation.
// One tensor instruction does 512 fused multiply-adds with 3 shared loads
// (the DFMA direct path needs ~16 instructions and ~8 loads for the same
// work, the FFT path ~10x the latency for these sizes).  x is staged with a
// row pitch of 10 doubles (conflict-free fragment loads), w with 8 zeros each
// side (the out-of-range Wq entries).

__device__ __forceinline__ void dmma16n8k4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

constexpr int DMMA_PITCH = 10;

// y[0..Lout) for x[0..L) (global) and the window weights w[0..M) (global);
// sbuf holds `cap` doubles of shared memory.  Returns executed flops.
__device__ double conv_dmma(const double* __restrict__ x, int64_t L, double* __restrict__ y, int64_t Lout,
                            const double* __restrict__ w, int M, double* sbuf, int cap, const Grp& g) {
  if (Lout <= 0) return 0.0;
  const int Q = (M + 14) / 8;
  const int wlen = 8 * Q + 16;
  double* sw = sbuf;                 // w[-8 .. 8Q+7]
  double* sx = sbuf + wlen;          // rows of eight at pitch 10
  const int rows_cap = (cap - wlen) / DMMA_PITCH;
  const int lane = g.t & 31, wid = g.t >> 5, nwarps = (g.n + 31) >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  // outputs per chunk: whole 16-row tiles whose x rows fit
  const int tiles_fit = (rows_cap - Q - 1) / 16;
  if (tiles_fit < 1) return -1.0;
  for (int i = g.t; i < wlen; i += g.n) sw[i] = (i >= 8 && i - 8 < M) ? w[i - 8] : 0.0;
  for (int64_t k0 = 0; k0 < Lout; k0 += (int64_t)tiles_fit * 128) {
    const int64_t nk = (Lout - k0 < (int64_t)tiles_fit * 128) ? Lout - k0 : (int64_t)tiles_fit * 128;
    const int tiles = (int)((nk + 127) / 128);
    const int rows = tiles * 16 + Q;
    for (int i = g.t; i < rows * 8; i += g.n) {
      const int64_t src = k0 + i;
      sx[(i >> 3) * DMMA_PITCH + (i & 7)] = (src < L) ? x[src] : 0.0;
    }
    gsync(g);
    for (int tile = wid; tile < tiles; tile += nwarps) {
      double d[4] = {0.0, 0.0, 0.0, 0.0};
      const double* xa = sx + (tile * 16 + gq) * DMMA_PITCH + tq;
      const double* wb = sw + 8 + tq - gq;
#pragma unroll 2
      for (int q = 0; q < Q; ++q) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const double a0 = xa[q * DMMA_PITCH + 4 * kk];
          const double a1 = xa[(q + 8) * DMMA_PITCH + 4 * kk];
          const double b0 = wb[8 * q + 4 * kk];
          dmma16n8k4(d, a0, a1, b0);
        }
      }
      const int64_t o0 = k0 + (int64_t)tile * 128 + 8 * gq + 2 * tq;
      const int64_t o1 = o0 + 64;
      const int64_t lim = k0 + nk;
      if (o0 < lim) y[o0] = d[0];
      if (o0 + 1 < lim) y[o0 + 1] = d[1];
      if (o1 < lim) y[o1] = d[2];
      if (o1 + 1 < lim) y[o1 + 1] = d[3];
    }
    gsync(g);
  }
  return 2.0 * (double)Lout * (double)(8 * Q + 8);
}

// Window of a composed kernel from its halves: W_h[rlo_h + r] = sum_u W_a[u]
// W_b[rlo_h + r - u] over the halves' windows (pa = W_a[rlo_a ..], pb = W_b[rlo_b
// ..]); the tails outside the windows carry < 2e-22 of the mass each.
__device__ void compose_window(const double* __restrict__ pa, int64_t rlo_a, int Ma, const double* __restrict__ pb,
                               int64_t rlo_b, int Mb, double* __restrict__ out, int64_t rlo_h, int Mh, const Grp& g) {
  for (int r = g.t; r < Mh; r += g.n) {
    const int64_t R = rlo_h + r;
    int64_t u0 = R - (rlo_b + Mb - 1), u1 = R - rlo_b;  // W_b index in window
    if (u0 < rlo_a) u0 = rlo_a;
    if (u1 > rlo_a + Ma - 1) u1 = rlo_a + Ma - 1;
    double acc = 0.0;
    for (int64_t u = u0; u <= u1; ++u) acc = fma(pa[u - rlo_a], pb[R - u - rlo_b], acc);
    out[r] = acc;
  }
}

}  // namespace fl
