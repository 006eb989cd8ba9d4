// fl_sweep.cu -- time-resident O(T^2) sweeps: the reference's explicit
// baselines with the whole lattice row held in registers.
//
//   put_sweep_kernel   replaces _accel.put_march_window     (_accel.py:163-200)
//                      as driven by bsm.baseline_put_fd       (bsm.py:273-338)
//   call_sweep_kernel  replaces _accel.american_call_backward (_accel.py:62-102)
//                      as driven by binomial.baseline_american_call (binomial.py:94-158)
//                      and, without the projection, _accel.european_backward
//                      (_accel.py:49-59, binomial.baseline_european binomial.py:80-91)
//
// One CTA owns one option for all T rows: thread t holds CPT consecutive
// cells of the row (and their exercise values) in registers for the whole
// sweep, so a row costs CPT cell updates per thread from registers plus ONE
// shared-memory exchange of the two edge cells and one barrier -- instead of
// a global-memory ping-pong row per step (the round-1 kernels, kept below as
// the fallback for rows wider than the register tile).  Edge buffers are
// double-buffered by row parity, so the exchange needs a single barrier per
// row.  The boundary record of row s (largest exercise column for the put,
// first exercise column for the call) is reduced per warp in the row itself
// and across warps one row later, after the next barrier, by warp 0.
//
// Arithmetic is the reference's, unfused and left to right
// (cm*cur + cu*right) + cd*left  and  wd*v[j] + wu*v[j+1], ties as the
// reference (put exercise iff payoff >= lin, call continuation iff lin >=
// exercise).  The exercise tables come from the device exp (<= 1 ulp from
// numpy's), as in the round-1 kernels.
#include <cooperative_groups.h>
#include <cstdlib>

#include "fl_common.cuh"
#include "fl_kernels.h"

namespace fl {

constexpr int64_t SWEEP_NO_REC = INT64_MIN;
constexpr int SWEEP_RB = 8;  // rows per boundary-record flush

// ---------------------------------------------------------------------------
// put: forward march n = 1..T over 2T+1 columns, valid window [s, 2T - s]

template <int NT, int CPT>
__global__ void __launch_bounds__(NT) put_sweep_kernel(const PutParams* __restrict__ opts,
                                                       const int32_t* __restrict__ order, int nwork, BatchOut out) {
  apply_dlist(out, order, nwork);
  __shared__ double eL[2][NT], eR[2][NT];
  __shared__ int wlg[2][SWEEP_RB][NT / 32];  // records: chunk parity, row of the chunk, warp
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool rec = out.bt != nullptr && out.cap > 0;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int o = order[w];
    const PutParams P = opts[o];
    const int n = (int)P.n;
    const int W = 2 * n + 1;
    const int64_t lo = P.ks - P.n;
    const int c0 = t * CPT;
    double v[CPT], p[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int k = c0 + c;
      p[c] = (k < W) ? 1.0 - exp((double)(lo + k) * P.ds) : 0.0;  // bsm.py:241-244
      v[c] = p[c] > 0.0 ? p[c] : 0.0;
    }
    if (rec && t == 0) {
      out.bt[(int64_t)o * out.cap] = 0;
      out.bc[(int64_t)o * out.cap] = (P.ks + P.n < 0) ? P.ks + P.n : 0;
    }
    // records of a finished chunk of SWEEP_RB rows (rows r0 ..): thread j
    // combines row r0+j's per-warp maxima (one barrier-free pass per chunk
    // instead of a reduction on one warp's path every row)
    auto flush_chunk = [&](int r0, int qq) {
      if (rec && t < SWEEP_RB && r0 + t <= n && r0 + t < out.cap) {
        int m = -1;
        for (int wi = 0; wi < NT / 32; ++wi) m = wlg[qq][t][wi] > m ? wlg[qq][t][wi] : m;
        out.bt[(int64_t)o * out.cap + r0 + t] = r0 + t;
        out.bc[(int64_t)o * out.cap + r0 + t] = (m < 0) ? SWEEP_NO_REC : lo + m;
      }
    };
    for (int s = 1; s <= n; ++s) {
      const int b = s & 1;
      const int ch = (s - 1) / SWEEP_RB, cq = ch & 1, cr = (s - 1) - ch * SWEEP_RB;
      eL[b][t] = v[0];
      eR[b][t] = v[CPT - 1];
      __syncthreads();
      if (cr == 0 && ch > 0) flush_chunk(1 + (ch - 1) * SWEEP_RB, cq ^ 1);
      int lg = -1;
      if (c0 + CPT - 1 >= s && c0 <= W - 1 - s) {
        double left = (t > 0) ? eR[b][t - 1] : 0.0;
        const double right_edge = (t < NT - 1) ? eL[b][t + 1] : 0.0;
        // branch-free over the tile (cells outside the valid window keep
        // their value): predicated selects keep the tile in registers
        const unsigned span = (unsigned)(W - 1 - 2 * s);
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int k = c0 + c;
          const double cur = v[c];
          const double right = (c + 1 < CPT) ? v[c + 1] : right_edge;
          // _accel.py:192-199: cm*cur + cu*right + cd*left, no contraction
          const double lin = __dadd_rn(__dadd_rn(__dmul_rn(P.cm, cur), __dmul_rn(P.cu, right)),
                                       __dmul_rn(P.cd, left));
          const bool in = (unsigned)(k - s) <= span;
          const bool red = lin > p[c];
          v[c] = in ? (red ? lin : p[c]) : cur;
          lg = (in && !red) ? k : lg;
          left = cur;
        }
      }
      if (rec) {
        lg = warp_max_i32(lg);
        if (lane == 0) wlg[cq][cr][warp] = lg;
      }
    }
    __syncthreads();
    if (n >= 1) flush_chunk(1 + ((n - 1) / SWEEP_RB) * SWEEP_RB, ((n - 1) / SWEEP_RB) & 1);
    // the apex is column n (array offset T of the window)
    if (n >= c0 && n < c0 + CPT) {
      double apex = 0.0;
#pragma unroll
      for (int c = 0; c < CPT; ++c)
        if (c0 + c == n) apex = v[c];
      out.price[o] = P.K * apex;
      out.status[o] = 0;
      if (out.bcount) out.bcount[o] = n + 1;
    }
    __syncthreads();  // the next option reuses the edge / record buffers
  }
}

// ---------------------------------------------------------------------------
// put, one option over a CLUSTER of C CTAs (C SMs), time-tiled: CTA r owns the
// window columns [a, b) = [r W/C, (r+1) W/C) and holds them plus a K-column
// halo on each side in registers.  Every K rows the CTAs publish their K edge
// columns in shared memory (double-buffered by tile parity), one cluster
// barrier makes them visible, and each CTA reads its neighbours' edges through
// distributed shared memory; then K rows run locally (per-row edge exchange
// inside the CTA, as put_sweep_kernel), the halo's stale cells shrinking by
// one per row and never reaching the owned columns.  One cluster barrier per
// K rows instead of per row; a single option gets C SMs of FP64 throughput.
// Boundary records: per row, each CTA's largest exercise column among its
// owned columns, combined across the cluster by atomicMax into the record
// (initialised to NO_GREEN).  Same per-cell arithmetic as put_sweep_kernel.

namespace cg = cooperative_groups;

template <int NT, int CPT, int K>
__global__ void __launch_bounds__(NT) put_sweep_cluster_kernel(const PutParams* __restrict__ opts,
                                                               const int32_t* __restrict__ order, int nwork,
                                                               BatchOut out) {
  apply_dlist(out, order, nwork);
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), r = (int)cl.block_rank();
  const int cid = blockIdx.x / C, ncl = gridDim.x / C;
  __shared__ double exL[2][K], exR[2][K];  // my first / last K owned columns, by tile parity
  __shared__ double eL[2][NT], eR[2][NT];
  __shared__ int wlg[2][K][NT / 32];  // per tile parity, row of the tile, warp
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool rec = out.bt != nullptr && out.cap > 0;
  for (int w = cid; w < nwork; w += ncl) {
    const int o = order[w];
    const PutParams P = opts[o];
    const int n = (int)P.n;
    const int W = 2 * n + 1;
    const int64_t lo = P.ks - P.n;
    const int chunk = (W + C - 1) / C;
    const int a = r * chunk < W ? r * chunk : W, b = (r + 1) * chunk < W ? (r + 1) * chunk : W;
    const int x0 = a - K;  // first extended column
    const int c0 = x0 + t * CPT;
    double v[CPT], p[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int k = c0 + c;
      p[c] = (k >= 0 && k < W) ? 1.0 - exp((double)(lo + k) * P.ds) : 0.0;  // bsm.py:241-244
      v[c] = p[c] > 0.0 ? p[c] : 0.0;
    }
    if (rec) {  // records of rows r, r+C, ...: time and NO_GREEN (the atomicMax identity)
      for (int row = r + C * t; row <= n && row < out.cap; row += C * NT) {
        out.bt[(int64_t)o * out.cap + row] = row;
        out.bc[(int64_t)o * out.cap + row] = (row == 0) ? ((P.ks + P.n < 0) ? P.ks + P.n : 0) : SWEEP_NO_REC;
      }
    }
    cl.sync();  // records initialised; previous item's export reads done
    // the records of a finished tile: thread j < K combines row s0+j's warp
    // maxima (this CTA's largest owned exercise column) into the cluster's record
    auto flush_tile = [&](int ts0, int qq) {
      if (rec && t < K && ts0 + t <= n) {
        int m = -1;
        for (int wi = 0; wi < NT / 32; ++wi) m = wlg[qq][t][wi] > m ? wlg[qq][t][wi] : m;
        const int row = ts0 + t;
        if (m >= 0 && row < out.cap)
          atomicMax(reinterpret_cast<long long*>(out.bc + (int64_t)o * out.cap + row), (long long)(lo + m));
      }
    };
    int tile = 0;
    for (int s0 = 1; s0 <= n; s0 += K, ++tile) {
      const int q = tile & 1;
      // publish my edge columns (row s0-1), then take the neighbours' as my halo
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int k = c0 + c;
        if (k >= a && k < a + K) exL[q][k - a] = v[c];
        if (k >= b - K && k < b) exR[q][k - (b - K)] = v[c];
      }
      cl.sync();
      if (tile > 0) flush_tile(s0 - K, q ^ 1);
      const double* nbR = r > 0 ? cl.map_shared_rank(&exR[q][0], r - 1) : nullptr;     // left neighbour's last K
      const double* nbL = r + 1 < C ? cl.map_shared_rank(&exL[q][0], r + 1) : nullptr;  // right neighbour's first K
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int k = c0 + c;
        if (nbR && k >= a - K && k < a) v[c] = nbR[k - (a - K)];
        if (nbL && k >= b && k < b + K) v[c] = nbL[k - b];
      }
      const int s1 = (s0 + K - 1 < n) ? s0 + K - 1 : n;
      for (int s = s0; s <= s1; ++s) {
        const int bb = s & 1;
        eL[bb][t] = v[0];
        eR[bb][t] = v[CPT - 1];
        __syncthreads();
        int lg = -1;
        double left = (t > 0) ? eR[bb][t - 1] : 0.0;
        const double right_edge = (t < NT - 1) ? eL[bb][t + 1] : 0.0;
        {
          const unsigned span = (unsigned)(W - 1 - 2 * s);
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const int k = c0 + c;
            const double cur = v[c];
            const double right = (c + 1 < CPT) ? v[c + 1] : right_edge;
            const double lin = __dadd_rn(__dadd_rn(__dmul_rn(P.cm, cur), __dmul_rn(P.cu, right)),
                                         __dmul_rn(P.cd, left));
            const bool in = (unsigned)(k - s) <= span;
            const bool red = lin > p[c];
            v[c] = in ? (red ? lin : p[c]) : cur;
            lg = (in && !red && k >= a && k < b) ? k : lg;
            left = cur;
          }
        }
        if (rec) {
          lg = warp_max_i32(lg);
          if (lane == 0) wlg[q][s - s0][warp] = lg;
        }
      }
    }
    __syncthreads();
    if (tile > 0) flush_tile(1 + (tile - 1) * K, (tile - 1) & 1);
    if (n >= a && n < b && n >= c0 && n < c0 + CPT) {  // the apex column is mine
      double apex = 0.0;
#pragma unroll
      for (int c = 0; c < CPT; ++c)
        if (c0 + c == n) apex = v[c];
      out.price[o] = P.K * apex;
      out.status[o] = 0;
      if (out.bcount) out.bcount[o] = n + 1;
    }
    __syncthreads();
  }
  cl.sync();  // no CTA leaves while a neighbour may still read its exports
}

// ---------------------------------------------------------------------------
// call / European: backward induction i = T-1..0 over columns 0..i

template <int NT, int CPT, bool PROJ>
__global__ void __launch_bounds__(NT) call_sweep_kernel(const CallParams* __restrict__ copts,
                                                        const EuroParams* __restrict__ eopts,
                                                        const int32_t* __restrict__ order, int nwork, BatchOut out) {
  apply_dlist(out, order, nwork);
  __shared__ double eL[2][NT];
  __shared__ double sscale[2];
  __shared__ int wfg[2][SWEEP_RB][NT / 32];  // records: chunk parity, row of the chunk, warp
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool rec = PROJ && out.bt != nullptr && out.cap > 0;
  constexpr int NONE = 0x7fffffff;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int o = order[w];
    double S0, K, wd, wu, lu;
    int n;
    if (PROJ) {
      const CallParams& P = copts[o];
      S0 = P.S; K = P.K; wd = P.wd; wu = P.wu; lu = P.lu; n = (int)P.n;
    } else {
      const EuroParams& E = eopts[o];
      S0 = E.S; K = E.K; wd = E.wd; wu = E.wu; lu = E.lu; n = (int)E.n;
    }
    const int c0 = t * CPT;
    double v[CPT], u2[CPT];
    int fg = NONE;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int j = c0 + c;
      // u2[j] = exp((2j - T) log_up), leaf = spot * u2 - strike (binomial.py:64-77, 139-145)
      u2[c] = exp(__dmul_rn(__dsub_rn(2.0 * (double)j, (double)n), lu));
      const double leaf = __dsub_rn(__dmul_rn(S0, u2[c]), K);
      v[c] = (j <= n && leaf > 0.0) ? leaf : 0.0;
      if (PROJ && j <= n && leaf > 0.0 && fg == NONE) fg = j;
    }
    // records in chunks of SWEEP_RB rows (step j = n - row; chunk j / RB):
    // thread q combines the per-warp minima of step j0+q
    auto flush_chunk = [&](int j0, int qq) {
      const int row = n - (j0 + t);
      if (rec && t < SWEEP_RB && row >= 0 && row < out.cap) {
        int m = NONE;
        for (int wi = 0; wi < NT / 32; ++wi) m = wfg[qq][t][wi] < m ? wfg[qq][t][wi] : m;
        out.bt[(int64_t)o * out.cap + row] = row;
        out.bc[(int64_t)o * out.cap + row] = (m == NONE) ? SWEEP_NO_REC : (int64_t)m;
      }
    };
    if (rec) {  // step 0: the leaf row
      fg = warp_min_i32(fg);
      if (lane == 0) wfg[0][0][warp] = fg;
    }
    if (PROJ && t == 0 && n >= 1) sscale[(n - 1) & 1] = __dmul_rn(S0, exp((double)1 * lu));
    for (int i = n - 1; i >= 0; --i) {
      const int b = i & 1;
      const int jstep = n - i, ch = jstep / SWEEP_RB, cq = ch & 1, cr = jstep - ch * SWEEP_RB;
      eL[b][t] = v[0];
      __syncthreads();
      if (cr == 0) flush_chunk((ch - 1) * SWEEP_RB, cq ^ 1);
      double scale = 0.0;
      if (PROJ) {
        scale = sscale[b];
        // row i-1's exercise scale spot * e^{(T - i + 1) log_up}, one exp per row
        if (t == 0 && i >= 1) sscale[b ^ 1] = __dmul_rn(S0, exp((double)(n - i + 1) * lu));
      }
      fg = NONE;
      if (c0 <= i) {
        const double right_edge = (t < NT - 1) ? eL[b][t + 1] : 0.0;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const int j = c0 + c;
          const double right = (c + 1 < CPT) ? v[c + 1] : right_edge;
          const bool in = j <= i;
          const double lin = __dadd_rn(__dmul_rn(wd, v[c]), __dmul_rn(wu, right));
          if (PROJ) {
            const double grn = __dsub_rn(__dmul_rn(scale, u2[c]), K);
            const bool red = lin >= grn;
            v[c] = in ? (red ? lin : grn) : v[c];
            fg = (in && !red && fg == NONE) ? j : fg;
          } else {
            v[c] = in ? lin : v[c];
          }
        }
      }
      if (rec) {
        fg = warp_min_i32(fg);
        if (lane == 0) wfg[cq][cr][warp] = fg;
      }
    }
    __syncthreads();
    flush_chunk((n / SWEEP_RB) * SWEEP_RB, (n / SWEEP_RB) & 1);
    if (t == 0) {
      out.price[o] = v[0];
      out.status[o] = 0;
      if (out.bcount) out.bcount[o] = PROJ ? n + 1 : 0;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// call / European, one option over a CLUSTER of C CTAs, time-tiled as
// put_sweep_cluster_kernel.  The backward induction reads only the right
// neighbour (wd v[j] + wu v[j+1]), so CTA r owns columns [a, b) and holds a
// K-column halo on its right only; every K rows each CTA publishes its first
// K owned columns for its left neighbour.  First-exercise records combine by
// atomicMin (the identity INT64_MAX, turned into NO_GREEN at the end).

template <int NT, int CPT, bool PROJ, int K>
__global__ void __launch_bounds__(NT) call_sweep_cluster_kernel(const CallParams* __restrict__ copts,
                                                                const EuroParams* __restrict__ eopts,
                                                                const int32_t* __restrict__ order, int nwork,
                                                                BatchOut out) {
  apply_dlist(out, order, nwork);
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), r = (int)cl.block_rank();
  const int cid = blockIdx.x / C, ncl = gridDim.x / C;
  __shared__ double exL[2][K];  // my first K owned columns, by tile parity
  __shared__ double eL[2][NT];
  __shared__ double sscale[2];
  __shared__ int wfg[2][K][NT / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool rec = PROJ && out.bt != nullptr && out.cap > 0;
  constexpr int NONE = 0x7fffffff;
  constexpr long long REC_ID = 0x7fffffffffffffffll;  // atomicMin identity
  for (int w = cid; w < nwork; w += ncl) {
    const int o = order[w];
    double S0, K0, wd, wu, lu;
    int n;
    if (PROJ) {
      const CallParams& P = copts[o];
      S0 = P.S; K0 = P.K; wd = P.wd; wu = P.wu; lu = P.lu; n = (int)P.n;
    } else {
      const EuroParams& E = eopts[o];
      S0 = E.S; K0 = E.K; wd = E.wd; wu = E.wu; lu = E.lu; n = (int)E.n;
    }
    const int Wc = n + 1;
    const int chunk = (Wc + C - 1) / C;
    const int a = r * chunk < Wc ? r * chunk : Wc, b = (r + 1) * chunk < Wc ? (r + 1) * chunk : Wc;
    const int c0 = a + t * CPT;
    double v[CPT], u2[CPT];
    int fg = NONE;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int j = c0 + c;
      u2[c] = exp(__dmul_rn(__dsub_rn(2.0 * (double)j, (double)n), lu));
      const double leaf = __dsub_rn(__dmul_rn(S0, u2[c]), K0);
      v[c] = (j <= n && leaf > 0.0) ? leaf : 0.0;
      if (PROJ && j < b && j <= n && leaf > 0.0 && fg == NONE) fg = j;
    }
    if (rec) {
      for (int row = r + C * t; row <= n && row < out.cap; row += C * NT) {
        out.bt[(int64_t)o * out.cap + row] = row;
        out.bc[(int64_t)o * out.cap + row] = REC_ID;
      }
    }
    if (PROJ && t == 0 && n >= 1) sscale[(n - 1) & 1] = __dmul_rn(S0, exp((double)1 * lu));
    cl.sync();  // records initialised
    if (rec) {  // the leaf row (step 0)
      fg = warp_min_i32(fg);
      if (lane == 0 && fg != NONE && n < out.cap)
        atomicMin(reinterpret_cast<long long*>(out.bc + (int64_t)o * out.cap + n), (long long)fg);
    }
    auto flush_tile = [&](int i0, int qq) {  // rows i0, i0-1, .. of a finished tile
      const int row = i0 - t;
      if (rec && t < K && row >= 0 && row < out.cap) {
        int m = NONE;
        for (int wi = 0; wi < NT / 32; ++wi) m = wfg[qq][t][wi] < m ? wfg[qq][t][wi] : m;
        if (m != NONE) atomicMin(reinterpret_cast<long long*>(out.bc + (int64_t)o * out.cap + row), (long long)m);
      }
    };
    int tile = 0;
    for (int i0 = n - 1; i0 >= 0; i0 -= K, ++tile) {
      const int q = tile & 1;
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int j = c0 + c;
        if (j >= a && j < a + K) exL[q][j - a] = v[c];
      }
      cl.sync();
      if (tile > 0) flush_tile(i0 + K, q ^ 1);
      const double* nb = r + 1 < C ? cl.map_shared_rank(&exL[q][0], r + 1) : nullptr;  // right neighbour's first K
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int j = c0 + c;
        if (nb && j >= b && j < b + K) v[c] = nb[j - b];
      }
      const int i1 = (i0 - K + 1 > 0) ? i0 - K + 1 : 0;
      for (int i = i0; i >= i1; --i) {
        const int bb = i & 1;
        eL[bb][t] = v[0];
        __syncthreads();
        double scale = 0.0;
        if (PROJ) {
          scale = sscale[bb];
          if (t == 0 && i >= 1) sscale[bb ^ 1] = __dmul_rn(S0, exp((double)(n - i + 1) * lu));
        }
        fg = NONE;
        if (c0 <= i) {
          const double right_edge = (t < NT - 1) ? eL[bb][t + 1] : 0.0;
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const int j = c0 + c;
            const double right = (c + 1 < CPT) ? v[c + 1] : right_edge;
            const bool in = j <= i;
            const double lin = __dadd_rn(__dmul_rn(wd, v[c]), __dmul_rn(wu, right));
            if (PROJ) {
              const double grn = __dsub_rn(__dmul_rn(scale, u2[c]), K0);
              const bool red = lin >= grn;
              v[c] = in ? (red ? lin : grn) : v[c];
              fg = (in && !red && fg == NONE && j < b) ? j : fg;
            } else {
              v[c] = in ? lin : v[c];
            }
          }
        }
        if (rec) {
          fg = warp_min_i32(fg);
          if (lane == 0) wfg[q][i0 - i][warp] = fg;
        }
      }
    }
    __syncthreads();
    if (tile > 0) flush_tile(n - 1 - (tile - 1) * K, (tile - 1) & 1);
    cl.sync();  // every record combined: the untouched identities are NO_GREEN
    if (rec) {
      for (int row = r + C * t; row <= n && row < out.cap; row += C * NT) {
        long long* pc = reinterpret_cast<long long*>(out.bc + (int64_t)o * out.cap + row);
        if (*pc == REC_ID) *pc = SWEEP_NO_REC;
      }
    }
    if (r == 0 && t == 0) {
      out.price[o] = v[0];
      out.status[o] = 0;
      if (out.bcount) out.bcount[o] = PROJ ? n + 1 : 0;
    }
    __syncthreads();
  }
  cl.sync();
}

// ---------------------------------------------------------------------------
// launchers: the smallest tile that holds the batch's widest row

struct SweepTile {
  int nt, cpt;
};
// (threads, cells per thread): registers cap CPT (two doubles per cell), so
// the widest tiles use fewer threads
constexpr SweepTile kSweepTiles[] = {{128, 2}, {256, 4}, {512, 8}, {768, 11}, {512, 20}};
constexpr int64_t kSweepMaxCells = 512 * 20;

inline int sweep_tile_for(int64_t cells) {
  for (int i = 0; i < (int)(sizeof(kSweepTiles) / sizeof(kSweepTiles[0])); ++i)
    if ((int64_t)kSweepTiles[i].nt * kSweepTiles[i].cpt >= cells) return i;
  return -1;
}

int64_t sweep_max_cells() { return kSweepMaxCells; }

// FL_NO_SWEEP=1 (A/B tools only): route every baseline to the round-1
// global-memory march
bool sweep_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("FL_NO_SWEEP");
    return e && e[0] == '1';
  }();
  return off;
}

// A few options: C = 2..8 CTAs per option (a cluster), K = 8 rows per cluster
// barrier.  Returns cudaErrorNotSupported when the batch is large enough to
// fill the GPU with one CTA per option (put_sweep_kernel is then cheaper).
constexpr int SWEEP_K = 8;

template <int NT, int CPT>
static cudaError_t launch_put_cluster_t(const PutParams* opts, const int32_t* order, int nwork, int C,
                                        BatchOut out, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * nwork), 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, put_sweep_cluster_kernel<NT, CPT, SWEEP_K>, opts, order, nwork, out);
}

cudaError_t launch_put_sweep_cluster(const PutParams* opts, const int32_t* order, int nwork, int64_t n_max,
                                     BatchOut out, cudaStream_t stream) {
  int dev = 0, nsm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t W = 2 * n_max + 1;
  int C = 8;
  // every CTA but the last owns >= 2K columns (its exports are its own columns)
  while (C > 1 && (C * nwork > nsm || (W + C - 1) / C < 2 * SWEEP_K)) C >>= 1;
  if (C < 2 || sweep_disabled()) return cudaErrorNotSupported;
  const int64_t ext = (W + C - 1) / C + 2 * SWEEP_K;
  // (measured: 1024-thread CTAs with 1-2 cells each are slower than 256
  // threads with 4-8 cells: the per-row barrier dominates)
  if (ext <= 128 * 2) return launch_put_cluster_t<128, 2>(opts, order, nwork, C, out, stream);
  if (ext <= 256 * 4) return launch_put_cluster_t<256, 4>(opts, order, nwork, C, out, stream);
  if (ext <= 256 * 8) return launch_put_cluster_t<256, 8>(opts, order, nwork, C, out, stream);
  if (ext <= 512 * 8) return launch_put_cluster_t<512, 8>(opts, order, nwork, C, out, stream);
  return cudaErrorNotSupported;
}

cudaError_t launch_put_sweep(const PutParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                             BatchOut out, cudaStream_t stream) {
  const int ti = sweep_tile_for(2 * n_max + 1);
  if (ti < 0) return cudaErrorInvalidValue;
  if (grid <= 0) return cudaSuccess;
  switch (ti) {
    case 0: put_sweep_kernel<128, 2><<<grid, 128, 0, stream>>>(opts, order, nwork, out); break;
    case 1: put_sweep_kernel<256, 4><<<grid, 256, 0, stream>>>(opts, order, nwork, out); break;
    case 2: put_sweep_kernel<512, 8><<<grid, 512, 0, stream>>>(opts, order, nwork, out); break;
    case 3: put_sweep_kernel<768, 11><<<grid, 768, 0, stream>>>(opts, order, nwork, out); break;
    default: put_sweep_kernel<512, 20><<<grid, 512, 0, stream>>>(opts, order, nwork, out); break;
  }
  return cudaGetLastError();
}

template <bool PROJ>
static cudaError_t launch_call_sweep_t(const CallParams* copts, const EuroParams* eopts, const int32_t* order,
                                       int nwork, int64_t n_max, int grid, BatchOut out, cudaStream_t stream) {
  const int ti = sweep_tile_for(n_max + 1);
  if (ti < 0) return cudaErrorInvalidValue;
  if (grid <= 0) return cudaSuccess;
  switch (ti) {
    case 0: call_sweep_kernel<128, 2, PROJ><<<grid, 128, 0, stream>>>(copts, eopts, order, nwork, out); break;
    case 1: call_sweep_kernel<256, 4, PROJ><<<grid, 256, 0, stream>>>(copts, eopts, order, nwork, out); break;
    case 2: call_sweep_kernel<512, 8, PROJ><<<grid, 512, 0, stream>>>(copts, eopts, order, nwork, out); break;
    case 3: call_sweep_kernel<768, 11, PROJ><<<grid, 768, 0, stream>>>(copts, eopts, order, nwork, out); break;
    default: call_sweep_kernel<512, 20, PROJ><<<grid, 512, 0, stream>>>(copts, eopts, order, nwork, out); break;
  }
  return cudaGetLastError();
}

template <int NT, int CPT, bool PROJ>
static cudaError_t launch_call_cluster_t(const CallParams* copts, const EuroParams* eopts, const int32_t* order,
                                         int nwork, int C, BatchOut out, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * nwork), 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, call_sweep_cluster_kernel<NT, CPT, PROJ, SWEEP_K>, copts, eopts, order, nwork, out);
}

// a few call / European options: a cluster of SMs per option (cudaErrorNotSupported otherwise)
template <bool PROJ>
static cudaError_t launch_call_sweep_cluster(const CallParams* copts, const EuroParams* eopts, const int32_t* order,
                                             int nwork, int64_t n_max, BatchOut out, cudaStream_t stream) {
  if (out.dlist || sweep_disabled()) return cudaErrorNotSupported;
  int dev = 0, nsm = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  const int64_t W = n_max + 1;
  int C = 8;
  while (C > 1 && (C * nwork > nsm || (W + C - 1) / C < 2 * SWEEP_K)) C >>= 1;
  if (C < 2) return cudaErrorNotSupported;
  const int64_t ext = (W + C - 1) / C + SWEEP_K;
  if (ext <= 128 * 2) return launch_call_cluster_t<128, 2, PROJ>(copts, eopts, order, nwork, C, out, stream);
  if (ext <= 256 * 4) return launch_call_cluster_t<256, 4, PROJ>(copts, eopts, order, nwork, C, out, stream);
  if (ext <= 256 * 8) return launch_call_cluster_t<256, 8, PROJ>(copts, eopts, order, nwork, C, out, stream);
  if (ext <= 512 * 8) return launch_call_cluster_t<512, 8, PROJ>(copts, eopts, order, nwork, C, out, stream);
  return cudaErrorNotSupported;
}

cudaError_t launch_call_sweep(const CallParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                              BatchOut out, cudaStream_t stream) {
  const cudaError_t e = launch_call_sweep_cluster<true>(opts, nullptr, order, nwork, n_max, out, stream);
  if (e != cudaErrorNotSupported) return e;
  return launch_call_sweep_t<true>(opts, nullptr, order, nwork, n_max, grid, out, stream);
}

cudaError_t launch_euro_sweep(const EuroParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                              BatchOut out, cudaStream_t stream) {
  const cudaError_t e = launch_call_sweep_cluster<false>(nullptr, opts, order, nwork, n_max, out, stream);
  if (e != cudaErrorNotSupported) return e;
  return launch_call_sweep_t<false>(nullptr, opts, order, nwork, n_max, grid, out, stream);
}

}  // namespace fl
