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
#include <cstdlib>

#include "fl_common.cuh"
#include "fl_kernels.h"

namespace fl {

constexpr int64_t SWEEP_NO_REC = INT64_MIN;

// ---------------------------------------------------------------------------
// put: forward march n = 1..T over 2T+1 columns, valid window [s, 2T - s]

template <int NT, int CPT>
__global__ void __launch_bounds__(NT) put_sweep_kernel(const PutParams* __restrict__ opts,
                                                       const int32_t* __restrict__ order, int nwork, BatchOut out) {
  apply_dlist(out, order, nwork);
  __shared__ double eL[2][NT], eR[2][NT];
  __shared__ int wlg[2][NT / 32];
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
    auto flush = [&](int row, int b) {  // warp 0: the record of `row` from its per-warp maxima
      if (rec && warp == 0) {
        int m = lane < NT / 32 ? wlg[b][lane] : -1;
        m = warp_max_i32(m);
        if (lane == 0 && row < out.cap) {
          out.bt[(int64_t)o * out.cap + row] = row;
          out.bc[(int64_t)o * out.cap + row] = (m < 0) ? SWEEP_NO_REC : lo + m;
        }
      }
    };
    for (int s = 1; s <= n; ++s) {
      const int b = s & 1;
      eL[b][t] = v[0];
      eR[b][t] = v[CPT - 1];
      __syncthreads();
      if (s >= 2) flush(s - 1, b ^ 1);
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
        if (lane == 0) wlg[b][warp] = lg;
      }
    }
    __syncthreads();
    if (n >= 1) flush(n, n & 1);
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
// call / European: backward induction i = T-1..0 over columns 0..i

template <int NT, int CPT, bool PROJ>
__global__ void __launch_bounds__(NT) call_sweep_kernel(const CallParams* __restrict__ copts,
                                                        const EuroParams* __restrict__ eopts,
                                                        const int32_t* __restrict__ order, int nwork, BatchOut out) {
  apply_dlist(out, order, nwork);
  __shared__ double eL[2][NT];
  __shared__ double sscale[2];
  __shared__ int wfg[2][NT / 32];
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
    auto flush = [&](int row, int b) {  // warp 0: first exercise column of `row`
      if (rec && warp == 0) {
        int m = lane < NT / 32 ? wfg[b][lane] : NONE;
        m = warp_min_i32(m);
        if (lane == 0 && row < out.cap) {
          out.bt[(int64_t)o * out.cap + row] = row;
          out.bc[(int64_t)o * out.cap + row] = (m == NONE) ? SWEEP_NO_REC : (int64_t)m;
        }
      }
    };
    if (rec) {
      fg = warp_min_i32(fg);
      if (lane == 0) wfg[n & 1][warp] = fg;
    }
    if (PROJ && t == 0 && n >= 1) sscale[(n - 1) & 1] = __dmul_rn(S0, exp((double)1 * lu));
    for (int i = n - 1; i >= 0; --i) {
      const int b = i & 1;
      eL[b][t] = v[0];
      __syncthreads();
      if (i + 1 <= n) flush(i + 1, b ^ 1);
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
        if (lane == 0) wfg[b][warp] = fg;
      }
    }
    __syncthreads();
    flush(0, 0);
    if (t == 0) {
      out.price[o] = v[0];
      out.status[o] = 0;
      if (out.bcount) out.bcount[o] = PROJ ? n + 1 : 0;
    }
    __syncthreads();
  }
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

cudaError_t launch_call_sweep(const CallParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                              BatchOut out, cudaStream_t stream) {
  return launch_call_sweep_t<true>(opts, nullptr, order, nwork, n_max, grid, out, stream);
}

cudaError_t launch_euro_sweep(const EuroParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                              BatchOut out, cudaStream_t stream) {
  return launch_call_sweep_t<false>(nullptr, opts, order, nwork, n_max, grid, out, stream);
}

}  // namespace fl
