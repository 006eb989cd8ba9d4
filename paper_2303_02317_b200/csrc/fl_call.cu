// fl_call.cu -- American call on the binomial lattice: device trapezoid
// decomposition (replaces american.fast_american_call and its recursion,
// american.py:201-530) and the O(T^2) projected induction (replaces
// binomial.baseline_american_call / _accel.american_call_backward,
// binomial.py:94-130, _accel.py:62-102).
//
// Same execution model as the put (fl_put.cu): a persistent CTA per option,
// explicit CTA-uniform recursion stack, linear jumps through conv_fft,
// nonlinear leaves on warp 0 (one cell per lane, first-green by warp min),
// the ceil(sqrt(T))-row residual strip as a shared-memory CTA sweep.
#include <cstdint>

#include "fl_common.cuh"
#include "fl_conv.cuh"
#include "fl_kernels.h"
#include "fl_strip.cuh"
#include "host_params.h"

namespace fl {

constexpr int CALL_LEAF = 32;
constexpr int CALL_MAX_DEPTH = 28;
constexpr int CALL_LOGN_MAX = 13;
constexpr int CALL_SLOTS = smem_complex_slots(1 << (CALL_LOGN_MAX - 1));
constexpr int CALL_RESID_CPT = 8;  // residual strip: cells per thread (width <= 2048)

int64_t call_ws_doubles(int64_t n_max) { return 2 * (n_max + 8) + (2 * n_max + 16 * CALL_MAX_DEPTH) + 64; }
int call_fast_smem_bytes() { return CALL_SLOTS * (int)sizeof(double2); }

__device__ __forceinline__ int64_t first_green_rec(int64_t i, int64_t j) {  // american.py:361-363
  return j >= i ? INT64_MIN : j + 1;
}

// Leaf strip (binomial_strip_sweep with lo = j-h+1, height h, h <= 32):
// lane l holds column lo+l.  Reads in_org[lo..j], writes out_org[lo..jp].
__device__ int64_t call_leaf_warp(const CallParams& P, const double* __restrict__ in_org,
                                  double* __restrict__ out_org, int64_t lo, int64_t top_row, int64_t j0,
                                  int height, double* cells) {
  const int lane = threadIdx.x & 31;
  const int W = (int)(j0 - lo + 1);
  const int64_t col = lo + lane;
  double v = (lane < W) ? in_org[col] : 0.0;
  const double e2_me = exp(2.0 * (double)lane * P.lu);         // e2[col - lo]
  const double e2_nx = exp(2.0 * (double)(lane + 1) * P.lu);   // e2[col + 1 - lo]
  // B[t] = S exp((2 lo - (top_row - t)) lu), t = 0..height: parent base of step t
  const double Bl = P.S * exp((double)(2 * lo - (top_row - lane)) * P.lu);
  const double B32 = P.S * exp((double)(2 * lo - (top_row - 32)) * P.lu);
  int64_t j = j0;
  for (int s = 0; s < height; ++s) {
    if (j < lo) break;
    const int64_t child = top_row - s - 1;
    const int64_t top = j < child ? j : child;
    *cells += (double)(top - lo + 1);
    const double bp = __shfl_sync(FULL, Bl, s);
    const double bc = (s + 1 < 32) ? __shfl_sync(FULL, Bl, s + 1) : B32;
    const double right = __shfl_down_sync(FULL, v, 1);
    int fg = INT32_MAX;
    if (col <= top) {
      const double vr = (col + 1 <= j) ? right : fma(bp, e2_nx, -P.K);
      const double lin = fma(P.wd, v, P.wu * vr);
      const double grn = fma(bc, e2_me, -P.K);
      if (lin >= grn) {
        v = lin;
      } else {
        v = grn;
        fg = lane;
      }
    }
    fg = warp_min_i32(fg);
    j = (fg == INT32_MAX) ? top : lo + fg - 1;
  }
  if (col <= j && lane < W) out_org[col] = v;
  return j;
}

// Residual strip over the whole run (american.py:499-521): lo = 0, height = i,
// CTA-wide in shared memory.  Returns j0 and leaves row values in sv.
__device__ int64_t call_resid_cta(const CallParams& P, const double* row_org, int64_t i, int64_t j0, double* sv,
                                  double* se2, int* s_fg, double* cells) {
  const int64_t W = j0 + 1;
  for (int64_t c = threadIdx.x; c <= W; c += CTA_THREADS) {
    sv[c] = (c < W) ? row_org[c] : 0.0;
    se2[c] = exp(2.0 * (double)c * P.lu);
  }
  __syncthreads();
  int64_t j = j0;
  for (int64_t s = 0; s < i; ++s) {
    if (j < 0) break;
    const int64_t parent = i - s, child = parent - 1;
    const int64_t top = j < child ? j : child;
    *cells += (double)(top + 1);
    const double bc = P.S * exp((double)(0 - child) * P.lu);
    const double bp = P.S * exp((double)(0 - parent) * P.lu);
    if (threadIdx.x == 0) *s_fg = INT32_MAX;
    // two-phase update (Jacobi): read all, sync, write
    double nv[CALL_RESID_CPT];
    int k = 0;
    int myfg = INT32_MAX;
    for (int64_t c = threadIdx.x; c <= top && k < CALL_RESID_CPT; c += CTA_THREADS, ++k) {
      const double vr = (c + 1 <= j) ? sv[c + 1] : fma(bp, se2[c + 1], -P.K);
      const double lin = fma(P.wd, sv[c], P.wu * vr);
      const double grn = fma(bc, se2[c], -P.K);
      if (lin >= grn) {
        nv[k] = lin;
      } else {
        nv[k] = grn;
        if (myfg == INT32_MAX) myfg = (int)c;
      }
    }
    myfg = warp_min_i32(myfg);
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && myfg != INT32_MAX) atomicMin(s_fg, myfg);
    k = 0;
    for (int64_t c = threadIdx.x; c <= top && k < CALL_RESID_CPT; c += CTA_THREADS, ++k) sv[c] = nv[k];
    __syncthreads();
    const int fg = *s_fg;
    j = (fg == INT32_MAX) ? top : (int64_t)fg - 1;
    __syncthreads();
  }
  return j;
}

struct CallFrame {
  int64_t i, j, jm;
  double* in_org;
  double* out_org;
  double* asm_org;
  int64_t arena;
  int h, state;
};

__device__ __forceinline__ void cta_bcast(int64_t& v, int64_t* slot) {
  if (threadIdx.x == 0) *slot = v;
  __syncthreads();
  v = *slot;
  __syncthreads();
}

// _solve (american.py:201-257) with an explicit stack.  vals = in_org[j-h+1 .. j];
// writes out_org[j-h+1 .. jp]; returns jp.
__device__ int64_t call_solve(const CallParams& P, const Stencil& st, int64_t i0, int64_t j0, int h0,
                              double* in_org, double* out_org, double* frames, int64_t arena0, double2* sbuf,
                              int64_t* slot, int32_t* err, double* fl) {
  CallFrame stk[CALL_MAX_DEPTH];
  stk[0].i = i0; stk[0].j = j0; stk[0].h = h0; stk[0].in_org = in_org; stk[0].out_org = out_org;
  stk[0].arena = arena0; stk[0].state = 0;
  int sp = 1;
  int64_t ret = 0;
  while (sp > 0) {
    CallFrame& F = stk[sp - 1];
    const int h = F.h;
    const int h1 = (h + 1) / 2, h2 = h - h1;
    if (F.state == 0) {
      if (h <= CALL_LEAF) {
        int64_t jp = 0;
        double cells = 0.0;
        if (threadIdx.x < 32) jp = call_leaf_warp(P, F.in_org, F.out_org, F.j - h + 1, F.i, F.j, h, &cells);
        cta_bcast(jp, slot);
        *fl += 5.0 * cells;  // meaningful on thread 0 (the accumulating thread)
        ret = jp;
        --sp;
        continue;
      }
      const int64_t lo = F.j - h + 1;
      F.asm_org = frames + F.arena - lo;
      // mid: cols lo .. j-h1 of row i-h1
      *fl += conv_fft(F.in_org + lo, h, F.asm_org + lo, h2, h1, st, sbuf, CALL_LOGN_MAX, fl_tw, Grp{(int)threadIdx.x, CTA_THREADS, 0});
      F.state = 1;
      CallFrame& C = stk[sp];
      C.i = F.i; C.j = F.j; C.h = h1; C.in_org = F.in_org; C.out_org = F.asm_org;
      C.arena = F.arena + h + 8; C.state = 0;
      if (++sp >= CALL_MAX_DEPTH) { *err = FL_E_CAPACITY | 1; return 0; }
    } else if (F.state == 1) {
      const int64_t jm = ret;
      if (jm < F.j - h1 || jm > F.j) { *err = FL_E_GEOMETRY | 1; return 0; }
      F.jm = jm;
      const int64_t lo = F.j - h + 1;
      const int64_t A = jm - lo + 1;  // assembled cols lo .. jm
      // bottom: cols lo .. jm-h2 of row i-h
      *fl += conv_fft(F.asm_org + lo, A, F.out_org + lo, A - h2, h2, st, sbuf, CALL_LOGN_MAX, fl_tw, Grp{(int)threadIdx.x, CTA_THREADS, 0});
      F.state = 2;
      CallFrame& C = stk[sp];
      C.i = F.i - h1; C.j = jm; C.h = h2; C.in_org = F.asm_org; C.out_org = F.out_org;
      C.arena = F.arena + h + 8; C.state = 0;
      ++sp;
    } else {
      const int64_t jp = ret;
      if (jp < F.jm - h2 || jp > F.jm) { *err = FL_E_GEOMETRY | 2; return 0; }
      --sp;
    }
  }
  return ret;
}

__device__ void call_record(const BatchOut& out, int o, int32_t& cnt, int64_t t, int64_t c) {
  if (threadIdx.x == 0 && out.bt != nullptr && cnt < out.cap) {
    out.bt[(int64_t)o * out.cap + cnt] = t;
    out.bc[(int64_t)o * out.cap + cnt] = c;
  }
  ++cnt;
}

__global__ void __launch_bounds__(CTA_THREADS, 2)
call_fast_kernel(const CallParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork,
                 int32_t* counter, double* __restrict__ ws, int64_t ws_stride, BatchOut out) {
  extern __shared__ double2 sbuf[];
  __shared__ int s_work;
  __shared__ int s_fg;
  __shared__ int64_t s_slot;
  double* arena = ws + (int64_t)blockIdx.x * ws_stride;
  for (;;) {
    if (threadIdx.x == 0) s_work = atomicAdd(counter, 1);
    __syncthreads();
    const int w = s_work;
    __syncthreads();
    if (w >= nwork) break;
    const int o = order[w];
    const CallParams P = opts[o];
    const int64_t n = P.n;
    double* rowA = arena;
    double* rowB = arena + (n + 8);
    double* frames = arena + 2 * (n + 8);
    const Stencil st{P.wd, P.wu, 0.0, 1};
    double flops = 0.0;
    int32_t err = 0, cnt = 0;
    call_record(out, o, cnt, n, first_green_rec(n, P.top_b));
    int64_t i = n - 1, j = P.junc_j;
    call_record(out, o, cnt, i, first_green_rec(i, j));
    // junction row T-1 (american.py:412-422)
    const int64_t start = P.top_b > 0 ? P.top_b : 0;
    for (int64_t c = threadIdx.x; c <= j; c += CTA_THREADS) {
      double v = 0.0;
      if (c >= start) {
        double l0 = P.S * exp((2.0 * (double)c - (double)n) * P.lu) - P.K;
        double l1 = P.S * exp((2.0 * (double)(c + 1) - (double)n) * P.lu) - P.K;
        l0 = l0 > 0.0 ? l0 : 0.0;
        l1 = l1 > 0.0 ? l1 : 0.0;
        v = fma(P.wd, l0, P.wu * l1);
      }
      rowA[c] = v;
    }
    __syncthreads();
    const int64_t resid = (int64_t)floor(sqrt((double)(n - 1))) + 1;  // isqrt(n-1)+1 (exact below 2^52)
    double* cur = rowA;
    double* nxt = rowB;
    while (i > resid && j >= 0) {
      const int64_t hh = (j + 1 < i - resid) ? j + 1 : i - resid;
      const int h = (int)hh;
      // left: cols 0 .. j-h of row i-h (american.py:341-344)
      if (j + 1 > hh) flops += conv_fft(cur, j + 1, nxt, j + 1 - hh, h, st, sbuf, CALL_LOGN_MAX, fl_tw, Grp{(int)threadIdx.x, CTA_THREADS, 0});
      const int64_t jp = call_solve(P, st, i, j, h, cur, nxt, frames, 0, sbuf, &s_slot, &err, &flops);
      if (err) break;
      i -= hh;
      j = jp;
      call_record(out, o, cnt, i, first_green_rec(i, j));
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
    double price = 0.0;
    if (!err) {
      if (j < 0) {
        price = P.S - P.K;
      } else {
        double* sv = (double*)sbuf;
        double* se2 = sv + (CALL_SLOTS);
        if (j + 2 > CALL_SLOTS || j + 1 > (int64_t)CALL_RESID_CPT * CTA_THREADS) {
          err = FL_E_CAPACITY | 2;
        } else {
          double cells = 0.0;
          const int64_t j0 = call_resid_cta(P, cur, i, j, sv, se2, &s_fg, &cells);
          flops += 5.0 * cells;
          price = (j0 >= 0) ? sv[0] : P.S - P.K;
          if (i > 0) call_record(out, o, cnt, 0, first_green_rec(0, j0));
          __syncthreads();
        }
      }
    }
    if (threadIdx.x == 0) {
      out.price[o] = err ? 0.0 : price;
      out.status[o] = err;
      if (out.bcount) out.bcount[o] = err ? 0 : cnt;
      if (out.flops) atomicAdd(out.flops, (unsigned long long)flops);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// O(T^2) projected backward induction (american_call_backward).

__global__ void __launch_bounds__(CTA_THREADS)
call_baseline_kernel(const CallParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork,
                     double* __restrict__ ws, int64_t ws_stride, BatchOut out) {
  __shared__ int s_fg;
  const int w = blockIdx.x;
  if (w >= nwork) return;
  const int o = order[w];
  const CallParams P = opts[o];
  const int64_t n = P.n;
  double* a = ws + (int64_t)blockIdx.x * ws_stride;
  double* b = a + (n + 2);
  double* u2 = b + (n + 2);
  const bool rec = out.bt != nullptr;
  if (threadIdx.x == 0) s_fg = INT32_MAX;
  __syncthreads();
  for (int64_t j = threadIdx.x; j <= n; j += CTA_THREADS) {
    const double u = exp((2.0 * (double)j - (double)n) * P.lu);
    u2[j] = u;
    const double v = P.S * exp((2.0 * (double)j - (double)n) * P.lu) - P.K;  // leaf_row
    a[j] = v > 0.0 ? v : 0.0;
    if (P.S * u - P.K > 0.0) atomicMin(&s_fg, (int)j);
  }
  __syncthreads();
  auto put_rec = [&](int64_t row, int fg) {
    if (rec && threadIdx.x == 0 && row < out.cap) {
      out.bt[(int64_t)o * out.cap + row] = row;
      out.bc[(int64_t)o * out.cap + row] = (fg == INT32_MAX) ? INT64_MIN : (int64_t)fg;
    }
  };
  put_rec(n, s_fg);
  __syncthreads();
  for (int64_t i = n - 1; i >= 0; --i) {
    if (threadIdx.x == 0) s_fg = INT32_MAX;
    __syncthreads();
    const double scale = P.S * exp((double)(n - i) * P.lu);
    int myfg = INT32_MAX;
    for (int64_t j = threadIdx.x; j <= i; j += CTA_THREADS) {
      const double lin = fma(P.wd, a[j], P.wu * a[j + 1]);
      const double grn = fma(scale, u2[j], -P.K);
      if (lin >= grn) {
        b[j] = lin;
      } else {
        b[j] = grn;
        if (myfg == INT32_MAX) myfg = (int)j;
      }
    }
    if (rec) {
      myfg = warp_min_i32(myfg);
      if ((threadIdx.x & 31) == 0 && myfg != INT32_MAX) atomicMin(&s_fg, myfg);
    }
    __syncthreads();
    put_rec(i, s_fg);
    double* t = a;
    a = b;
    b = t;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out.price[o] = a[0];
    out.status[o] = 0;
    if (out.bcount) out.bcount[o] = (int32_t)(n + 1);
  }
}

cudaError_t launch_call_fast(const CallParams* opts, const int32_t* order, int nwork, int32_t* counter, double* ws,
                             int64_t ws_stride, int grid, BatchOut out, cudaStream_t stream) {
  static bool configured = false;
  const int smem = call_fast_smem_bytes();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(call_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (nwork <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  call_fast_kernel<<<grid, CTA_THREADS, smem, stream>>>(opts, order, nwork, counter, ws, ws_stride, out);
  return cudaGetLastError();
}

cudaError_t launch_call_baseline(const CallParams* opts, const int32_t* order, int nwork, double* ws,
                                 int64_t ws_stride, BatchOut out, cudaStream_t stream) {
  if (nwork <= 0) return cudaSuccess;
  call_baseline_kernel<<<nwork, CTA_THREADS, 0, stream>>>(opts, order, nwork, ws, ws_stride, out);
  return cudaGetLastError();
}

}  // namespace fl
