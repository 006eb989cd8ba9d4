// fl_put.cu -- American put on the anchored BSM grid: device divide-and-conquer
// (replaces bsm.fast_put_bsm and its recursion, bsm.py:402-713) and the O(T^2)
// projected march (replaces bsm.baseline_put_fd / _accel.put_march_window,
// bsm.py:273-338, _accel.py:163-200).
//
// Fast path: one persistent CTA per option at a time (options pulled from an
// atomic queue in cost order).  The whole halving recursion runs on device with
// an explicit per-thread stack (every thread holds an identical copy; control
// flow is CTA-uniform), so there are no host round-trips:
//   * linear jumps (far / mid / bottom) -> conv_valid (fl_conv.cuh), all warps;
//   * nonlinear leaves (h <= LEAF)      -> put_strip_warp, warp 0;
//   * apex finish (rem <= 2 cutoff)     -> CTA sweep in shared memory.
// Row data live in a per-CTA HBM arena, column-indexed so that concatenations
// in the reference (upper|mid, lower|bottom, near|far) are free.
#include <cstdint>

#include "fl_common.cuh"
#include "fl_conv.cuh"
#include "fl_kernels.h"
#include "fl_strip.cuh"
#include "host_params.h"

namespace fl {

constexpr int PUT_LEAF = 32;                     // device recursion leaf height
constexpr int PUT_CPL = (4 * PUT_LEAF + 2 + 31) / 32;  // cells per lane in a leaf strip
constexpr int PUT_MAX_DEPTH = 24;
constexpr int CONV_LOGN_MAX = 13;                // real FFT block <= 8192
constexpr int CONV_SLOTS = smem_complex_slots(1 << (CONV_LOGN_MAX - 1));

struct PutFrame {
  int64_t f, km;
  double* in_org;
  double* out_org;
  double* asm_org;
  int64_t arena;  // offset of this frame's assembled-row buffer in the frame arena
  int h, state;
};

struct PutLayout {
  int64_t colbase;  // lowest column held in the stage / payoff buffers
  int64_t span;     // buffer length
};

__host__ __device__ inline PutLayout put_layout(int64_t n, int64_t ks) {
  PutLayout L;
  const int64_t lowest = (ks - n < -n ? ks - n : -n);
  L.colbase = lowest - 4 * PUT_LEAF - 16;
  L.span = (ks + n + 8) - L.colbase + 1;
  return L;
}

// doubles needed per CTA for a batch whose options have at most these sizes
int64_t put_ws_doubles(int64_t n_max, int64_t ks_pos_max) {
  const int64_t span = 2 * n_max + ks_pos_max + 4 * PUT_LEAF + 32;
  const int64_t frames = 2 * n_max + 64 * PUT_MAX_DEPTH;
  return 3 * span + frames + 64;
}

__device__ __forceinline__ void cta_bcast_i64(int64_t& v, int64_t* slot) {
  if (threadIdx.x == 0) *slot = v;
  __syncthreads();
  v = *slot;
  __syncthreads();
}

// Apex cone sweep in shared memory (bsm._apex_finish, bsm.py:679-713), restricted
// to the apex dependency cone [ks-rem-1, ks+rem] (identical arithmetic for
// every cell the apex depends on).
__device__ double put_apex(const PutParams& P, const double* cur_org, const double* pay_org, int64_t f,
                           int64_t rem, double* sA, double* sB, int64_t* slot) {
  const int64_t lo = P.ks - rem - 1, hi = P.ks + rem;
  const int W = (int)(hi - lo + 1);
  for (int i = threadIdx.x; i < W; i += CTA_THREADS) {
    const int64_t col = lo + i;
    sA[i] = (col <= f) ? pay_org[col] : cur_org[col];
    sB[i] = sA[i];
  }
  __syncthreads();
  double* a = sA;
  double* b = sB;
  for (int s = 1; s <= rem; ++s) {
    for (int i = s + threadIdx.x; i <= W - 1 - s; i += CTA_THREADS) {
      const double lin = fma(P.cd, a[i - 1], fma(P.cu, a[i + 1], P.cm * a[i]));
      const double pay = pay_org[lo + i];
      b[i] = lin > pay ? lin : pay;
    }
    __syncthreads();
    double* t = a;
    a = b;
    b = t;
  }
  const double r = a[P.ks - lo];
  __syncthreads();
  return r;
}

// _solve_q (bsm.py:443-501) as an explicit-stack loop.  Returns kp or an error
// status through *err.
__device__ int64_t put_solve_q(const PutParams& P, const Stencil& st, int64_t f0, double* in_org,
                               double* out_org, int h0, const double* pay_org, double* frames,
                               double2* sbuf, int64_t* slot, int32_t* err, double* fl) {
  PutFrame stk[PUT_MAX_DEPTH];
  int sp = 0;
  stk[0].f = f0; stk[0].h = h0; stk[0].in_org = in_org; stk[0].out_org = out_org;
  stk[0].arena = 0; stk[0].state = 0;
  sp = 1;
  int64_t ret = 0;
  while (sp > 0) {
    PutFrame& F = stk[sp - 1];
    const int h = F.h;
    if (F.state == 0) {
      if (h <= PUT_LEAF) {
        int64_t kb = 0;
        if (threadIdx.x < 32) {
          kb = put_strip_warp<PUT_CPL>(F.in_org, F.out_org, pay_org, F.f - 2 * h - 1, F.f + 2 * h, F.f, h,
                                       P.cd, P.cm, P.cu);
        }
        cta_bcast_i64(kb, slot);
        *fl += 5.0 * (3.0 * (double)h * h + h);  // cells of a (4h+2)-wide, h-high strip
        if (kb == NONE_SEEN || kb < F.f - h || kb > F.f) { *err = FL_E_GEOMETRY | 1; return 0; }
        ret = kb;
        --sp;
        continue;
      }
      const int h1 = (h + 1) / 2;
      F.asm_org = frames + F.arena - (F.f - h1 + 1);
      // mid: cols f+h1+1 .. f+2h-h1 of row t+h1 from the 2h inputs
      *fl += conv_valid(F.in_org + F.f + 1, 2 * (int64_t)h, F.asm_org + F.f + h1 + 1, 2 * (int64_t)(h - h1), h1, st,
                 sbuf, CONV_LOGN_MAX);
      F.state = 1;
      PutFrame& C = stk[sp];
      C.f = F.f; C.h = h1; C.in_org = F.in_org; C.out_org = F.asm_org;
      C.arena = F.arena + 2 * (int64_t)h + 8; C.state = 0;
      ++sp;
      if (sp >= PUT_MAX_DEPTH) { *err = FL_E_CAPACITY | 1; return 0; }
    } else if (F.state == 1) {
      const int h1 = (h + 1) / 2, h2 = h - h1;
      const int64_t km = ret;
      if (km < F.f - h1 || km > F.f) { *err = FL_E_GEOMETRY | 2; return 0; }
      F.km = km;
      const int64_t A = F.f + 2 * (int64_t)h - h1 - km;  // assembled cols km+1 .. f+2h-h1
      // bottom: cols km+h2+1 .. f+h of row t+h
      *fl += conv_valid(F.asm_org + km + 1, A, F.out_org + km + h2 + 1, A - 2 * (int64_t)h2, h2, st, sbuf,
                 CONV_LOGN_MAX);
      F.state = 2;
      PutFrame& C = stk[sp];
      C.f = km; C.h = h2; C.in_org = F.asm_org; C.out_org = F.out_org;
      C.arena = F.arena + 2 * (int64_t)h + 8; C.state = 0;
      ++sp;
    } else {
      const int h1 = (h + 1) / 2, h2 = h - h1;
      (void)h1;
      const int64_t kp = ret;
      if (kp < F.km - h2 || kp > F.km) { *err = FL_E_GEOMETRY | 3; return 0; }
      --sp;
    }
  }
  return ret;
}

__device__ void put_record(const BatchOut& out, int o, int32_t& cnt, int64_t t, int64_t c) {
  if (threadIdx.x == 0 && out.bt != nullptr && cnt < out.cap) {
    out.bt[(int64_t)o * out.cap + cnt] = t;
    out.bc[(int64_t)o * out.cap + cnt] = c;
  }
  ++cnt;
}

__global__ void __launch_bounds__(CTA_THREADS, 2)
put_fast_kernel(const PutParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork,
                int32_t* counter, double* __restrict__ ws, int64_t ws_stride, BatchOut out) {
  extern __shared__ double2 sbuf[];
  __shared__ int s_work;
  __shared__ int64_t s_slot;
  double* arena = ws + (int64_t)blockIdx.x * ws_stride;
  for (;;) {
    if (threadIdx.x == 0) s_work = atomicAdd(counter, 1);
    __syncthreads();
    const int w = s_work;
    __syncthreads();
    if (w >= nwork) break;
    const int o = order[w];
    const PutParams P = opts[o];
    const int64_t n = P.n, ks = P.ks;
    const PutLayout Lo = put_layout(n, ks);
    double* bufA = arena;
    double* bufB = arena + Lo.span;
    double* pay = arena + 2 * Lo.span;
    double* frames = arena + 3 * Lo.span;
    double* pay_org = pay - Lo.colbase;
    double* cur_org = bufA - Lo.colbase;
    double* nxt_org = bufB - Lo.colbase;
    // payoff table 1 - e^{col ds} (bsm.py:238-244) and the initial row: zeros on 1..ks+n
    for (int64_t i = threadIdx.x; i < Lo.span; i += CTA_THREADS) {
      const int64_t col = Lo.colbase + i;
      pay[i] = 1.0 - exp((double)col * P.ds);
      bufA[i] = 0.0;
    }
    __syncthreads();
    const Stencil st{P.cd, P.cm, P.cu, 2};
    int32_t err = 0, cnt = 0;
    int64_t m = 0, f = 0;
    double price = 0.0, flops = 0.0;
    put_record(out, o, cnt, 0, 0);
    for (;;) {
      const int64_t rem = n - m;
      const int64_t red = ks + rem - f;
      if (red < 0) { err = FL_E_GEOMETRY | 4; break; }
      if (red == 0) { price = P.K * (1.0 - exp((double)ks * P.ds)); break; }
      if (rem <= 2 * (int64_t)P.cutoff) {
        if (2 * rem + 2 > CONV_SLOTS) { err = FL_E_CAPACITY | 2; break; }
        price = P.K * put_apex(P, cur_org, pay_org, f, rem, (double*)sbuf, ((double*)sbuf) + CONV_SLOTS, &s_slot);
        flops += 5.0 * ((double)rem * rem + rem);
        break;
      }
      const int64_t hh = (rem / 2 < red / 2) ? rem / 2 : red / 2;
      if (hh < 1) {
        int64_t kb = 0;
        if (threadIdx.x < 32)
          kb = put_strip_warp<PUT_CPL>(cur_org, nxt_org, pay_org, f - 3, f + 1, f, 1, P.cd, P.cm, P.cu);
        cta_bcast_i64(kb, &s_slot);
        flops += 15.0;
        if (kb == NONE_SEEN || kb < f - 1 || kb > f) { err = FL_E_GEOMETRY | 5; break; }
        f = kb;
        m += 1;
      } else {
        const int h = (int)hh;
        if (red > 2 * hh)  // far: cols f+h+1 .. ks+rem-h stay linear
          flops += conv_valid(cur_org + f + 1, red, nxt_org + f + h + 1, red - 2 * hh, h, st, sbuf, CONV_LOGN_MAX);
        const int64_t kp =
            put_solve_q(P, st, f, cur_org, nxt_org, h, pay_org, frames, sbuf, &s_slot, &err, &flops);
        if (err) break;
        f = kp;
        m += hh;
      }
      put_record(out, o, cnt, m, f);
      double* t = cur_org;
      cur_org = nxt_org;
      nxt_org = t;
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
// O(T^2) projected march over the shrinking window (baseline_put_fd).

__global__ void __launch_bounds__(CTA_THREADS)
put_baseline_kernel(const PutParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork,
                    double* __restrict__ ws, int64_t ws_stride, BatchOut out) {
  __shared__ int s_red[CTA_THREADS / 32];
  const int w = blockIdx.x;
  if (w >= nwork) return;
  const int o = order[w];
  const PutParams P = opts[o];
  const int64_t n = P.n;
  const int64_t W = 2 * n + 1;
  const int64_t lo = P.ks - n;
  double* a = ws + (int64_t)blockIdx.x * ws_stride;
  double* b = a + W;
  double* pay = b + W;
  for (int64_t k = threadIdx.x; k < W; k += CTA_THREADS) {
    const double p = 1.0 - exp((double)(lo + k) * P.ds);
    pay[k] = p;
    a[k] = p > 0.0 ? p : 0.0;
    b[k] = a[k];
  }
  __syncthreads();
  const bool rec = out.bt != nullptr;
  if (rec && threadIdx.x == 0 && out.cap > 0) {
    out.bt[(int64_t)o * out.cap] = 0;
    out.bc[(int64_t)o * out.cap] = (P.ks + n < 0) ? P.ks + n : 0;
  }
  for (int64_t s = 1; s <= n; ++s) {
    int lg = -1;
    for (int64_t k = s + threadIdx.x; k <= W - 1 - s; k += CTA_THREADS) {
      const double lin = fma(P.cd, a[k - 1], fma(P.cu, a[k + 1], P.cm * a[k]));
      const double p = pay[k];
      const bool red = lin > p;
      b[k] = red ? lin : p;
      if (!red) lg = (int)k;
    }
    if (rec) {
      lg = warp_max_i32(lg);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = lg;
    }
    __syncthreads();
    if (rec && threadIdx.x == 0 && s < out.cap) {
      int m = -1;
      for (int i = 0; i < CTA_THREADS / 32; ++i) m = s_red[i] > m ? s_red[i] : m;
      out.bt[(int64_t)o * out.cap + s] = s;
      out.bc[(int64_t)o * out.cap + s] = (m < 0) ? INT64_MIN : lo + m;
    }
    double* t = a;
    a = b;
    b = t;
  }
  if (threadIdx.x == 0) {
    out.price[o] = P.K * a[n];
    out.status[o] = 0;
    if (out.bcount) out.bcount[o] = (int32_t)(n + 1);
  }
}

// ---------------------------------------------------------------------------
// launchers

int put_fast_smem_bytes() { return CONV_SLOTS * (int)sizeof(double2); }

cudaError_t launch_put_fast(const PutParams* opts, const int32_t* order, int nwork, int32_t* counter, double* ws,
                            int64_t ws_stride, int grid, BatchOut out, cudaStream_t stream) {
  static bool configured = false;
  const int smem = put_fast_smem_bytes();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(put_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (nwork <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  put_fast_kernel<<<grid, CTA_THREADS, smem, stream>>>(opts, order, nwork, counter, ws, ws_stride, out);
  return cudaGetLastError();
}

cudaError_t launch_put_baseline(const PutParams* opts, const int32_t* order, int nwork, double* ws,
                                int64_t ws_stride, BatchOut out, cudaStream_t stream) {
  if (nwork <= 0) return cudaSuccess;
  put_baseline_kernel<<<nwork, CTA_THREADS, 0, stream>>>(opts, order, nwork, ws, ws_stride, out);
  return cudaGetLastError();
}

}  // namespace fl
