// fl_common.cuh -- shared device helpers for the fftlattice B200 kernels.
//
// fp64 complex arithmetic, the global twiddle table, status codes and the
// per-option parameter records produced by the host (host_params.h).
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "fl_status.h"

namespace fl {

// ---------------------------------------------------------------------------
// fp64 complex helpers (double2: .x = re, .y = im)

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double cnorm2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// ---------------------------------------------------------------------------
// Twiddle table: fl_tw[m] = exp(-2 pi i m / TW_N), TW_N = largest real block.

constexpr int TW_LOG = 13;
constexpr int TW_N = 1 << TW_LOG;
constexpr int TWQ = TW_N / 4;  // quarter-wave table length (entries 0..TWQ-1 suffice)

// Defined here: the library is one translation unit (csrc/fl_lib.cu).
__device__ double2 fl_tw[TW_N];

__device__ __forceinline__ double2 tw_get(int m) { return __ldg(&fl_tw[m]); }

// W_L^m = exp(-2 pi i m / L) for L a power of two <= TW_N.
__device__ __forceinline__ double2 tw_l(int m, int log_l) { return tw_get(m << (TW_LOG - log_l)); }

// Global quarter-wave copy (kernels without a shared copy).
__device__ double2 fl_twq[TWQ];

// exp(-2 pi i m / TW_N), m in [0, TW_N), from a quarter-wave table
// tq[0..TWQ) (shared memory or fl_twq): W^(m+TWQ) = -i W^m.
__device__ __forceinline__ double2 twq(const double2* tq, int m) {
  // branch-free: lanes of a warp sit in different quadrants
  const double2 b = tq[m & (TWQ - 1)];
  const int q = m >> (TW_LOG - 2);
  const double x = (q & 1) ? b.y : b.x;
  const double y = (q & 1) ? -b.x : b.y;
  const double s = (q & 2) ? -1.0 : 1.0;
  return make_double2(s * x, s * y);
}

// ---------------------------------------------------------------------------
// warp helpers

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int warp_max_i32(int v) { return __reduce_max_sync(FULL, v); }
__device__ __forceinline__ int warp_min_i32(int v) { return __reduce_min_sync(FULL, v); }

// ---------------------------------------------------------------------------
// Kernel attributes (cudaFuncSetAttribute) belong to the current device's
// context: run `set` once per device, tracked in a bit mask (a lost race only
// sets the same attribute twice).
template <class F>
inline cudaError_t once_per_device(std::atomic<unsigned long long>& mask, F&& set) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  const unsigned long long bit = 1ull << dev;
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = set();
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

}  // namespace fl
