// fl_euro.cu -- binomial European call: O(T) fast price (replaces
// binomial.fast_european, binomial.py:161-194) and the O(T^2) backward
// induction (replaces binomial.baseline_european / _accel.european_backward,
// binomial.py:80-91, _accel.py:49-59).
//
// Fast path: price = sum_r W_r * leaf_r with the gauged composed weights
// W_r = C(T,r) a^(T-r) b^r, a = wd, b = wu e^{2 lu} (binomial.py:166-194).  The
// reference builds W from an x87 long-double log-ratio cumsum (fft.py:166-200);
// on device each weight is evaluated independently and in parallel with
// Loader's saddle-point form of the binomial law,
//     W_r = (a+b)^T * dbinom(r; T, b/(a+b)),
//     log dbinom = stirlerr(T) - stirlerr(r) - stirlerr(T-r)
//                  - bd0(r, Tp) - bd0(T-r, Tq) - log(2 pi r (T-r)/T)/2,
// (C. Loader, "Fast and accurate computation of binomial probabilities",
// 2000), accurate to a few ulp in fp64 with no extended precision -- tighter
// than a plain lgamma form, whose cancellation costs ~1e-10 relative at
// T=2^16.  The dot product is a fixed-order CTA tree reduction (deterministic).
#include <cstdint>

#include "fl_common.cuh"
#include "fl_kernels.h"
#include "host_params.h"

namespace fl {

// stirlerr(n) = lgamma(n+1) - (n+1/2) log n + n - log(2 pi)/2, n = 0..15
// (computed in extended precision; the usual published table).
__constant__ double c_stirl[16] = {
    0.0,
    0.081061466795327258197,
    0.041340695955409294054,
    0.027677925684998339387,
    0.020790672103765092877,
    0.016644691189821192434,
    0.013876128823070748165,
    0.011896709945891770124,
    0.010411265261972095064,
    0.0092554621827127343185,
    0.0083305634333628722564,
    0.0075736754879518429213,
    0.0069428401072095287795,
    0.0064089941880042077395,
    0.0059513701127588489593,
    0.0055547335519627999141,
};

__device__ __forceinline__ double stirlerr(double n) {
  constexpr double S0 = 1.0 / 12.0, S1 = 1.0 / 360.0, S2 = 1.0 / 1260.0, S3 = 1.0 / 1680.0, S4 = 1.0 / 1188.0;
  if (n <= 15.0) return c_stirl[(int)n];
  const double nn = n * n;
  if (n > 500.0) return (S0 - S1 / nn) / n;
  if (n > 80.0) return (S0 - (S1 - S2 / nn) / nn) / n;
  if (n > 35.0) return (S0 - (S1 - (S2 - S3 / nn) / nn) / nn) / n;
  return (S0 - (S1 - (S2 - (S3 - S4 / nn) / nn) / nn) / nn) / n;
}

// deviance term x log(x/np) + np - x, computed without cancellation
__device__ __forceinline__ double bd0(double x, double np) {
  if (fabs(x - np) < 0.1 * (x + np)) {
    double v = (x - np) / (x + np);
    double s = (x - np) * v;
    double ej = 2.0 * x * v;
    const double v2 = v * v;
    for (int j = 1; j < 1000; ++j) {
      ej *= v2;
      const double s1 = s + ej / (double)(2 * j + 1);
      if (s1 == s) return s1;
      s = s1;
    }
    return s;
  }
  return x * log(x / np) + np - x;
}

// log of W_r = (a+b)^T dbinom(r; T, p), p = b/(a+b), q = a/(a+b)
__device__ __forceinline__ double log_weight(int64_t r, int64_t T, double p, double q, double logsum_T) {
  const double n = (double)T, x = (double)r;
  double lc;
  if (r == 0) {
    lc = (p < 0.1) ? -bd0(n, n * q) - n * p : n * log(q);
    return lc + logsum_T;
  }
  if (r == T) {
    lc = (q < 0.1) ? -bd0(n, n * p) - n * q : n * log(p);
    return lc + logsum_T;
  }
  lc = stirlerr(n) - stirlerr(x) - stirlerr(n - x) - bd0(x, n * p) - bd0(n - x, n * q);
  const double lf = 1.8378770664093454836 + log(x) + log1p(-x / n);  // log(2 pi x (n-x)/n)
  return lc - 0.5 * lf + logsum_T;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  // fixed-order tree: warp shuffle tree, then warp partials in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NT / 32; ++i) s += red[i];
  }
  __syncthreads();
  return s;
}

constexpr int EURO_THREADS = 256;

__global__ void __launch_bounds__(EURO_THREADS)
euro_fast_kernel(const EuroParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork, BatchOut out) {
  __shared__ double red[EURO_THREADS / 32];
  apply_dlist(out, order, nwork);
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
  const int o = order[w];
  const EuroParams E = opts[o];
  const int64_t T = E.n;
  const double sum = E.wd + E.bg;
  const double p = E.bg / sum, q = E.wd / sum;
  const double logsum_T = (double)T * log(sum);
  const double x0 = E.S * exp(-(double)T * E.lu);  // spot * u^-T (binomial.py:188-193)
  // first in-the-money leaf: x0 - K e^{-2 r lu} > 0  <=>  r > log(K/x0) / (2 lu)
  int64_t r0 = 0;
  if (E.K > 0.0) {
    const double t = log(E.K / x0) / (2.0 * E.lu);
    r0 = (t < 0.0) ? 0 : (int64_t)floor(t) - 1;
    if (r0 < 0) r0 = 0;
    if (r0 > T) r0 = T + 1;
  }
  double acc = 0.0;
  for (int64_t r = r0 + threadIdx.x; r <= T; r += EURO_THREADS) {
    double leaf = x0 - E.K * exp(-2.0 * (double)r * E.lu);
    if (leaf > 0.0) acc = fma(exp(log_weight(r, T, p, q, logsum_T)), leaf, acc);
  }
  const double s = block_sum<EURO_THREADS>(acc, red);
  if (threadIdx.x == 0) {
    out.price[o] = s;
    out.status[o] = 0;
    if (out.bcount) out.bcount[o] = 0;
  }
  __syncthreads();
  }
}

// O(T^2) backward induction of the leaf row (european_backward), one CTA per option.
__global__ void __launch_bounds__(EURO_THREADS)
euro_baseline_kernel(const EuroParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork, double* __restrict__ ws, int64_t ws_stride,
                     BatchOut out) {
  apply_dlist(out, order, nwork);
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
  const int o = order[w];
  const EuroParams E = opts[o];
  const double wd = E.wd, wu = E.wu;
  const int64_t n = E.n;
  double* a = ws + (int64_t)blockIdx.x * ws_stride;
  double* b = a + n + 1;
  for (int64_t j = threadIdx.x; j <= n; j += EURO_THREADS) {
    const double v = E.S * exp((2.0 * (double)j - (double)n) * E.lu) - E.K;  // leaf_row (binomial.py:64-77)
    a[j] = v > 0.0 ? v : 0.0;
  }
  __syncthreads();
  for (int64_t i = n; i > 0; --i) {
    for (int64_t j = threadIdx.x; j < i; j += EURO_THREADS) b[j] = fma(wd, a[j], wu * a[j + 1]);
    __syncthreads();
    double* t = a;
    a = b;
    b = t;
  }
  if (threadIdx.x == 0) {
    out.price[o] = a[0];
    out.status[o] = 0;
    if (out.bcount) out.bcount[o] = 0;
  }
  __syncthreads();
  }
}

cudaError_t launch_euro_fast(const EuroParams* opts, const int32_t* order, int nwork, int grid, BatchOut out,
                             cudaStream_t stream) {
  if (nwork <= 0 || grid <= 0) return cudaSuccess;
  euro_fast_kernel<<<grid, EURO_THREADS, 0, stream>>>(opts, order, nwork, out);
  return cudaGetLastError();
}

cudaError_t launch_euro_baseline(const EuroParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                                 double* ws, int64_t ws_stride, BatchOut out, cudaStream_t stream) {
  if (nwork <= 0 || grid <= 0) return cudaSuccess;
  if (n_max + 1 <= sweep_max_cells() && !sweep_disabled()) return launch_euro_sweep(opts, order, nwork, n_max, grid, out, stream);
  euro_baseline_kernel<<<grid, EURO_THREADS, 0, stream>>>(opts, order, nwork, ws, ws_stride, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Normal-limit approximations (binomial.py:197-296).  One CTA per option for
// the Gaussian window sum (fixed-order tree reduction), one thread per option
// for the closed form.

__global__ void __launch_bounds__(CTA_THREADS)
euro_gauss_kernel(const EuroApprox* __restrict__ opts, int n_opts, double* __restrict__ price) {
  __shared__ double red[CTA_THREADS];
  const int o = blockIdx.x;
  if (o >= n_opts) return;
  const EuroApprox A = opts[o];
  double acc = 0.0;
  const double norm = sqrt(2.0 * 3.141592653589793 * A.sigma);
  for (int64_t x = A.lo + threadIdx.x; x <= A.hi; x += CTA_THREADS) {
    const double xd = (double)x;
    const double dens = exp(-((xd + A.mu) * (xd + A.mu)) / (2.0 * A.sigma)) / norm;
    double leaf = A.S * exp((2.0 * xd - (double)A.n) * A.lu) - A.K;
    leaf = leaf > 0.0 ? leaf : 0.0;
    acc = fma(dens, leaf, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = CTA_THREADS / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) price[o] = A.disc * red[0];
}

__global__ void euro_closed_kernel(const EuroApprox* __restrict__ opts, int n_opts, double* __restrict__ price) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_opts) return;
  const EuroApprox A = opts[o];
  if (A.x0 > A.n) { price[o] = 0.0; return; }
  const double root = sqrt(2.0 * A.sigma);
  const double n = (double)A.n, x0 = (double)A.x0;
  const double bn = (n + A.mu) / root, bx = (x0 + A.mu) / root;
  const double an = bn - A.lu * root, ax = bx - A.lu * root;
  const double spot_leg = A.S * exp(A.lu * (2.0 * A.sigma * A.lu - 2.0 * A.mu - n)) * (erf(an) - erf(ax));
  const double strike_leg = A.K * (erf(bn) - erf(bx));
  price[o] = 0.5 * A.disc * (spot_leg - strike_leg);
}

cudaError_t launch_euro_approx(const EuroApprox* opts, int n_opts, int method, double* price, cudaStream_t stream) {
  if (n_opts <= 0) return cudaSuccess;
  if (method == 2) euro_gauss_kernel<<<n_opts, CTA_THREADS, 0, stream>>>(opts, n_opts, price);
  else euro_closed_kernel<<<(n_opts + 127) / 128, 128, 0, stream>>>(opts, n_opts, price);
  return cudaGetLastError();
}

}  // namespace fl
