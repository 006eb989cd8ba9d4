// fl_conv.cu -- twiddle table and the standalone batched correlation entry
// (apply_linear_steps on device; fft.py:263-329).
#include <cmath>
#include <vector>

#include "fl_common.cuh"
#include "fl_conv.cuh"
#include "fl_kernels.h"

namespace fl {

void init_twiddles(cudaStream_t stream) {
  std::vector<double2> h(TW_N);
  const long double two_pi = 6.283185307179586476925286766559L;
  for (int m = 0; m < TW_N; ++m) {
    const long double a = two_pi * (long double)m / (long double)TW_N;
    h[m] = make_double2((double)cosl(a), (double)(-sinl(a)));
  }
  cudaMemcpyToSymbolAsync(fl_tw, h.data(), sizeof(double2) * TW_N, 0, cudaMemcpyHostToDevice, stream);
  std::vector<double2> q(TWQ);
  for (int i = 0; i < TWQ; ++i) q[i] = h[i];
  cudaMemcpyToSymbolAsync(fl_twq, q.data(), sizeof(double2) * TWQ, 0, cudaMemcpyHostToDevice, stream);
  cudaStreamSynchronize(stream);
}

constexpr int LS_LOGN_MAX = 13;

// FP64 DFMA throughput probe (8 independent chains per thread, 2 CTAs x 1024
// threads per SM); used by bench.py for the live roofline denominator.
__global__ void __launch_bounds__(1024) fp64_probe_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

cudaError_t probe_fp64(double* tflops, cudaStream_t stream) {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = 2 * nsm, block = 1024, iters = 2048;
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(double) * grid * block);
  if (e != cudaSuccess) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fp64_probe_kernel<<<grid, block, 0, stream>>>(d, 64, 0.999, 1e-3);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, stream);
    fp64_probe_kernel<<<grid, block, 0, stream>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1, stream);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  e = cudaGetLastError();
  *tflops = 2.0 * 8 * 16 * (double)iters * grid * block / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return e;
}

// Short jumps (h <= LS_DIRECT_H) go through the composed weights directly:
// W_h by h - 1 real-space convolutions with the stencil in shared memory (all
// terms nonnegative), then y[k] = sum_r W_h[r] x[k + r] -- as the pricers'
// subtree correlations do, so a run of exact zeros stays exactly zero (the
// windowed FFT leaves round-off of order 1e-16 max|x| there).  Longer jumps:
// the truncated overlap-save FFT with the analytic spectrum (conv_fft).
constexpr int LS_DIRECT_H = 64;

// fp64 exp / log throughput probes (8 independent chains per thread): the
// European path is transcendental-bound; its roofline counts
// each exp / log at its measured DFMA-equivalent cost.
__global__ void __launch_bounds__(1024) exp_probe_kernel(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 0.1 + 1e-3 * k + threadIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = exp(-x[k]);  // converges to the fixed point 0.567
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(1024) log_probe_kernel(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 3.0 + 1e-3 * k + threadIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = log(x[k]) + 2.5;  // fixed point near 3.5
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

cudaError_t probe_transcendentals(double* exp_per_s, double* log_per_s, cudaStream_t stream) {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = 2 * nsm, block = 1024, iters = 256;
  double* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(double) * grid * block);
  if (e != cudaSuccess) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int which = 0; which < 2; ++which) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0, stream);
      if (which == 0) exp_probe_kernel<<<grid, block, 0, stream>>>(d, rep == 0 ? 8 : iters);
      else log_probe_kernel<<<grid, block, 0, stream>>>(d, rep == 0 ? 8 : iters);
      cudaEventRecord(e1, stream);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0) best = ms < best ? ms : best;
    }
    const double evals = 8.0 * iters * (double)grid * block;
    (which == 0 ? *exp_per_s : *log_per_s) = evals / (best * 1e-3);
  }
  e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return e;
}

__global__ void __launch_bounds__(CTA_THREADS)
linear_steps_kernel(const double* __restrict__ x, int64_t L, double* __restrict__ y, int64_t Lout, int h,
                    Stencil st) {
  extern __shared__ double2 sbuf[];
  if (h <= LS_DIRECT_H) {
    double* w = reinterpret_cast<double*>(sbuf);
    double* t = w + (2 * LS_DIRECT_H + 2);
    const int M = h * st.span + 1;
    const double s[3] = {st.c0, st.c1, st.c2};
    for (int r = threadIdx.x; r < M; r += CTA_THREADS) w[r] = (r <= st.span) ? s[r] : 0.0;
    __syncthreads();
    for (int m = 2; m <= h; ++m) {  // W_m = W_{m-1} (*) stencil, lengths (m-1) span + 1 -> m span + 1
      const int len = m * st.span + 1;
      for (int r = threadIdx.x; r < len; r += CTA_THREADS) {
        double acc = 0.0;
        for (int j = 0; j <= st.span; ++j) {
          const int q = r - j;
          if (q >= 0 && q <= (m - 1) * st.span) acc = fma(w[q], s[j], acc);
        }
        t[r] = acc;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < len; r += CTA_THREADS) w[r] = t[r];
      __syncthreads();
    }
    for (int64_t k = threadIdx.x; k < Lout; k += CTA_THREADS) {
      double acc = 0.0;
      for (int r = 0; r < M; ++r) acc = fma(w[r], x[k + r], acc);
      y[k] = acc;
    }
    return;
  }
  conv_fft(x, L, y, Lout, h, st, sbuf, LS_LOGN_MAX, fl_twq, Grp{(int)threadIdx.x, CTA_THREADS, 0});
}

int linear_steps_smem_bytes() { return smem_complex_slots(1 << (LS_LOGN_MAX - 1)) * (int)sizeof(double2); }

cudaError_t launch_linear_steps(const double* x, int64_t L, double* y, int64_t Lout, int h, double c0, double c1,
                                double c2, int span, cudaStream_t stream) {
  static std::atomic<unsigned long long> configured{0};
  const int smem = linear_steps_smem_bytes();
  {
    cudaError_t e = once_per_device(configured, [&] {
      return cudaFuncSetAttribute(linear_steps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    });
    if (e != cudaSuccess) return e;
  }
  Stencil st{c0, c1, c2, span};
  linear_steps_kernel<<<1, CTA_THREADS, smem, stream>>>(x, L, y, Lout, h, st);
  return cudaGetLastError();
}

}  // namespace fl
