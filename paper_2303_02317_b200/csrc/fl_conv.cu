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
  cudaStreamSynchronize(stream);
}

constexpr int LS_LOGN_MAX = 13;

__global__ void __launch_bounds__(CTA_THREADS)
linear_steps_kernel(const double* __restrict__ x, int64_t L, double* __restrict__ y, int64_t Lout, int h,
                    Stencil st) {
  extern __shared__ double2 sbuf[];
  conv_valid(x, L, y, Lout, h, st, sbuf, LS_LOGN_MAX);
}

int linear_steps_smem_bytes() { return smem_complex_slots(1 << (LS_LOGN_MAX - 1)) * (int)sizeof(double2); }

cudaError_t launch_linear_steps(const double* x, int64_t L, double* y, int64_t Lout, int h, double c0, double c1,
                                double c2, int span, cudaStream_t stream) {
  static bool configured = false;
  const int smem = linear_steps_smem_bytes();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(linear_steps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  Stencil st{c0, c1, c2, span};
  linear_steps_kernel<<<1, CTA_THREADS, smem, stream>>>(x, L, y, Lout, h, st);
  return cudaGetLastError();
}

}  // namespace fl
