// Microbenchmark: put strip cycles/row while other warps hammer smem (mode 1) or DFMA (mode 2).
#include <cstdio>
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "strip_variants.cuh"
#include "../paper_2303_02317_b200/csrc/fl_conv.cuh"

using namespace fl;
__global__ void __launch_bounds__(288, 1) k(double* in, double* out, double* pay, long long* cyc, int reps, int mode, volatile int* stop) {
  __shared__ double sm[4096];
  extern __shared__ double2 sbuf[];
  const int warp = threadIdx.x >> 5;
  if (warp == 8) {
    long long t0 = clock64();
    int64_t acc = 0;
    for (int r = 0; r < reps; ++r) acc += put_strip_warp<5>(in, out, pay, 0, 129, 64, 32, 0.4, 0.2, 0.39);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) { cyc[0] = t1 - t0; cyc[1] = acc; *stop = 1; }
    return;
  }
  double x = threadIdx.x, y = 1.0;
  int i = threadIdx.x;
  while (!*stop) {
    if (mode == 1) {
      for (int j = 0; j < 64; ++j) { x += sm[(i + 17 * j) & 4095]; sm[(i * 3 + j) & 4095] = x; }
    } else if (mode == 2) {
      for (int j = 0; j < 64; ++j) { x = fma(x, 0.999, y); y = fma(y, 0.999, x); }
    } else if (mode == 4) {
      Grp g{(int)threadIdx.x, 256, 1};
      Stencil st{0.4, 0.2, 0.39, 2};
      x += conv_fft(in, 8192, out + 300, 2048, 1024, st, sbuf, 13, g);
      if (g.t == 0) __threadfence();
    } else if (mode == 5) {
      Grp g{(int)threadIdx.x, 256, 1};
      Stencil st{0.4, 0.2, 0.39, 2};
      for (int q = 0; q < 4; ++q) { x += conv_fft(in, 600, out + 300, 200, 64, st, sbuf, 13, g); if (g.t == 0) __threadfence(); }
    } else if (mode == 6) {
      for (int j = 0; j < 64; ++j) { if ((threadIdx.x & 31) == 0) __threadfence(); x += 1.0; }
    } else if (mode == 7) {
      for (int j = 0; j < 8; ++j) { if ((threadIdx.x & 31) == 0) __nanosleep(20); x += 1.0; }
    } else if (mode == 3) {
      for (int j = 0; j < 64; ++j) { x += __shfl_xor_sync(0xffffffff, x, 1); }
    }
  }
  if (x == 12345.0) out[0] = x + y;
}
int main() {
  double *in, *out, *pay; long long* c; int* stop;
  cudaMalloc(&in, 8 * 16384); cudaMalloc(&out, 8 * 16384); cudaMalloc(&pay, 8 * 256); cudaMalloc(&c, 16); cudaMalloc(&stop, 4);
  cudaMemset(in, 0, 8*16384); cudaMemset(pay, 0, 2048);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int mode = 0; mode < 8; ++mode) {
    cudaMemset(stop, 0, 4);
    k<<<1, 288, 80000>>>(in, out, pay, c, 200, mode, stop);
    long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("mode %d (0 alone, 1 smem, 2 dfma, 3 shfl): %.1f cycles/row (%s)\n", mode, (double)h[0] / (200.0 * 32), cudaGetErrorString(cudaGetLastError()));
  }
}
