// Microbenchmark: cycles per conv_fft call (the FFT groups' task body) for a
// 4-warp group vs a single warp, at the task shapes the medium group serves
// (h = 128 .. 512 jumps of the put recursion just above the subtrees).
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "../paper_2303_02317_b200/csrc/fl_conv.cuh"
using namespace fl;
__global__ void __launch_bounds__(128, 1) kb(const double* x, double* y, int64_t L, int64_t Lout, int h, int nthr,
                                             int logN, long long* cyc, int reps) {
  extern __shared__ double2 sd[];
  double2* tq = sd;
  for (int i = threadIdx.x; i < TWQ; i += blockDim.x) tq[twq_swz(i)] = fl_tw[i];
  __syncthreads();
  const int grp = threadIdx.x / nthr;
  double2* buf = sd + TWQ + grp * smem_complex_slots(1 << (logN - 1));
  Grp g{(int)threadIdx.x % nthr, nthr, nthr == 32 ? -1 : 1};
  Stencil st{0.399, 0.2, 0.401, 2};
  long long t0 = clock64();
  double f = 0;
  for (int r = 0; r < reps; ++r) f += conv_fft(x + grp * (L + 64), L, y + grp * (Lout + 64), Lout, h, st, buf, logN, tq, g);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = (long long)f; }
}
int main() {
  std::vector<double2> hv(TW_N);
  for (int m = 0; m < TW_N; ++m) { long double a = 6.283185307179586476925286766559L * m / TW_N; hv[m] = make_double2((double)cosl(a), -(double)sinl(a)); }
  cudaMemcpyToSymbol(fl_tw, hv.data(), sizeof(double2) * TW_N);
  double *x, *y; long long* c;
  cudaMalloc(&x, 8 << 20); cudaMalloc(&y, 8 << 20); cudaMalloc(&c, 64); cudaMemset(x, 0, 8 << 20);
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 220000);
  struct Case { int64_t Lout; int hh; int logN; };
  Case cs[] = {{256, 128, 10}, {512, 256, 10}, {512, 256, 11}, {768, 256, 11}, {1024, 512, 11}, {1024, 512, 12}, {2048, 512, 12}};
  for (auto& k : cs) {
    const int64_t L = k.Lout + 2 * k.hh;
    for (int nthr : {128, 32}) {
      const int ngrp = 128 / nthr;
      const int smem = (TWQ + ngrp * smem_complex_slots(1 << (k.logN - 1))) * 16;
      if (smem > 220000) continue;
      kb<<<1, 128, smem>>>(x, y, L, k.Lout, k.hh, nthr, k.logN, c, 2);
      kb<<<1, 128, smem>>>(x, y, L, k.Lout, k.hh, nthr, k.logN, c, 20);
      long long hc[2];
      cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
      printf("Lout %5lld h %4d logNmax %2d  %3d threads x %d groups: %7.0f cycles/task (%.0f per task per group-set)  %s\n",
             (long long)k.Lout, k.hh, k.logN, nthr, ngrp, hc[0] / 20.0, hc[0] / 20.0 / ngrp,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
