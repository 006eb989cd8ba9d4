// Microbenchmark: cycles per conv_fft / conv_direct call for one thread group, alone on an SM.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "fl_conv_instr.cuh"
using namespace fl;
__global__ void __launch_bounds__(256, 1) kb(const double* x, double* y, int64_t L, int64_t Lout, int h, int nthr,
                                             int logN, long long* cyc, int reps, int smem_tw) {
  extern __shared__ double2 sd[];
  double2* tq = sd;
  double2* buf = sd + TWQ;
  for (int i = threadIdx.x; i < TWQ; i += blockDim.x) tq[i] = fl_tw[i];
  __syncthreads();
  if ((int)threadIdx.x >= nthr) return;
  Grp g{(int)threadIdx.x, nthr, nthr == 32 ? -1 : 1};
  Stencil st{0.399, 0.2, 0.4, 2};
  long long ph[5] = {0,0,0,0,0};
  long long t0 = clock64();
  double f = 0;
  for (int r = 0; r < reps; ++r) f += conv_fft(x, L, y, Lout, h, st, buf, logN, smem_tw ? tq : fl_tw, g, ph);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = (long long)f; for (int i = 0; i < 5; ++i) cyc[2+i] = ph[i]; }
}
int main(int argc, char** argv) {
  int only = argc > 1 ? atoi(argv[1]) : -1;
  int reps = argc > 2 ? atoi(argv[2]) : 10;
  std::vector<double2> h(TW_N);
  for (int m = 0; m < TW_N; ++m) { long double a = 6.283185307179586476925286766559L * m / TW_N; h[m] = make_double2((double)cosl(a), -(double)sinl(a)); }
  cudaMemcpyToSymbol(fl_tw, h.data(), sizeof(double2) * TW_N);
  double *x, *y; long long* c;
  cudaMalloc(&x, 8 << 20); cudaMalloc(&y, 8 << 20); cudaMalloc(&c, 64); cudaMemset(x, 0, 8 << 20);
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  struct Case { int nthr, logN; int64_t Lout; int hh; };
  Case cs[] = {{128, 12, 2048, 300}, {128, 12, 1024, 1000}, {128, 11, 1024, 512}, {128, 13, 4096, 2048},
               {128, 13, 16384, 8192}, {256, 13, 4096, 2048}, {256, 13, 16384, 8192}};
  int ci = -1;
  for (auto& k : cs) {
    ++ci; if (only >= 0 && ci != only) continue;
    int64_t L = k.Lout + 2 * k.hh;
    int smem = (TWQ + smem_complex_slots(1 << (k.logN - 1))) * 16;
    for (int tws = 1; tws < 2; ++tws) {
      kb<<<1, 256, smem>>>(x, y, L, k.Lout, k.hh, k.nthr, k.logN, c, 2, tws);
      kb<<<1, 256, smem>>>(x, y, L, k.Lout, k.hh, k.nthr, k.logN, c, reps, tws);
      long long hc[8]; cudaMemcpy(hc, c, 64, cudaMemcpyDeviceToHost);
      printf("   phases load %.0f dif %.0f combine %.0f dit %.0f store %.0f\n", hc[2]/(double)reps, hc[3]/(double)reps, hc[4]/(double)reps, hc[5]/(double)reps, hc[6]/(double)reps);
      printf("nthr %3d logNmax %2d Lout %6lld h %5d tw_%s: %8.0f cycles/call  (%.2f Mflop/call) %s\n", k.nthr, k.logN,
             (long long)k.Lout, k.hh, tws ? "smem" : "gmem", hc[0] / (double)reps, hc[1] / (double)reps / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
