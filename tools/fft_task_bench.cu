// conv_fft task latency (the FFT groups' task body) at the shapes the put
// recursion issues: two 4-warp groups per CTA (named barriers 1, 2, as in the
// kernel), each running its own stream of tasks; cycles per task per group and
// the outputs' max deviation from a direct fp64 correlation (sanity).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/fft_task_bench tools/fft_task_bench.cu
#include <cmath>
#include <cstdio>
#include <vector>

// phase timing: per group (g.bar), cycles from the previous mark; marks 4 (block
// start), 0 (loaded), 1 (forward), 2 (spectrum), 3 (inverse), 5 (stored)
__device__ long long fl_tlast[4];
__device__ long long fl_tacc[4][8];
#define FL_FFT_T(k)                                                    \
  if (g.t == 0) {                                                      \
    const long long _t = clock64();                                    \
    if ((k) != 4) fl_tacc[g.bar & 3][k] += _t - fl_tlast[g.bar & 3];   \
    fl_tlast[g.bar & 3] = _t;                                          \
  }
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "../paper_2303_02317_b200/csrc/fl_conv.cuh"
using namespace fl;

constexpr double CD = 0.39790368627109396, CM = 0.199951171875, CU = 0.4020963137289061;

__global__ void __launch_bounds__(256, 1) kt(const double* x, double* y, int64_t L, int64_t Lout, int h, int logN,
                                             int ngrp, int reps, long long* cyc, int gsz = 128) {
  extern __shared__ double2 sd[];
  double2* tq = sd;
  for (int i = threadIdx.x; i < TWQ; i += blockDim.x) tq[i] = fl_tw[i];
  __syncthreads();
  const int grp = threadIdx.x / gsz;
  if (grp >= ngrp) return;
  double2* buf = sd + TWQ + grp * smem_complex_slots(1 << (logN - 1));
  const Grp g{(int)(threadIdx.x % gsz), gsz, gsz == 32 ? -1 : 1 + grp};
  const Stencil st{CD, CM, CU, 2};
  const double* xg = x + grp * (L + 64);
  double* yg = y + grp * (Lout + 64);
  gsync(g);
  const long long t0 = clock64();
  double f = 0.0;
  for (int r = 0; r < reps; ++r) f += conv_fft(xg, L, yg, Lout, h, st, buf, logN, tq, g);
  const long long t1 = clock64();
  if (g.t == 0) { cyc[2 * grp] = t1 - t0; cyc[2 * grp + 1] = (long long)f; }
}

// composed weights W_h (P(z) = CD + CM z + CU z^2) by repeated convolution (host, long double)
static std::vector<double> weights(int h) {
  std::vector<long double> w(1, 1.0L);
  for (int s = 0; s < h; ++s) {
    std::vector<long double> n(w.size() + 2, 0.0L);
    for (size_t i = 0; i < w.size(); ++i) {
      n[i] += w[i] * CD;
      n[i + 1] += w[i] * CM;
      n[i + 2] += w[i] * CU;
    }
    w.swap(n);
  }
  return std::vector<double>(w.begin(), w.end());
}

int main() {
  std::vector<double2> hv(TW_N);
  for (int m = 0; m < TW_N; ++m) {
    const long double a = 6.283185307179586476925286766559L * m / TW_N;
    hv[m] = make_double2((double)cosl(a), -(double)sinl(a));
  }
  cudaMemcpyToSymbol(fl_tw, hv.data(), sizeof(double2) * TW_N);
  struct Case { int64_t Lout; int h; int logN; };
  const Case cs[] = {{512, 256, 12}, {1024, 512, 12}, {1024, 512, 11}, {2048, 1024, 13}, {4096, 2048, 13}, {8192, 4096, 13}};
  double *x, *y;
  long long* c;
  const int64_t XN = 1 << 16;
  cudaMalloc(&x, 8 * XN); cudaMalloc(&y, 8 * XN); cudaMalloc(&c, 256);
  std::vector<double> hx(XN);
  for (int64_t i = 0; i < XN; ++i) hx[i] = 1.0 + 0.5 * sin(0.01 * (double)i) + 1e-3 * (double)(i % 7);
  cudaMemcpy(x, hx.data(), 8 * XN, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (const Case& k : cs) {
    const int64_t L = k.Lout + 2 * k.h;
    struct Cfg { int gsz, ngrp; };
    const Cfg cf[] = {{128, 1}, {128, 2}, {64, 1}, {64, 2}, {64, 4}};
    for (const Cfg& q : cf) {
      if (q.gsz == 64 && k.logN > 12) continue;
      const int smem = (TWQ + q.ngrp * smem_complex_slots(1 << (k.logN - 1))) * 16;
      if (smem > 227 * 1024) continue;
      kt<<<1, 256, smem>>>(x, y, L, k.Lout, k.h, k.logN, q.ngrp, 2, c, q.gsz);
      kt<<<1, 256, smem>>>(x, y, L, k.Lout, k.h, k.logN, q.ngrp, 20, c, q.gsz);
      long long hc[16];
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hc, c, 8 * 2 * q.ngrp, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < q.ngrp; ++i) mx = fmax(mx, (double)hc[2 * i]);
      printf("Lout %5lld h %5d logNmax %2d  %3d thr x %d grp: %8.0f cycles/task, %8.0f cycles per task per SM-set  %s\n",
             (long long)k.Lout, k.h, k.logN, q.gsz, q.ngrp, mx / 20.0, mx / 20.0 / q.ngrp, cudaGetErrorString(e));
      if (q.gsz == 128 && q.ngrp == 1) {  // sanity: against a direct long-double correlation
        std::vector<double> hy(k.Lout);
        cudaMemcpy(hy.data(), y, 8 * k.Lout, cudaMemcpyDeviceToHost);
        const std::vector<double> w = weights(k.h);
        double dev = 0.0;
        for (int64_t o = 0; o < k.Lout; o += 37) {
          long double a = 0.0L;
          for (size_t r = 0; r < w.size(); ++r) a += (long double)w[r] * hx[o + r];
          dev = fmax(dev, fabs((double)a - hy[o]));
        }
        printf("      max |y - direct| = %.3g\n", dev);
      }
      long long ta[4][8];
      cudaMemcpyFromSymbol(ta, fl_tacc, sizeof(ta));
      cudaMemset(c, 0, 8);
      const long long zero[32] = {0};
      cudaMemcpyToSymbol(fl_tacc, zero, sizeof(zero));
      const double nt = 22.0;  // tasks timed (2 + 20 reps)
      printf("      group 1 per task: load %6.0f  forward %6.0f  spectrum %6.0f  inverse %6.0f  store %6.0f\n",
             ta[1][0] / nt, ta[1][1] / nt, ta[1][2] / nt, ta[1][3] / nt, ta[1][5] / nt);
    }
  }
  return 0;
}
