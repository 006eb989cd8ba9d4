// Strip latency under co-resident load: warp 0 runs the production leaf strip
// (put_strip_ghost<5>, h = 64) from shared memory while warps 4, 8, 12 (same
// SMSP) run a noise loop of one kind: FP64 FMAs, shared loads, shuffles,
// nanosleep polls, or a long straight-line code block (instruction cache).
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "../paper_2303_02317_b200/csrc/fl_strip.cuh"
#include "strip_variants.cuh"
using namespace fl;
constexpr int NC = 1201, C0 = -600;
constexpr double CD = 0.39790368627109396, CM = 0.199951171875, CU = 0.4020963137289061;

template <int K>
__device__ __noinline__ double bigcode(double x, double a) {
  // ~K x 64 distinct FMAs (straight-line code, no loop inside)
#pragma unroll
  for (int i = 0; i < K * 64; ++i) x = fma(x, a, (double)(i & 7) * 1e-3);
  return x;
}

template <int NOISE, int OTHER>
__global__ void __launch_bounds__(512, 1) k(const double* in, const double* pay, long long* cyc, int reps, int height,
                                           long long f, volatile int* stop) {
  __shared__ double spay[NC], sin_[NC], sout[NC], sn[2048];
  for (int i = threadIdx.x; i < NC; i += blockDim.x) { spay[i] = pay[i]; sin_[i] = in[i]; }
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sn[i] = i;
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    long long t0 = clock64();
    int64_t acc = 0;
    for (int r = 0; r < reps; ++r)
      acc += put_strip_ghost<5, 0>(sin_ - C0, sout - C0, spay - C0, f, height, CD, CM, CU);
    long long t1 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = acc; *stop = 1; }
    return;
  }
  if (NOISE == 0) return;
  if (OTHER == 2 ? w != 4 : OTHER ? !(w == 1 || w == 2 || w == 3) : (w & 3) != 0) return;
  double x = lane, a = 0.999;
  int i = lane;
  while (!*stop) {
    if (NOISE == 1) {
#pragma unroll
      for (int j = 0; j < 64; ++j) x = fma(x, a, 1e-3);
    } else if (NOISE == 2) {
#pragma unroll
      for (int j = 0; j < 16; ++j) { x += sn[(i * 8 + j * 33) & 2047]; i += 5; }
    } else if (NOISE == 3) {
#pragma unroll
      for (int j = 0; j < 16; ++j) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
    } else if (NOISE == 4) {
      __nanosleep(256);
    } else if (NOISE == 6) {
#pragma unroll
      for (int j = 0; j < 16; ++j) { x += sn[(lane + j * 32 + i) & 2047]; i += 64; }
    } else if (NOISE == 7) {
#pragma unroll
      for (int j = 0; j < 16; ++j) { x += sn[((lane * 2) + j * 64 + i) & 2047]; i += 64; }
    } else if (NOISE == 8) {  // a second strip (another chain on the same SMSP)
      put_strip_ghost<5, 0>(sin_ - C0, sout + 0 * NC - C0, spay - C0, f, height, CD, CM, CU);
    } else if (NOISE == 5) {
      x = bigcode<64>(x, a);  // 4096 FMAs of straight-line code (~64 KB)
    }
  }
  if (x == 12345.0) cyc[2] = 1;
}

int main() {
  std::vector<double> pay(NC), a(NC), b(NC);
  const double DS = 0.0069877124296868435;
  for (int i = 0; i < NC; ++i) { pay[i] = 1.0 - exp((double)(C0 + i) * DS); a[i] = pay[i] > 0 ? pay[i] : 0.0; }
  long long f = 0;
  for (int s = 1; s <= 300; ++s) {
    long long lg = -100000;
    for (int i = s; i < NC - s; ++i) {
      double lin = CD * a[i - 1] + CU * a[i + 1] + CM * a[i];
      bool red = lin > pay[i];
      b[i] = red ? lin : pay[i];
      if (!red) lg = C0 + i;
    }
    std::swap(a, b);
    f = lg;
  }
  double *d_in, *d_pay; long long* c; int* stop;
  cudaMalloc(&d_in, 8 * NC); cudaMalloc(&d_pay, 8 * NC); cudaMalloc(&c, 32); cudaMalloc(&stop, 4);
  cudaMemcpy(d_in, a.data(), 8 * NC, cudaMemcpyHostToDevice);
  cudaMemcpy(d_pay, pay.data(), 8 * NC, cudaMemcpyHostToDevice);
  const char* names[] = {"alone", "fp64 fma", "shared loads", "shuffles", "nanosleep polls", "64 KB code", "lds no-conflict", "lds 2-way", "2nd strip"};
  for (int mode = 0; mode < 17; ++mode) {
    const int m = mode < 12 ? mode % 6 : mode < 16 ? 6 + (mode - 12) % 2 : 8;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(stop, 0, 4);
      auto run = [&](int reps) {
        switch (mode) {
          case 0: k<0, 0><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 6: k<0, 1><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 1: k<1, 0><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 7: k<1, 1><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 2: k<2, 0><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 8: k<2, 1><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 3: k<3, 0><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 9: k<3, 1><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 4: k<4, 0><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 10: k<4, 1><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 5: k<5, 0><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 16: k<8, 2><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 12: k<6, 0><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 13: k<7, 0><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 14: k<6, 1><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 15: k<7, 1><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
          case 11: k<5, 1><<<1, 512>>>(d_in, d_pay, c, reps, 64, f, stop); break;
        }
      };
      run(rep == 0 ? 2 : 500);
      cudaDeviceSynchronize();
    }
    long long h[2];
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("%-16s %s strip %.1f cycles/row  (kb %lld) %s\n", names[m], (mode < 6 || mode == 12 || mode == 13) ? "same SMSP  " : "other SMSPs", h[0] / (500.0 * 64), h[1] / 500,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
