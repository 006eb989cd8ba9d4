// Microbenchmark + equivalence check: warp put strip, plain vs time-tiled.
#include <cstdio>
#include <cmath>
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "strip_variants.cuh"
using namespace fl;
template <int MODE>
__global__ void k(double* in, double* out, double* pay, long long* cyc, int reps, int height) {
  int64_t lo = 0, hi = 129, f = 64;
  long long t0 = clock64();
  int64_t acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (MODE == 0) acc += put_strip_warp<5>(in, out, pay, lo, hi, f, height, 0.4, 0.2, 0.39);
    if (MODE == 2) acc += put_strip_tiled<5, 2>(in, out, pay, lo, hi, f, height, 0.4, 0.2, 0.39);
    if (MODE == 3) acc += put_strip_tiled<5, 3>(in, out, pay, lo, hi, f, height, 0.4, 0.2, 0.39);
    if (MODE == 4) acc += put_strip_tiled<5, 4>(in, out, pay, lo, hi, f, height, 0.4, 0.2, 0.39);
    if (MODE == 5) acc += put_strip_v2<4>(in, out, pay, hi, f, height, 0.4, 0.2, 0.39);
    if (MODE == 6) acc += put_strip_pipe<5>(in, out, pay, lo, hi, f, height, 0.4, 0.2, 0.39);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = acc; }
}
int main() {
  double *in, *out, *pay; long long* c;
  cudaMalloc(&in, 8 * 256); cudaMalloc(&out, 8 * 256); cudaMalloc(&pay, 8 * 256); cudaMalloc(&c, 16);
  double h_in[256], h_pay[256];
  for (int i = 0; i < 256; ++i) { h_pay[i] = 1.0 - exp((i - 64) * 0.01); h_in[i] = (i > 64) ? 0.05 * exp(-(i - 64) * 0.03) + (h_pay[i] > 0 ? h_pay[i] : 0) : h_pay[i]; }
  cudaMemcpy(in, h_in, 2048, cudaMemcpyHostToDevice); cudaMemcpy(pay, h_pay, 2048, cudaMemcpyHostToDevice);
  double ref[256];
  long long h[2];
  for (int height : {32, 31, 17}) {
    for (int mode : {0, 6, 5}) {
      cudaMemset(out, 0, 2048);
      auto run = [&](int reps) {
        if (mode == 0) k<0><<<1, 32>>>(in, out, pay, c, reps, height);
        if (mode == 2) k<2><<<1, 32>>>(in, out, pay, c, reps, height);
        if (mode == 3) k<3><<<1, 32>>>(in, out, pay, c, reps, height);
        if (mode == 4) k<4><<<1, 32>>>(in, out, pay, c, reps, height);
        if (mode == 5) k<5><<<1, 32>>>(in, out, pay, c, reps, height);
        if (mode == 6) k<6><<<1, 32>>>(in, out, pay, c, reps, height);
      };
      run(1);
      double o[256]; cudaMemcpy(o, out, 2048, cudaMemcpyDeviceToHost);
      cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
      long long kb = h[1];
      if (mode == 0) for (int i = 0; i < 256; ++i) ref[i] = o[i];
      int diff = 0; for (int i = 0; i < 256; ++i) diff += (o[i] != ref[i]);
      run(1000);
      cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
      printf("height %d mode %d: %.1f cycles/row  kb %lld  diffs vs plain %d  (%s)\n", height, mode,
             (double)h[0] / (1000.0 * height), kb, diff, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
