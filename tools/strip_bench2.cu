// Microbenchmark + equivalence check of the put leaf strip: put_strip_warp
// (full 4h+2 frame) vs put_strip_v2 (3h+2 frame, peeled green mask), on a
// realistic row produced by marching the projected put stencil from the payoff.
#include <cmath>
#include <cstdio>
#include <vector>

#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "strip_variants.cuh"
using namespace fl;

constexpr int NC = 1201, C0 = -600;  // columns C0 .. C0+NC-1
constexpr double CD = 0.39790368627109396, CM = 0.199951171875, CU = 0.4020963137289061, DS = 0.0069877124296868435;

template <int MODE>
__global__ void k(const double* in, double* out, const double* pay, long long* cyc, int reps, int height, long long f,
                  long long hi) {
  const double* in_org = in - C0;
  double* out_org = out - C0;
  const double* pay_org = pay - C0;
  long long t0 = clock64();
  int64_t acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (MODE == 0) acc += put_strip_warp<5>(in_org, out_org, pay_org, f - 2 * height - 1, hi, f, height, CD, CM, CU);
    if (MODE == 1) acc += put_strip_v2<4>(in_org, out_org, pay_org, hi, f, height, CD, CM, CU);
    if (MODE == 2) acc += put_strip_v2<3>(in_org, out_org, pay_org, hi, f, height, CD, CM, CU);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = acc / reps; }
}

int main() {
  std::vector<double> pay(NC), a(NC), b(NC);
  for (int i = 0; i < NC; ++i) { pay[i] = 1.0 - exp((double)(C0 + i) * DS); a[i] = pay[i] > 0 ? pay[i] : 0.0; }
  long long f = 0;
  for (int s = 1; s <= 300; ++s) {  // march the projected scheme (Jacobi), track the last green column
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
  printf("boundary after 300 rows: %lld\n", f);
  double *d_in, *d_out, *d_pay;
  long long* c;
  cudaMalloc(&d_in, 8 * NC); cudaMalloc(&d_out, 8 * NC); cudaMalloc(&d_pay, 8 * NC); cudaMalloc(&c, 16);
  cudaMemcpy(d_in, a.data(), 8 * NC, cudaMemcpyHostToDevice);
  cudaMemcpy(d_pay, pay.data(), 8 * NC, cudaMemcpyHostToDevice);
  for (int height : {32, 31, 24, 17}) {
    std::vector<double> ref(NC);
    long long kref = 0;
    for (int mode : {0, 1, 2}) {
      if (mode == 2 && 3 * height + 2 > 96) continue;
      const long long hi = f + 2 * height;
      cudaMemset(d_out, 0, 8 * NC);
      auto run = [&](int reps) {
        if (mode == 0) k<0><<<1, 32>>>(d_in, d_out, d_pay, c, reps, height, f, hi);
        if (mode == 1) k<1><<<1, 32>>>(d_in, d_out, d_pay, c, reps, height, f, hi);
        if (mode == 2) k<2><<<1, 32>>>(d_in, d_out, d_pay, c, reps, height, f, hi);
      };
      run(1);
      std::vector<double> o(NC);
      long long h[2];
      cudaMemcpy(o.data(), d_out, 8 * NC, cudaMemcpyDeviceToHost);
      cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
      if (mode == 0) { ref = o; kref = h[1]; }
      int diff = 0;
      for (int i = 0; i < NC; ++i) diff += (o[i] != ref[i]);
      long long kb = h[1];
      run(2000);
      cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
      printf("h %2d mode %d: %6.1f cycles/row  kb %lld (ref %lld)  output diffs %d  %s\n", height, mode,
             (double)h[0] / (2000.0 * height), kb, kref, diff, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
