// Microbenchmark: call leaf strips (v2 vs v3) alone on one warp, cycles per row.
#include <cstdio>
#include <cmath>
#include "fl_lib.cu"
#include "strip_variants.cuh"
using namespace fl;
template <int MODE>
__global__ void k(const CallParams P, const double* in, double* out, double* e2, long long* cyc, int reps, int height) {
  __shared__ double se2[40];
  if (threadIdx.x < 33) se2[threadIdx.x] = exp(2.0 * (double)threadIdx.x * P.lu);
  __syncwarp();
  const int64_t j0 = 1000, lo = j0 - height + 1, top = 2000;
  double cells = 0;
  long long t0 = clock64();
  int64_t acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (MODE == 0) acc += call_leaf_v2(P, in, out, lo, top, j0, height, &cells);
    else acc += call_leaf_v3(P, in, out, lo, top, j0, height, &cells, se2);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = acc; }
}
int main() {
  CallParams P{};
  P.S = 100; P.K = 95; P.lu = 0.002; P.wd = 0.4985; P.wu = 0.5012;
  double *in, *out, *e2; long long* c;
  cudaMalloc(&in, 8 * 4096); cudaMalloc(&out, 8 * 4096); cudaMalloc(&e2, 8 * 64); cudaMalloc(&c, 16);
  double h_in[4096];
  for (int i = 0; i < 4096; ++i) h_in[i] = fmax(100 * exp((2 * i - 2000) * 0.002) - 95, 0.0) + 1.0;
  cudaMemcpy(in, h_in, sizeof(h_in), cudaMemcpyHostToDevice);
  for (int height : {32, 17}) for (int mode : {0, 1}) {
    long long h[2];
    auto run = [&](int reps) { if (mode == 0) k<0><<<1, 32>>>(P, in, out, e2, c, reps, height); else k<1><<<1, 32>>>(P, in, out, e2, c, reps, height); };
    run(1); run(1000);
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("height %d mode %d: %.1f cycles/row (incl. setup) jp %lld (%s)\n", height, mode, h[0] / (1000.0 * height), h[1] / 1000, cudaGetErrorString(cudaGetLastError()));
  }
}
