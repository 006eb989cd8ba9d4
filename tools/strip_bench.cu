// Microbenchmark: cycles per row of the warp-level put strip (fl_strip.cuh), alone.
#include <cstdio>
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "../paper_2303_02317_b200/csrc/fl_strip.cuh"
using namespace fl;
__global__ void k(double* in, double* out, double* pay, long long* cyc, int reps) {
  int64_t lo = 0, hi = 129, f = 64;
  long long t0 = clock64();
  int64_t acc = 0;
  for (int r = 0; r < reps; ++r) acc += put_strip_warp<5>(in, out, pay, lo, hi, f, 32, 0.4, 0.2, 0.39);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = acc; }
}
int main() {
  double *in, *out, *pay; long long* c;
  cudaMalloc(&in, 8 * 256); cudaMalloc(&out, 8 * 256); cudaMalloc(&pay, 8 * 256); cudaMalloc(&c, 16);
  cudaMemset(in, 0, 2048); cudaMemset(pay, 0, 2048);
  k<<<1, 32>>>(in, out, pay, c, 10);
  k<<<1, 32>>>(in, out, pay, c, 1000);
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("put strip: %.1f cycles/row (err %s)\n", (double)h[0] / (1000.0 * 32), cudaGetErrorString(cudaGetLastError()));
}
