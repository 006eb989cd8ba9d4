// Direct correlation throughput on one warp: weights in shared vs global memory,
// at the subtree chunk sizes (Lout = 64, M = 65 / 129 / 257).
#include <cstdio>
#include "../paper_2303_02317_b200/csrc/fl_sched.cuh"
using namespace fl;
__global__ void k(long long* cyc, double* sink, const double* gw, int Lout, int M, int reps, int wglobal) {
  __shared__ double sx[1024], sw[300], sy[256];
  for (int i = threadIdx.x; i < 1024; i += 32) sx[i] = 1.0 / (1 + i);
  for (int i = threadIdx.x; i < 300; i += 32) sw[i] = gw[i];
  __syncwarp();
  const double* w = wglobal ? gw : sw;
  long long t0 = clock64();
  double acc = 0;
  for (int r = 0; r < reps; ++r) acc += warp_conv_direct(sx + (r & 1), sy, Lout, w, M);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; sink[0] = acc + sy[3]; }
}
int main() {
  long long* c; double *s, *gw;
  cudaMalloc(&c, 8); cudaMalloc(&s, 8); cudaMalloc(&gw, 8 * 300);
  double h[300]; for (int i = 0; i < 300; ++i) h[i] = 0.001 * i; cudaMemcpy(gw, h, 2400, cudaMemcpyHostToDevice);
  int cases[][2] = {{64, 65}, {64, 129}, {64, 257}, {128, 257}};
  for (auto& cs : cases) for (int g = 0; g < 2; ++g) {
    k<<<1, 32>>>(c, s, gw, cs[0], cs[1], 500, g);
    long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("Lout %3d M %3d w_%s: %7.1f cycles/call  %.2f FMA/cycle\n", cs[0], cs[1], g ? "global" : "shared", hc / 500.0,
           cs[0] * cs[1] / (hc / 500.0));
  }
}
