// Microbenchmark of the warp direct correlation (fl_sched.cuh: warp_conv_direct)
// from shared memory, at the fused-node sizes (Lout ~ 2h-2h1, M = 2h1+1).
#include <cstdio>

#include "../paper_2303_02317_b200/csrc/fl_sched.cuh"
using namespace fl;

__global__ void k(long long* cyc, double* sink, int Lout, int M, int reps) {
  __shared__ double sx[512], sw[160], sy[256];
  for (int i = threadIdx.x; i < 512; i += 32) sx[i] = 1.0 / (1 + i);
  for (int i = threadIdx.x; i < 160; i += 32) sw[i] = 0.01 * i;
  __syncwarp();
  long long t0 = clock64();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    acc += warp_conv_direct(sx + (r & 1), sy, Lout, sw, M);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; sink[0] = acc + sy[3]; }
}

int main() {
  long long* c;
  double* s;
  cudaMalloc(&c, 8);
  cudaMalloc(&s, 8);
  int cases[][2] = {{48, 49}, {64, 65}, {32, 33}, {128, 129}, {96, 65}};
  for (auto& cs : cases) {
    k<<<1, 32>>>(c, s, cs[0], cs[1], 1000);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("Lout %3d M %3d: %7.1f cycles/call  (%s)\n", cs[0], cs[1], h / 1000.0, cudaGetErrorString(cudaGetLastError()));
  }
}
