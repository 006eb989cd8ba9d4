// Microbenchmark: FP64 DFMA throughput and latency on the device (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void shfl_lat(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __shfl_down_sync(0xffffffffu, x, 1) + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; long long* c; cudaMalloc(&d, 1 << 26); cudaMalloc(&c, 64);
  int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bs : {256, 512, 1024}) {
    int grid = 148 * (2048 / bs);
    dfma_tput<<<grid, bs>>>(d, 16, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_tput<<<grid, bs>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * grid * bs;
    printf("dfma_tput bs=%d grid=%d: %.3f ms  %.2f TFLOP/s\n", bs, grid, ms, flops / ms / 1e9);
  }
  long long h;
  dfma_lat<<<1, 32>>>(d, c, iters, 0.999, 1e-3);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("dfma latency: %.2f cycles\n", (double)h / (16.0 * iters));
  shfl_lat<<<1, 32>>>(d, c, iters);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("shfl64+dadd latency: %.2f cycles\n", (double)h / (16.0 * iters));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr: %d kHz\n", clk);
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
