// FP64 tensor-core (mma.sync .f64) availability, fragment layout and
// throughput on this GPU, against the DFMA pipe.
#include <cstdio>
#include <cmath>

__device__ __forceinline__ void mma16n8k4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b0));
}

// layout probe: A[r][k] = r*10 + k, B[k][n] = (k == n%4) ? 1 : 0 -> D[r][n] = A[r][n%4]
__global__ void layout(double* out) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  const double a0 = g * 10 + t, a1 = (g + 8) * 10 + t;   // assumed: a0 (row g, col t), a1 (row g+8, col t)
  const double b0 = (t == (g % 4)) ? 1.0 : 0.0;          // assumed: b0 (row t, col g)
  double d[4] = {0, 0, 0, 0};
  mma16n8k4(d, a0, a1, b0);
  for (int i = 0; i < 4; ++i) out[lane * 4 + i] = d[i];
}

template <int CH>
__global__ void __launch_bounds__(256) mma_tp(double* out, int iters) {
  double d[CH][4];
  for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) d[c][i] = 0.0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma16n8k4(d[c], a0, a1, b0);
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) for (int i = 0; i < 4; ++i) s += d[c][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dfma_tp(double* out, int iters) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999, 1e-3);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// both at once: half the warps DMMA, half DFMA (do they share a pipe?)
template <int MODE>  // 0: both halves, 1: DMMA half only, 2: DFMA half only
__global__ void __launch_bounds__(512) mixed(double* out, int iters) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if ((MODE == 1 && !(w & 1)) || (MODE == 2 && (w & 1))) { out[blockIdx.x * blockDim.x + threadIdx.x] = 0; return; }
  if (w & 1) {
    double d[4][4] = {};
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = 0.5;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int c = 0; c < 4; ++c) mma16n8k4(d[c], a0, a1, b0);
    for (int c = 0; c < 4; ++c) for (int i = 0; i < 4; ++i) s += d[c][i];
  } else {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999, 1e-3);
    for (int k = 0; k < 8; ++k) s += x[k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8 << 20);
  double h[128];
  layout<<<1, 32>>>(d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("layout probe (%s):\n", cudaGetErrorString(cudaGetLastError()));
  int bad = 0;
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    // assumed: d0,d1 (row g, cols 2t, 2t+1); d2,d3 (row g+8, cols 2t, 2t+1)
    const double e[4] = {g * 10.0 + (2 * t) % 4, g * 10.0 + (2 * t + 1) % 4, (g + 8) * 10.0 + (2 * t) % 4,
                         (g + 8) * 10.0 + (2 * t + 1) % 4};
    for (int i = 0; i < 4; ++i) bad += h[lane * 4 + i] != e[i];
    if (lane < 4) printf("  lane %d: %g %g %g %g (expect %g %g %g %g)\n", lane, h[lane*4], h[lane*4+1], h[lane*4+2], h[lane*4+3], e[0], e[1], e[2], e[3]);
  }
  printf("layout mismatches: %d\n", bad);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto fn, double work, const char* name) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %.2f TFLOP/s (%s)\n", name, work / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  const int it = 4096;
  timeit([&] { mma_tp<4><<<nsm * 4, 256>>>(d, it); }, 2.0 * 512 * 4 * it * (nsm * 4.0 * 256 / 32), "dmma m16n8k4 (4 chains)");
  timeit([&] { mma_tp<8><<<nsm * 4, 256>>>(d, it); }, 2.0 * 512 * 8 * it * (nsm * 4.0 * 256 / 32), "dmma m16n8k4 (8 chains)");
  timeit([&] { dfma_tp<<<nsm * 4, 256>>>(d, it / 4); }, 2.0 * 16 * 8 * (it / 4) * (nsm * 4.0 * 256), "dfma");
  auto tms = [&](auto fn) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
  };
  const float m0 = tms([&] { mixed<0><<<nsm * 2, 512>>>(d, it / 2); });
  const float m1 = tms([&] { mixed<1><<<nsm * 2, 512>>>(d, it / 2); });
  const float m2 = tms([&] { mixed<2><<<nsm * 2, 512>>>(d, it / 2); });
  printf("DMMA warps alone %.3f ms, DFMA warps alone %.3f ms, both together %.3f ms (sum %.3f: %s)\n", m1, m2, m0,
         m1 + m2, m0 < 0.8 * (m1 + m2) ? "separate pipes, they overlap" : "one shared pipe");
  return 0;
}
