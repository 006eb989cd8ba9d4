// Single-warp issue rates of FP64 ops on one SMSP.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters, double a, double b, int mode) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (mode == 0) x[i] = fma(x[i], a, b);
      else if (mode == 1) x[i] = x[i] > b ? x[i] * a : b;   // DSETP + DMUL + select
      else if (mode == 2) x[i] = x[i] * a;
      else if (mode == 4) x[i] = fmax(x[i] * a, b);
      else if (mode == 5) { long long u = __double_as_longlong(x[i] * a), v = __double_as_longlong(b); x[i] = __longlong_as_double(u > v ? u : v); }
      else if (mode == 3) x[i] = x[i] + a;
    }
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 4096); cudaMalloc(&c, 8);
  const char* nm[] = {"dfma", "dsetp+dmul+sel", "dmul", "dadd", "dmul+fmax", "dmul+int-max"};
  for (int mode = 0; mode < 6; ++mode) {
    for (int warps : {1, 4}) {
      k<<<1, 32 * warps>>>(d, c, 10, 0.999, 1e-3, mode);
      k<<<1, 32 * warps>>>(d, c, 1000, 0.999, 1e-3, mode);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("%-16s warps %d: %.2f cycles per warp-op (per warp)\n", nm[mode], warps, (double)h / (1000.0 * 16));
    }
  }
}
