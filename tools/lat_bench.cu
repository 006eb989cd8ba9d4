// Dependent-latency microbenchmarks for the strip's critical path (one warp, templated per op).
#include <cstdio>
template <int MODE>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = out[threadIdx.x], p = out[threadIdx.x + 32];
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (MODE == 0) x = fma(x, a, b);
      if (MODE == 1) x = __shfl_xor_sync(0xffffffffu, x, 1);
      if (MODE == 2) x = (x > p) ? x : p * a;
      if (MODE == 3) x = x * a;
      if (MODE == 4) { double r = __shfl_down_sync(0xffffffffu, x, 1); double l = fma(a, r, b); x = (l > p) ? l : p; }
      if (MODE == 5) x = __int_as_float(__shfl_xor_sync(0xffffffffu, __float_as_int((float)x), 1));
      if (MODE == 6) x = x + a;
      if (MODE == 7) { float y = (float)x; y = fmaf(y, (float)a, (float)b); x = y; }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int M> void run(double* o, long long* c, const char* name) {
  k<M><<<1, 32>>>(o, c, 0.999, 1e-3, 10);
  k<M><<<1, 32>>>(o, c, 0.999, 1e-3, 1000);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %.1f cycles per dependent step\n", name, h / 16000.0);
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
  cudaMemset(o, 0, 64 * 8);
  run<0>(o, c, "dfma");
  run<3>(o, c, "dmul");
  run<6>(o, c, "dadd");
  run<1>(o, c, "shfl.f64 (2 x b32)");
  run<5>(o, c, "shfl.b32 + f2f round trip");
  run<2>(o, c, "dsetp/fsel (+dmul off path)");
  run<4>(o, c, "strip cycle shfl->dfma->dsetp/fsel");
  run<7>(o, c, "f64->f32 ffma ->f64");
}
