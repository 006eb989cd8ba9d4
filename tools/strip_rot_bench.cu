// put_strip_ghost with the payoff shift in registers (ROT = 0, unrolled by 2:
// register moves every row) vs the rotating payoff file (ROT = 1, rows in
// groups of CPL, no moves): identical outputs; cycles/row alone, under
// shared-memory load on the other SMSPs, and with a second strip on the same
// SMSP (the in-kernel condition of the two chain warps); variants 2 / 3 also
// compare on the integer pipe (proj_max_i).
#include <cmath>
#include <cstdio>
#include <vector>
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "strip_variants.cuh"
using namespace fl;
constexpr int NC = 1201, C0 = -600;
constexpr double CD = 0.39790368627109396, CM = 0.199951171875, CU = 0.4020963137289061;

template <int V>
__device__ __forceinline__ int64_t strip(const double* in, double* out, const double* pay, long long f, int h) {
  if (V == 0) return put_strip_ghost<5, 0>(in, out, pay, f, h, CD, CM, CU);
  return put_strip_ghost_rot<5, V>(in, out, pay, f, h, CD, CM, CU);
}

template <int V, int NOISE>
__global__ void __launch_bounds__(512, 1) k(const double* in, const double* pay, long long* cyc, double* outg, int reps,
                                           int height, long long f, volatile int* stop) {
  __shared__ double spay[NC], sin_[NC], sout[NC], sout2[NC], sn[2048];
  for (int i = threadIdx.x; i < NC; i += blockDim.x) { spay[i] = pay[i]; sin_[i] = in[i]; sout[i] = 0; sout2[i] = 0; }
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sn[i] = i;
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    long long t0 = clock64();
    int64_t acc = 0;
    for (int r = 0; r < reps; ++r) acc += strip<V>(sin_ - C0, sout - C0, spay - C0, f, height);
    long long t1 = clock64();
    for (int i = lane; i < NC; i += 32) outg[i] = sout[i];
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = acc; *stop = 1; }
    return;
  }
  if (NOISE == 0) return;
  if (NOISE == 1 && !(w == 1 || w == 2 || w == 3)) return;
  if (NOISE == 2 && w != 4) return;
  double x = lane;
  int i = lane;
  while (!*stop) {
    if (NOISE == 1) {
#pragma unroll
      for (int j = 0; j < 16; ++j) { x += sn[(lane + j * 32 + i) & 2047]; i += 64; }
    } else {
      strip<V>(sin_ - C0, sout2 - C0, spay - C0, f, height);
    }
  }
  if (x == 12345.0) cyc[2] = 1;
}

int main() {
  std::vector<double> pay(NC), a(NC), b(NC);
  const double DS = 0.0069877124296868435;
  for (int i = 0; i < NC; ++i) { pay[i] = 1.0 - exp((double)(C0 + i) * DS); a[i] = pay[i] > 0 ? pay[i] : 0.0; }
  long long f = 0;
  for (int s = 1; s <= 300; ++s) {
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
  double *d_in, *d_pay, *d_out; long long* c; int* stop;
  cudaMalloc(&d_in, 8 * NC); cudaMalloc(&d_pay, 8 * NC); cudaMalloc(&d_out, 8 * NC); cudaMalloc(&c, 32); cudaMalloc(&stop, 4);
  cudaMemcpy(d_in, a.data(), 8 * NC, cudaMemcpyHostToDevice);
  cudaMemcpy(d_pay, pay.data(), 8 * NC, cudaMemcpyHostToDevice);
  const char* names[] = {"alone", "shared loads, other SMSPs", "2nd strip, same SMSP"};
  for (int height : {64, 63, 17}) {
    std::vector<std::vector<double>> ov(4, std::vector<double>(NC));
    long long kb[4] = {0, 0, 0, 0};
    for (int noise = 0; noise < 3; ++noise) {
      double cyc_v[4];
      for (int v = 0; v < 4; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
          cudaMemset(stop, 0, 4);
          const int reps = rep == 0 ? 2 : 400;
          if (v == 0 && noise == 0) k<0, 0><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 0 && noise == 1) k<0, 1><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 0 && noise == 2) k<0, 2><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 1 && noise == 0) k<1, 0><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 1 && noise == 1) k<1, 1><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 1 && noise == 2) k<1, 2><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 2 && noise == 0) k<2, 0><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 2 && noise == 1) k<2, 1><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 2 && noise == 2) k<2, 2><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 3 && noise == 0) k<3, 0><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 3 && noise == 1) k<3, 1><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          if (v == 3 && noise == 2) k<3, 2><<<1, 512>>>(d_in, d_pay, c, d_out, reps, height, f, stop);
          cudaDeviceSynchronize();
        }
        long long h[2];
        cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
        cyc_v[v] = h[0] / (400.0 * height);
        if (noise == 0) {
          kb[v] = h[1] / 400;
          cudaMemcpy(ov[v].data(), d_out, 8 * NC, cudaMemcpyDeviceToHost);
        }
      }
      printf("h=%d %-28s shift %.1f  rotating %.1f  shift+icmp %.1f  rotating+icmp %.1f cycles/row  (%s)\n", height,
             names[noise], cyc_v[0], cyc_v[1], cyc_v[2], cyc_v[3], cudaGetErrorString(cudaGetLastError()));
    }
    bool same = true;
    for (int v = 1; v < 4; ++v) {
      same = same && kb[v] == kb[0];
      for (int i = 0; i < NC; ++i)
        same = same && (ov[0][i] == ov[v][i] || (std::isnan(ov[0][i]) && std::isnan(ov[v][i])));
    }
    printf("h=%d outputs bit-identical (4 variants): %s (kb %lld)\n", height, same ? "yes" : "NO", kb[0]);
  }
  return 0;
}
