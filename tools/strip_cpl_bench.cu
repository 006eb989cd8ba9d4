// Leaf-strip row cost against the frame's cells per lane: put_strip_ghost<CPL>
// at the tallest leaf each CPL holds (2h+2 <= 31 CPL: h = 30, 45, 61, 76 and
// the production h = 64 at CPL 5), alone, with a second strip on the same
// SMSP (the in-kernel pairing of the two chain warps), with conflict-free
// shared loads on the other SMSPs (FFT groups / helpers) and with both.
// Answers: how much of the in-kernel strip cost scales with the cells a lane
// carries.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2303_02317_b200/csrc/fl_common.cuh"
#include "../paper_2303_02317_b200/csrc/fl_strip.cuh"
#include "strip_variants.cuh"
using namespace fl;
constexpr int NC = 1201, C0 = -600;
constexpr double CD = 0.39790368627109396, CM = 0.199951171875, CU = 0.4020963137289061;


// Diagnostic copies of put_strip_ghost (timing only; V = 1, 2 give wrong values):
//   V 0: production body;  V 1: no payoff load (next payoff from registers);
//   V 2: no shuffles (left cells from the lane itself);
//   V 3: payoff loads 4 rows ahead (4-entry register queue, same values as V 0).
template <int CPL, int V>
__device__ int64_t strip_diag(const double* __restrict__ in_org, double* __restrict__ out_org,
                              const double* __restrict__ pay_org, int64_t f, int height, double cd, double cm,
                              double cu) {
  const int lane = threadIdx.x & 31;
  const int W = 2 * height + 2;
  const int j0 = (lane - 1) * CPL;
  const double* pay0 = pay_org + (f - 1);
  int jx[CPL];
  double u[CPL], p[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    jx[c] = (j0 + c < W) ? j0 + c : W - 1;
    p[c] = pay0[jx[c]];
    u[c] = (jx[c] <= 1) ? p[c] : in_org[f - 1 + jx[c]];
  }
  __syncwarp();
  const double* pq0 = pay0 - 1 + jx[0];
  double q0 = pq0[0], q1 = pq0[-1], q2 = pq0[-2], q3 = pq0[-3];
  double np0 = q0;
#pragma unroll 4
  for (int s = 0; s < height; ++s) {
    double L2, L1;
    if (V == 2) { L2 = u[CPL - 2]; L1 = u[CPL - 1]; }
    else { L2 = __shfl_up_sync(FULL, u[CPL - 2], 1); L1 = __shfl_up_sync(FULL, u[CPL - 1], 1); }
    double np[CPL];
    if (V == 3) {
      np[0] = q0; q0 = q1; q1 = q2; q2 = q3; q3 = pq0[-(s + 4)];
    } else {
      np[0] = np0;
      np0 = (V == 1) ? p[CPL - 1] : pq0[-(s + 1)];
    }
#pragma unroll
    for (int c = 1; c < CPL; ++c) np[c] = p[c - 1];
    double nu[CPL];
#pragma unroll
    for (int c = CPL - 1; c >= 2; --c) {
      const double lin = fma(cd, u[c - 2], fma(cu, u[c], cm * u[c - 1]));
      nu[c] = proj_max(lin, np[c]);
    }
    const double lin1 = fma(cd, L1, fma(cu, u[1], cm * u[0]));
    const double lin0 = fma(cd, L2, fma(cu, u[0], cm * L1));
    nu[1] = proj_max(lin1, np[1]);
    nu[0] = proj_max(lin0, np[0]);
#pragma unroll
    for (int c = 0; c < CPL; ++c) { u[c] = nu[c]; p[c] = np[c]; }
  }
  unsigned green = 0;
#pragma unroll
  for (int c = 0; c < CPL; ++c) green |= (u[c] == p[c] ? 1u : 0u) << c;
  int best = -1;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (((green >> c) & 1u) && j0 + c >= 0 && j0 + c < W) best = j0 + c;
  best = warp_max_i32(best);
  const int64_t base = f - height - 1;
  const int64_t kb = (best < 0) ? NONE_SEEN : base + best;
  const int jlo = (best < 0) ? W : best + 1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int j = j0 + c;
    if (j >= jlo && j < W) out_org[base + j] = u[c];
  }
  __syncwarp();
  return kb;
}


// Fixed-column frame, K rows per neighbour exchange: a lane holds K halo cells
// of each neighbour around its CPL cells and advances K rows on the tile
// (row r of the group recomputes the halo cone shrinking by one per side).
template <int CPL, int K>
__device__ int64_t strip_fixed_tiled(const double* __restrict__ in_org, double* __restrict__ out_org,
                                     const double* __restrict__ pay_org, int64_t f, int height, double cd, double cm,
                                     double cu) {
  constexpr int NT = CPL + 2 * K;
  const int lane = threadIdx.x & 31;
  const int h = height;
  const int Mx = 31 * CPL - 2 * h - 1;
  const int M = Mx < 2 * h ? Mx : 2 * h;
  const int64_t base = f - M;
  const int W = M + 2 * h + 1;
  const int j0 = (lane - 1) * CPL;
  double v[NT], p[NT];
#pragma unroll
  for (int c = 0; c < NT; ++c) {
    int j = j0 + c - K;
    j = j < W ? j : W - 1;
    int64_t col = base + j;
    col = col < f - 2 * h - 1 ? f - 2 * h - 1 : col;
    p[c] = pay_org[col];
    v[c] = (col <= f) ? p[c] : in_org[col];
  }
  __syncwarp();
  bool cont0 = false;
  int s = 0;
#pragma unroll 1
  for (; s + K <= h; s += K) {
    // halos from the neighbours' own cells
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double a = __shfl_up_sync(FULL, v[K + CPL - K + k], 1);
      const double b = __shfl_down_sync(FULL, v[K + k], 1);
      v[k] = a;
      v[K + CPL + k] = b;
    }
#pragma unroll
    for (int r = 1; r <= K; ++r) {
      double nv[NT];
#pragma unroll
      for (int c = r; c < NT - r; ++c) {
        const double lin = fma(cd, v[c - 1], fma(cu, v[c + 1], cm * v[c]));
        if (c == K) cont0 |= lin > p[c];
        nv[c] = proj_max(lin, p[c]);
      }
#pragma unroll
      for (int c = r; c < NT - r; ++c) v[c] = nv[c];
    }
  }
  for (; s < h; ++s) {  // remainder rows, one exchange each
    const double a = __shfl_up_sync(FULL, v[K + CPL - 1], 1);
    const double b = __shfl_down_sync(FULL, v[K], 1);
    v[K - 1] = a;
    v[K + CPL] = b;
    double nv[NT];
#pragma unroll
    for (int c = K; c < K + CPL; ++c) {
      const double lin = fma(cd, v[c - 1], fma(cu, v[c + 1], cm * v[c]));
      if (c == K) cont0 |= lin > p[c];
      nv[c] = proj_max(lin, p[c]);
    }
#pragma unroll
    for (int c = K; c < K + CPL; ++c) v[c] = nv[c];
  }
  if (__shfl_sync(FULL, cont0 ? 1 : 0, 1)) return FIXED_MISS;
  int best = -1;
#pragma unroll
  for (int c = 0; c < CPL; ++c)
    if (v[K + c] == p[K + c] && j0 + c >= 0 && j0 + c <= M + h) best = j0 + c;
  best = warp_max_i32(best);
  const int64_t kb = (best < 0) ? NONE_SEEN : base + best;
  const int jlo = (best < 0) ? W : best + 1;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int j = j0 + c;
    if (j >= jlo && j <= M + h) out_org[base + j] = v[K + c];
  }
  __syncwarp();
  return kb;
}

template <int CPL, int V>
__device__ __forceinline__ int64_t strip_sel(const double* in, double* out, const double* pay, int64_t f, int h) {
  if constexpr (V < 0) return put_strip_ghost<CPL, 0>(in, out, pay, f, h, CD, CM, CU);
  if constexpr (V == 10) return put_strip_fixed<CPL>(in, out, pay, f, h, CD, CM, CU);
  if constexpr (V >= 30) return strip_fixed_tiled<CPL, V - 29>(in, out, pay, f, h, CD, CM, CU);
  else return strip_diag<CPL, (V < 10 ? V : 0)>(in, out, pay, f, h, CD, CM, CU);
}

template <int CPL, int MODE, int V = -1>
__global__ void __launch_bounds__(512, 1) k(const double* in, const double* pay, long long* cyc, int reps, int height,
                                           long long f, volatile int* stop, double* gout) {
  __shared__ double spay[NC], sin_[NC], sout[2][NC], sn[512];
  for (int i = threadIdx.x; i < NC; i += blockDim.x) { spay[i] = pay[i]; sin_[i] = in[i]; sout[0][i] = -7.0; }
  for (int i = threadIdx.x; i < 512; i += blockDim.x) sn[i] = i;
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 3) {
    long long t0 = clock64();
    int64_t acc = 0;
    for (int r = 0; r < reps; ++r)
      acc += strip_sel<CPL, V>(sin_ - C0, sout[0] - C0, spay - C0, f, height);
    long long t1 = clock64();
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = acc; *stop = 1; }
    for (int i = lane; i < NC; i += 32) gout[i] = sout[0][i];
    return;
  }
  const bool pair = (MODE & 1) && w == 7;                 // same SMSP as warp 3
  const bool noise = (MODE & 2) && (w & 3) != 3 && w < 12;  // 9 warps on SMSPs 0-2
  if (!pair && !noise) return;
  double x = lane;
  int i = lane;
  while (!*stop) {
    if (pair) {
      strip_sel<CPL, V>(sin_ - C0, sout[1] - C0, spay - C0, f, height);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) { x += sn[(lane + j * 32 + i) & 511]; i += 64; }
    }
  }
  if (x == 12345.0) cyc[2] = 1;
}

double* gout;
std::vector<double> ref_out;
void check_out(const char* tag) {
  std::vector<double> o(NC);
  cudaMemcpy(o.data(), gout, 8 * NC, cudaMemcpyDeviceToHost);
  if (ref_out.empty()) { ref_out = o; return; }
  int diff = 0;
  for (int i = 0; i < NC; ++i) diff += (o[i] != ref_out[i]);
  printf("  %s: outputs vs ghost: %d differing cells\n", tag, diff);
}

template <int CPL, int V = -1>
void run_cpl(const double* d_in, const double* d_pay, long long* c, int* stop, long long f, int h) {
  const char* names[] = {"alone", "2nd strip same SMSP", "lds other SMSPs", "2nd strip + lds"};
  for (int mode = 0; mode < 4; ++mode) {
    double res = 0;
    long long kb = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(stop, 0, 4);
      const int reps = rep == 0 ? 2 : 400;
      switch (mode) {
        case 0: k<CPL, 0, V><<<1, 512>>>(d_in, d_pay, c, reps, h, f, stop, gout); break;
        case 1: k<CPL, 1, V><<<1, 512>>>(d_in, d_pay, c, reps, h, f, stop, gout); break;
        case 2: k<CPL, 2, V><<<1, 512>>>(d_in, d_pay, c, reps, h, f, stop, gout); break;
        case 3: k<CPL, 3, V><<<1, 512>>>(d_in, d_pay, c, reps, h, f, stop, gout); break;
      }
      cudaDeviceSynchronize();
      long long hh[2];
      cudaMemcpy(hh, c, 16, cudaMemcpyDeviceToHost);
      res = hh[0] / (double(reps) * h);
      kb = hh[1] / reps;
    }
    printf("V %2d CPL %d h %2d  %-22s %6.1f cycles/row  %6.0f cycles/strip  (kb %lld) %s\n", V, CPL, h, names[mode], res,
           res * h, kb, cudaGetErrorString(cudaGetLastError()));
    if (mode == 0 && h == 64 && CPL == 5 && (V == -1 || V >= 10)) check_out(V == -1 ? "ghost" : "variant");
  }
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
  double *d_in, *d_pay; long long* c; int* stop;
  cudaMalloc(&gout, 8 * NC);
  cudaMalloc(&d_in, 8 * NC); cudaMalloc(&d_pay, 8 * NC); cudaMalloc(&c, 32); cudaMalloc(&stop, 4);
  cudaMemcpy(d_in, a.data(), 8 * NC, cudaMemcpyHostToDevice);
  cudaMemcpy(d_pay, pay.data(), 8 * NC, cudaMemcpyHostToDevice);
  run_cpl<5>(d_in, d_pay, c, stop, f, 64);
  run_cpl<5, 10>(d_in, d_pay, c, stop, f, 64);
  run_cpl<5, 31>(d_in, d_pay, c, stop, f, 64);
  run_cpl<5, 32>(d_in, d_pay, c, stop, f, 64);
  run_cpl<5, 33>(d_in, d_pay, c, stop, f, 64);
  run_cpl<5, 35>(d_in, d_pay, c, stop, f, 64);
  run_cpl<4, 31>(d_in, d_pay, c, stop, f, 61);
  run_cpl<4, 32>(d_in, d_pay, c, stop, f, 61);
  run_cpl<5, 2>(d_in, d_pay, c, stop, f, 64);
  return 0;
}
