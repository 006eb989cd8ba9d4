// conv_dmma (tensor-core direct correlation) vs conv_fft for the recursion
// nodes' jump sizes, one 4-warp group alone on an SM: cycles per task and
// max |difference|.
#include <cstdio>
#include <cmath>
#include <vector>
#include "dmma_conv.cuh"
using namespace fl;

__global__ void kern(const double* x, int64_t L, double* y1, double* y2, int64_t Lout, int h, Stencil st,
                     const double* w, int M, int64_t rlo, long long* cyc, int reps) {
  extern __shared__ double2 sb[];
  __shared__ double2 tq[TWQ];
  for (int i = threadIdx.x; i < TWQ; i += blockDim.x) tq[i] = fl_tw[i];
  __syncthreads();
  const Grp g{(int)threadIdx.x, 128, 1};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) conv_dmma(x + rlo, L - rlo, y1, Lout, w, M, (double*)sb, 2 * smem_complex_slots(2048), g);
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) conv_fft(x, L, y2, Lout, h, st, sb, 12, tq, g);
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; cyc[1] = (t2 - t1) / reps; }
}

void init_tw() {
  std::vector<double2> h(TW_N);
  for (int m = 0; m < TW_N; ++m) { long double a = 6.283185307179586476925L * m / TW_N; h[m] = make_double2((double)cosl(a), (double)-sinl(a)); }
  cudaMemcpyToSymbol(fl_tw, h.data(), sizeof(double2) * TW_N);
}

int main() {
  init_tw();
  const Stencil st{0.39790368627109396, 0.199951171875, 0.4020963137289061, 2};
  for (int h : {256, 512}) {
    int64_t rlo; const int M = (int)window_width(st, h, &rlo);
    const int64_t Lout = 2 * h;   // a node's mid jump: 2h inputs -> ~h outputs; use 2h outputs for a bigger one
    const int64_t L = Lout + 2 * h + 1;
    // W_h by repeated convolution on the host
    std::vector<double> W(1, 1.0);
    for (int k = 0; k < h; ++k) { std::vector<double> n(W.size() + 2, 0.0); for (size_t i = 0; i < W.size(); ++i) { n[i] += st.c0 * W[i]; n[i + 1] += st.c1 * W[i]; n[i + 2] += st.c2 * W[i]; } W.swap(n); }
    std::vector<double> xs(L); for (int64_t i = 0; i < L; ++i) xs[i] = 1.0 + 0.5 * sin(0.01 * i);
    double *dx, *dy1, *dy2, *dw; long long* dc;
    cudaMalloc(&dx, 8 * L); cudaMalloc(&dy1, 8 * Lout); cudaMalloc(&dy2, 8 * Lout); cudaMalloc(&dw, 8 * M); cudaMalloc(&dc, 16);
    cudaMemcpy(dx, xs.data(), 8 * L, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, W.data() + rlo, 8 * M, cudaMemcpyHostToDevice);
    const int smem = smem_complex_slots(2048) * 16;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<1, 128, smem>>>(dx, L, dy1, dy2, Lout, h, st, dw, M, rlo, dc, 2);
    kern<<<1, 128, smem>>>(dx, L, dy1, dy2, Lout, h, st, dw, M, rlo, dc, 20);
    long long c[2]; cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
    std::vector<double> a(Lout), b(Lout); cudaMemcpy(a.data(), dy1, 8 * Lout, cudaMemcpyDeviceToHost); cudaMemcpy(b.data(), dy2, 8 * Lout, cudaMemcpyDeviceToHost);
    double md = 0; for (int64_t i = 0; i < Lout; ++i) md = fmax(md, fabs(a[i] - b[i]));
    printf("h=%d M=%d Lout=%lld: dmma %lld cycles, fft %lld cycles, max|diff| %.2e (%s)\n", h, M, (long long)Lout, c[0], c[1], md, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
