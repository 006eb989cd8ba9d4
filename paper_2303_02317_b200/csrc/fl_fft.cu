// fl_fft.cu -- the reference's generic transform utilities on the device:
// fft_forward / fft_inverse (fft.py:84-123: unnormalised power-of-two DFT and
// its 1/N inverse) and convolve (fft.py:130-163: full linear convolution by the
// transform pair, zero-padded to the next power of two >= len(x)+len(y)-1).
//
// Not on the pricing hot path (the pricers use the fused correlations of
// fl_conv.cuh); these serve the drop-in API.  Radix-2 Stockham autosort passes
// in global memory (natural-order in and out, one launch per pass), twiddles
// by sincospi of the exact ratio k / Ns.
#include <cstdint>

#include "fl_common.cuh"
#include "fl_kernels.h"

namespace fl {

// One radix-2 Stockham pass: sub-transforms of length Ns -> 2 Ns.
__global__ void fft_stockham_pass(const double2* __restrict__ in, double2* __restrict__ out, int64_t n, int64_t ns,
                                  double sign) {
  const int64_t half = n >> 1;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < half; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = j & (ns - 1);
    double s, c;
    sincospi(sign * (double)k / (double)ns, &s, &c);  // exp(sign * i * pi * k / ns)
    const double2 a = in[j];
    const double2 b0 = in[j + half];
    const double2 b = make_double2(b0.x * c - b0.y * s, b0.x * s + b0.y * c);
    const int64_t d = (j - k) * 2 + k;  // (j / ns) * 2 ns + k
    out[d] = make_double2(a.x + b.x, a.y + b.y);
    out[d + ns] = make_double2(a.x - b.x, a.y - b.y);
  }
}

__global__ void cmul_inplace(double2* __restrict__ a, const double2* __restrict__ b, int64_t n, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = a[i], y = b[i];
    a[i] = make_double2((x.x * y.x - x.y * y.y) * scale, (x.x * y.y + x.y * y.x) * scale);
  }
}

__global__ void cscale_inplace(double2* __restrict__ a, int64_t n, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = make_double2(a[i].x * scale, a[i].y * scale);
}

static int grid_for(int64_t work) {
  const int64_t g = (work + 255) / 256;
  return (int)(g < 148 * 8 ? (g < 1 ? 1 : g) : 148 * 8);
}

// In-place (ping-pong) transform of buf (n a power of two); returns the buffer
// holding the result (buf or tmp).  sign -1: forward, +1: inverse (unscaled).
cudaError_t fft_pow2(double2* buf, double2* tmp, int64_t n, int sign, double2** result, cudaStream_t stream) {
  double2* a = buf;
  double2* b = tmp;
  for (int64_t ns = 1; ns < n; ns <<= 1) {
    fft_stockham_pass<<<grid_for(n / 2), 256, 0, stream>>>(a, b, n, ns, (double)sign);
    double2* t = a;
    a = b;
    b = t;
  }
  *result = a;
  return cudaGetLastError();
}

cudaError_t launch_cmul(double2* a, const double2* b, int64_t n, double scale, cudaStream_t stream) {
  cmul_inplace<<<grid_for(n), 256, 0, stream>>>(a, b, n, scale);
  return cudaGetLastError();
}

// z -> z^h per bin by binary exponentiation (kernel_power's spectrum power,
// fft.py:255 `rfft(padded) ** h`), then the inverse transform's 1/N folded in.
__global__ void cpow_inplace(double2* __restrict__ a, int64_t n, int64_t h, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 base = a[i], acc = make_double2(1.0, 0.0);
    for (int64_t e = h; e > 0; e >>= 1) {
      if (e & 1) acc = cmul(acc, base);
      if (e > 1) base = cmul(base, base);
    }
    a[i] = make_double2(acc.x * scale, acc.y * scale);
  }
}

cudaError_t launch_cpow(double2* a, int64_t n, int64_t h, double scale, cudaStream_t stream) {
  cpow_inplace<<<grid_for(n), 256, 0, stream>>>(a, n, h, scale);
  return cudaGetLastError();
}

cudaError_t launch_cscale(double2* a, int64_t n, double scale, cudaStream_t stream) {
  cscale_inplace<<<grid_for(n), 256, 0, stream>>>(a, n, scale);
  return cudaGetLastError();
}

}  // namespace fl
