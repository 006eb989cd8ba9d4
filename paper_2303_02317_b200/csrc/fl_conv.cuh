// fl_conv.cuh -- fp64 valid-mode correlation with a composed stencil power,
// executed by a thread group (a whole CTA, or the worker warps of a
// warp-specialised CTA).
//
// Replaces the reference's `convolve` / `_valid_corr` / `kernel_power`
// (fft.py:130-163, 203-260; american.py:180-184; bsm.py:384-387):
//
//     y[k] = sum_{r=0}^{M-1} W_h[r] x[k+r],   k = 0 .. L-M,   M = h*span+1,
//
// where W_h are the coefficients of P(z)^h, P(z) = c0 + c1 z (+ c2 z^2).
//
// Two executors:
//  * conv_fft -- overlap-save real FFT blocks staged in shared memory.  The
//    composed kernel is never materialised: its spectrum on each block's own
//    grid is P(e^{i theta})^h, evaluated by binary exponentiation only where
//    |P|^h > 1e-24 (a few percent of the bins for large h; the rest are exact
//    zeros).  Because W_h is a (scaled) lattice-walk law, all but <= 2e-22 of
//    its mass lies in a Hoeffding window of half-width span*sqrt(h ln(2/eps)/2)
//    about its mean, so a block of N real points yields N - Mw + 1 valid
//    outputs with Mw ~ 20 sqrt(h) instead of 2h+1: every block fits in shared
//    memory and nothing is padded to next_pow2(L+M-1).  The dropped tail is
//    < 1e-21 of max|x|, far below the reference FFT's own ~1e-16 rounding.
//    Real-to-complex packing (N real = N/2 complex); in-place Stockham radix-16
//    passes in registers over a padded (bank-conflict-free) shared layout;
//    twiddles from a global fp64 table; the real split, spectrum multiply and
//    inverse pre-twist are one fused shared-memory pass.
//  * conv_direct -- small kernels (h <= DIRECT_H): explicit dot products
//    against cached real-space weights (built once per option and height by
//    conv_fft on a delta), shared-memory staged.
#pragma once

#include "fl_common.cuh"

namespace fl {

constexpr int CTA_THREADS = 256;

// A cooperating thread group: index t in [0, n), named barrier `bar`.
struct Grp {
  int t, n, bar;
};

__device__ __forceinline__ void gsync(const Grp& g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g.bar), "r"(g.n) : "memory");
}

// padded shared-memory index: one spare slot every 16 complex values
__device__ __forceinline__ int pidx(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int smem_complex_slots(int c) { return c + (c >> 4) + 1; }

// ---------------------------------------------------------------------------
// in-register radix-R DFT (forward, exp(-2 pi i / R)), natural order in/out

__device__ __forceinline__ double2 tw16(double2 d, int a16) {
  // d * exp(-2 pi i a16 / 16); a16 is a compile-time constant after unrolling
  constexpr double C1 = 0.92387953251128673848, S1 = 0.38268343236508978178;
  constexpr double R2 = 0.70710678118654752440;
  switch (a16) {
    case 0: return d;
    case 4: return make_double2(d.y, -d.x);
    case 2: return make_double2((d.x + d.y) * R2, (d.y - d.x) * R2);
    case 6: return make_double2((d.y - d.x) * R2, -(d.x + d.y) * R2);
    case 1: return make_double2(fma(d.x, C1, d.y * S1), fma(d.y, C1, -d.x * S1));
    case 3: return make_double2(fma(d.x, S1, d.y * C1), fma(d.y, S1, -d.x * C1));
    case 5: return make_double2(fma(-d.x, S1, d.y * C1), fma(-d.y, S1, -d.x * C1));
    default: return make_double2(fma(-d.x, C1, d.y * S1), fma(-d.y, C1, -d.x * S1));  // 7
  }
}

__host__ __device__ constexpr int brev(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}

template <int R>
__device__ __forceinline__ void fft_reg(double2 (&v)[R]) {
  constexpr int LOGR = (R == 2) ? 1 : (R == 4) ? 2 : (R == 8) ? 3 : 4;
#pragma unroll
  for (int half = R / 2; half >= 1; half >>= 1) {
#pragma unroll
    for (int s = 0; s < R; s += 2 * half) {
#pragma unroll
      for (int k = 0; k < half; ++k) {
        double2 a = v[s + k], b = v[s + k + half];
        v[s + k] = cadd(a, b);
        v[s + k + half] = tw16(csub(a, b), k * (16 / (2 * half)));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int r = brev(i, LOGR);
    if (i < r) {
      double2 t = v[i];
      v[i] = v[r];
      v[r] = t;
    }
  }
}

// One in-place Stockham DIT pass of radix R over C complex points (C/R <= g.n).
template <int R>
__device__ __forceinline__ void stockham_pass(double2* buf, int C, int Ns, int logNsR, const Grp& g) {
  const int nb = C / R;
  const int j = g.t;
  double2 v[R];
  const bool act = j < nb;
  if (act) {
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = buf[pidx(j + r * nb)];
    const int k = j & (Ns - 1);
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw_l(r * k, logNsR));
    }
    fft_reg<R>(v);
  }
  gsync(g);
  if (act) {
    const int k = j & (Ns - 1);
    const int d = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[pidx(d + r * Ns)] = v[r];
  }
  gsync(g);
}

// Forward complex FFT of C = 2^logC points (32 <= C <= 16 * g.n), in place, natural order.
__device__ __noinline__ void fft_grp(double2* buf, int logC, Grp g) {
  const int C = 1 << logC;
  int rem = logC % 4;
  int Ns = 1, logNs = 0;
  if (rem == 1) { stockham_pass<2>(buf, C, Ns, logNs + 1, g); Ns <<= 1; logNs += 1; }
  else if (rem == 2) { stockham_pass<4>(buf, C, Ns, logNs + 2, g); Ns <<= 2; logNs += 2; }
  else if (rem == 3) { stockham_pass<8>(buf, C, Ns, logNs + 3, g); Ns <<= 3; logNs += 3; }
  while (logNs < logC) {
    stockham_pass<16>(buf, C, Ns, logNs + 4, g);
    Ns <<= 4;
    logNs += 4;
  }
}

// ---------------------------------------------------------------------------
// composed-stencil description and the per-task window plan

struct Stencil {
  double c0, c1, c2;  // P(z) = c0 + c1 z + c2 z^2 (c2 = 0 for two taps)
  int span;           // taps - 1
};

struct ConvPlan {
  int64_t rlo;     // first kernel index kept in the window
  int64_t P;       // valid outputs per block
  int logN;        // real block size N = 2^logN
  double tau;      // |P(e^{i th})|^2 below tau -> |P|^h < 1e-24 -> bin zeroed
};

constexpr double LN_2_OVER_EPS = 50.656872045869936;  // ln(2 / 2e-22)

// Window + block plan for one task; uniform across the group (every thread computes it).
__device__ __forceinline__ ConvPlan plan_conv(const Stencil& st, int h, int64_t Lout, int logNmax) {
  ConvPlan p;
  const int64_t M = (int64_t)h * st.span + 1;
  const double mass = st.c0 + st.c1 + st.c2;
  const double mu = (double)h * (st.c1 + 2.0 * st.c2) / mass;
  const double t = (double)st.span * sqrt(0.5 * (double)h * LN_2_OVER_EPS);
  int64_t rlo = (int64_t)floor(mu - t) - 1;
  int64_t rhi = (int64_t)ceil(mu + t) + 1;
  if (rlo < 0) rlo = 0;
  if (rhi > M - 1) rhi = M - 1;
  const int64_t Mw = rhi - rlo + 1;
  const int64_t need = Lout + Mw - 1;
  int logN = 6;
  while (logN < logNmax && ((int64_t)1 << logN) < need) ++logN;
  p.rlo = rlo;
  p.logN = logN;
  p.P = ((int64_t)1 << logN) - Mw + 1;
  // |P|^h < 1e-24  <=>  |P|^2 < 1e-48^(1/h)
  p.tau = exp(-110.52408446371488 / (double)h);
  return p;
}

__device__ __forceinline__ double2 cpow_int(double2 b, int e) {
  double2 r = make_double2(1.0, 0.0);
#pragma unroll 1
  while (e) {
    if (e & 1) r = cmul(r, b);
    e >>= 1;
    if (e) b = cmul(b, b);
  }
  return r;
}

// Spectrum value at omega = exp(+i theta), times the window phase and 1/C.
__device__ __forceinline__ double2 spectrum(const Stencil& st, double2 om, double2 phase, int h,
                                            double tau, double inv_c) {
  double2 om2 = cmul(om, om);
  double2 base = make_double2(st.c0 + st.c1 * om.x + st.c2 * om2.x, st.c1 * om.y + st.c2 * om2.y);
  if (cnorm2(base) < tau) return make_double2(0.0, 0.0);
  return cscale(cmul(cpow_int(base, h), phase), inv_c);
}

// ---------------------------------------------------------------------------
// FFT executor.  y[k] = sum_r W_h[r] x[k+r], k in [0, Lout); x has L >= Lout + h*span
// values.  buf: smem_complex_slots(2^(logNmax-1)) double2.  Returns the executed
// fp64 flops (FFT convention 5 C log2 C per complex transform, two per block,
// plus 16 C for the split / spectrum / re-pack pass).  P < 1 (window wider
// than the largest block) returns -1.
__device__ double conv_fft(const double* __restrict__ x, int64_t L, double* __restrict__ y, int64_t Lout, int h,
                           const Stencil& st, double2* buf, int logNmax, const Grp& g) {
  if (Lout <= 0) return 0.0;
  const ConvPlan pl = plan_conv(st, h, Lout, logNmax);
  if (pl.P < 1) return -1.0;
  const int logN = pl.logN;
  const int logC = logN - 1;
  const int C = 1 << logC;
  const int N = 1 << logN;
  const double inv_c = 1.0 / (double)C;
  const int64_t rlo_modN = pl.rlo & (N - 1);
  const double rlo_sign = (pl.rlo & 1) ? -1.0 : 1.0;
  const int64_t nblk = (Lout + pl.P - 1) / pl.P;

  for (int64_t k0 = 0; k0 < Lout; k0 += pl.P) {
    // -- load packed pairs z[n] = x[s+2n] + i x[s+2n+1]
    const int64_t s0 = k0 + pl.rlo;
#pragma unroll 1
    for (int n = g.t; n < C; n += g.n) {
      const int64_t i0 = s0 + 2 * (int64_t)n;
      const double a = (i0 < L) ? x[i0] : 0.0;
      const double b = (i0 + 1 < L) ? x[i0 + 1] : 0.0;
      buf[pidx(n)] = make_double2(a, b);
    }
    gsync(g);
    fft_grp(buf, logC, g);
    // -- split to the real spectrum, multiply, re-pack for the inverse (conjugated, /C)
#pragma unroll 1
    for (int k = g.t; k <= C / 2; k += g.n) {
      const int kc = (C - k) & (C - 1);
      const double2 Zk = buf[pidx(k)];
      const double2 Zc = buf[pidx(kc)];
      const double2 Wk = tw_l(k, logN);  // exp(-2 pi i k / N)
      const double2 E = make_double2(0.5 * (Zk.x + Zc.x), 0.5 * (Zk.y - Zc.y));
      const double2 D = make_double2(Zk.x - Zc.x, Zk.y + Zc.y);  // Zk - conj(Zc)
      const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);     // D / (2i)
      const double2 WO = cmul(Wk, O);
      double2 Xk = cadd(E, WO);
      double2 Xc = cconj(csub(E, WO));
      if (k == 0) {  // X[0] and X[C] are real
        Xk = make_double2(Zk.x + Zk.y, 0.0);
        Xc = make_double2(Zk.x - Zk.y, 0.0);
      }
      // spectrum at omega_k = conj(Wk), omega_{C-k} = -Wk; window phase W^{k rlo}
      const int64_t ph_idx = ((int64_t)k * rlo_modN) & (N - 1);
      const double2 ph = tw_l((int)ph_idx, logN);
      const double2 Hk = spectrum(st, cconj(Wk), ph, h, pl.tau, inv_c);
      const double2 ph_c = cscale(cconj(ph), rlo_sign);
      const double2 Hc = spectrum(st, make_double2(-Wk.x, -Wk.y), ph_c, h, pl.tau, inv_c);
      const double2 Yk = cmul(Xk, Hk);
      const double2 Yc = cmul(Xc, Hc);
      // A = Yk + conj(Yc), B = Yk - conj(Yc); Zp[k] = (A + i conj(Wk) B)/2
      const double2 A = make_double2(Yk.x + Yc.x, Yk.y - Yc.y);
      const double2 B = make_double2(Yk.x - Yc.x, Yk.y + Yc.y);
      const double2 cWB = cmul(cconj(Wk), B);
      const double2 iCWB = make_double2(-cWB.y, cWB.x);
      const double2 Zpk = cscale(cadd(A, iCWB), 0.5);
      buf[pidx(k)] = cconj(Zpk);
      if (k != 0 && k != C / 2) buf[pidx(kc)] = cscale(csub(A, iCWB), 0.5);  // conj(Zp[C-k])
    }
    gsync(g);
    fft_grp(buf, logC, g);
    // -- store valid outputs: y[2n] = Re, y[2n+1] = -Im
    const int64_t lim = (Lout - k0 < pl.P) ? (Lout - k0) : pl.P;
#pragma unroll 1
    for (int n = g.t; n < C; n += g.n) {
      const double2 v = buf[pidx(n)];
      const int64_t j = 2 * (int64_t)n;
      if (j < lim) y[k0 + j] = v.x;
      if (j + 1 < lim) y[k0 + j + 1] = -v.y;
    }
    gsync(g);
  }
  return (double)nblk * (10.0 * (double)C * (double)logC + 16.0 * (double)C);
}

// ---------------------------------------------------------------------------
// Direct executor for small kernels.  wrev[i] = W_h[M-1-i] (as conv_fft of a delta
// returns it).  Stages x and the weights in shared memory (sx holds >= L + M
// doubles).  Returns executed flops.
__device__ double conv_direct(const double* __restrict__ x, int64_t L, double* __restrict__ y, int64_t Lout,
                              const double* __restrict__ wrev, int M, double* sx, const Grp& g) {
  if (Lout <= 0) return 0.0;
  double* sw = sx + L;
  for (int i = g.t; i < L; i += g.n) sx[i] = x[i];
  for (int i = g.t; i < M; i += g.n) sw[i] = wrev[M - 1 - i];  // sw[r] = W[r]
  gsync(g);
  // G threads per output (power of two, <= 32), taps strided by G
  int G = 1;
  while (G < 32 && (int64_t)(g.n / (2 * G)) >= Lout) G <<= 1;
  const int sub = g.t & (G - 1);
  const int per = g.n / G;
  for (int64_t k0 = 0; k0 < Lout; k0 += per) {
    const int64_t k = k0 + g.t / G;
    double a0 = 0.0, a1 = 0.0;
    if (k < Lout) {
      const double* xk = sx + k;
      int r = sub;
#pragma unroll 4
      for (; r + G < M; r += 2 * G) {
        a0 = fma(sw[r], xk[r], a0);
        a1 = fma(sw[r + G], xk[r + G], a1);
      }
      if (r < M) a0 = fma(sw[r], xk[r], a0);
    }
    double s = a0 + a1;
    for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (k < Lout && sub == 0) y[k] = s;
  }
  gsync(g);
  return 2.0 * (double)Lout * (double)M;
}

}  // namespace fl
