// fl_conv.cuh -- fp64 valid-mode correlation with a composed stencil power,
// executed by a thread group (one warp, the worker warps of a warp-specialised
// CTA, or a whole CTA).
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
//    Real-to-complex packing (N real = N/2 complex).  The complex transform is
//    in place: decimation-in-frequency radix-16 stages forward (natural ->
//    digit-reversed), decimation-in-time stages back (digit-reversed ->
//    natural), so no reordering pass exists and any number of threads can
//    share a stage (each butterfly writes back to the slots it read).  The
//    real split, spectrum multiply and inverse re-pack are one fused pass over
//    digit-reversed slots.  Twiddles come from a quarter-wave fp64 table.
//  * conv_direct -- small kernels: explicit dot products against cached
//    real-space weights (built once per option and height by conv_fft on a
//    delta), shared-memory staged.
#pragma once

#include "fl_common.cuh"

namespace fl {

constexpr int CTA_THREADS = 256;

#ifndef FL_FFT_T  // phase timing hook (tools/fft_task_bench.cu)
#define FL_FFT_T(k)
#endif
#ifndef FL_ASYNC_LOAD  // 1: conv_fft stages its block with cp.async (no register staging)
#define FL_ASYNC_LOAD 1
#endif
#ifndef FL_SPEC_SKIP  // 1: bin pairs whose spectrum values are both cut skip the split / multiply / re-pack
#define FL_SPEC_SKIP 1
#endif

// A cooperating thread group: index t in [0, n); bar >= 0 -> named barrier,
// bar < 0 -> the group is one warp (n == 32).
struct Grp {
  int t, n, bar;
};

__device__ __forceinline__ void gsync(const Grp& g) {
  if (g.bar < 0) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(g.bar), "r"(g.n) : "memory");
  }
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

// ---------------------------------------------------------------------------
// In-place mixed-radix transform of C = 2^logC complex points.  Stage radices:
// 16, 16, ..., then 2/4/8 for the remainder (last DIF stage, smallest span).

// w[q] = w1^q, q = 1..R-1, by a product tree of depth log2(R) (one table
// lookup per butterfly: strided table reads are heavily bank-conflicted).
template <int R>
__device__ __forceinline__ void tw_powers(double2 w1, double2 (&w)[R]) {
  w[1] = w1;
#pragma unroll
  for (int q = 2; q < R; ++q) w[q] = cmul(w[q / 2], w[q - q / 2]);
}


// DIF stage of radix R on spans of S = 2^logS points.
template <int R>
__device__ __forceinline__ void dif_stage(double2* buf, int logC, int logS, const double2* tq, const Grp& g) {
  constexpr int LR = (R == 2) ? 1 : (R == 4) ? 2 : (R == 8) ? 3 : 4;
  const int nb = 1 << (logC - LR);
  const int lstride = logS - LR;  // stride = S / R
  const int jmask = (1 << lstride) - 1;
  const int tshift = TW_LOG - logS;
#pragma unroll 1
  for (int u = g.t; u < nb; u += g.n) {
    const int j = u & jmask;
    const int base = ((u >> lstride) << logS) + j;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = buf[pidx(base + (r << lstride))];
    fft_reg<R>(v);
    double2 w[R];
    tw_powers<R>(twq(tq, j << tshift), w);
#pragma unroll
    for (int q = 1; q < R; ++q) v[q] = cmul(v[q], w[q]);
#pragma unroll
    for (int q = 0; q < R; ++q) buf[pidx(base + (q << lstride))] = v[q];
  }
  gsync(g);
}

// Inverse (DIT) stage: undoes dif_stage<R> up to the factor R.
template <int R>
__device__ __forceinline__ void dit_stage(double2* buf, int logC, int logS, const double2* tq, const Grp& g) {
  constexpr int LR = (R == 2) ? 1 : (R == 4) ? 2 : (R == 8) ? 3 : 4;
  const int nb = 1 << (logC - LR);
  const int lstride = logS - LR;
  const int jmask = (1 << lstride) - 1;
  const int tshift = TW_LOG - logS;
#pragma unroll 1
  for (int u = g.t; u < nb; u += g.n) {
    const int j = u & jmask;
    const int base = ((u >> lstride) << logS) + j;
    double2 v[R];
    // IDFT(conj-twiddled x) = conj(DFT(conj(x conj(w)))) = conj(DFT(conj(x) w))
    double2 w[R];
    tw_powers<R>(twq(tq, j << tshift), w);
    v[0] = cconj(buf[pidx(base)]);
#pragma unroll
    for (int q = 1; q < R; ++q) v[q] = cmul(cconj(buf[pidx(base + (q << lstride))]), w[q]);
    fft_reg<R>(v);
#pragma unroll
    for (int r = 0; r < R; ++r) buf[pidx(base + (r << lstride))] = cconj(v[r]);
  }
  gsync(g);
}

// Stage plan of a C = 2^logC transform: radix-16 stages from the largest span
// down, then (if 4 does not divide logC) one remainder stage of radix 2^last.
// Computed from logC in registers (a stage array in local memory cost a local
// load per stage and four per spectrum bin pair).  (Measured alternative:
// radix 4/8 stages keeping every group thread busy -- slower, N = 1024 task
// 9.9k -> 13.2k cycles, profiles/r01_experiments.md.)
struct FftPlan {
  int n16;   // radix-16 stages
  int n8;    // radix-8 stages after them (small transforms only, else 0)
  int last;  // log2 radix of the remainder stage (0: none, else 1..3)
};
#ifndef FL_FFT_R8  // 1: transforms with fewer radix-16 butterflies than group threads use radix-8 stages
#define FL_FFT_R8 1
#endif
#ifndef FL_FFT_R8_K
#define FL_FFT_R8_K 16
#endif
// A radix-16 stage of C points has C/16 butterflies: below 2048 points a
// 128-thread group runs them on one or two warps, i.e. on one or two SMSPs'
// FP64 pipes while the others idle (a radix-16 butterfly is ~300 FP64
// instructions).  Such transforms (the small ring's h = 256 / 512 jumps: 512
// and 1024 complex points) run radix-8 stages instead (C/8 butterflies of ~120
// instructions), then a radix-2 / 4 remainder.
__device__ __forceinline__ FftPlan fft_plan(int logC, int gn) {
  FftPlan p;
#if FL_FFT_R8
  if (logC >= 6 && (FL_FFT_R8_K << logC) < (gn << 8)) {  // C / 16 < gn (K = 32: gn / 2, measured slower)
    p.n16 = 0;
    p.n8 = logC / 3;
    p.last = logC - 3 * p.n8;
    return p;
  }
#endif
  p.n8 = 0;
  p.last = logC & 3;
  p.n16 = logC >> 2;
  return p;
}

// remainder stage: radix 2, 4 or 8 (each radix has one call site per
// direction: the instruction footprint counts); the radix-8 case also runs the
// n8 main stages of a small transform, `n` stages with spans stepping by 8
template <bool DIF>
__device__ __forceinline__ void fft_stage_rem(double2* buf, int lr, int logC, int logS, const double2* tq,
                                              const Grp& g, int n = 1) {
  switch (lr) {
    case 1: DIF ? dif_stage<2>(buf, logC, logS, tq, g) : dit_stage<2>(buf, logC, logS, tq, g); break;
    case 2: DIF ? dif_stage<4>(buf, logC, logS, tq, g) : dit_stage<4>(buf, logC, logS, tq, g); break;
    default:
#pragma unroll 1
      for (int s = 0; s < n; ++s) {
        if (DIF) {
          dif_stage<8>(buf, logC, logS, tq, g);
          logS -= 3;
        } else {
          dit_stage<8>(buf, logC, logS, tq, g);
          logS += 3;
        }
      }
      break;
  }
}

// Forward: natural order in, X[k] at slot P(k) out.
__device__ __forceinline__ void fft_dif(double2* buf, int logC, const double2* tq, Grp g, const FftPlan& pl) {
  int logS = logC;
#pragma unroll 1
  for (int s = 0; s < pl.n16; ++s) {
    dif_stage<16>(buf, logC, logS, tq, g);
    logS -= 4;
  }
#if FL_FFT_R8
  // the radix-8 stages of a small transform, then the remainder (one call site)
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    const int lr = pass == 0 ? (pl.n8 ? 3 : 0) : pl.last;
    const int n = pass == 0 ? pl.n8 : 1;
    if (lr) {
      fft_stage_rem<true>(buf, lr, logC, logS, tq, g, n);
      logS -= lr * n;
    }
  }
#else
  if (pl.last) fft_stage_rem<true>(buf, pl.last, logC, logS, tq, g);
#endif
}

// Inverse (unnormalised, x C): slot P(k) in, natural order out.
__device__ __forceinline__ void fft_dit(double2* buf, int logC, const double2* tq, Grp g, const FftPlan& pl) {
#if !FL_FFT_R8
  int logS = pl.last;
  if (pl.last) fft_stage_rem<false>(buf, pl.last, logC, logS, tq, g);
#else
  int logS = 0;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {  // remainder first, then the radix-8 stages (one call site)
    const int lr = pass == 0 ? pl.last : (pl.n8 ? 3 : 0);
    const int n = pass == 0 ? 1 : pl.n8;
    if (lr) {
      fft_stage_rem<false>(buf, lr, logC, logS + lr, tq, g, n);
      logS += lr * n;
    }
  }
#endif
#pragma unroll 1
  for (int s = 0; s < pl.n16; ++s) {
    logS += 4;
    dit_stage<16>(buf, logC, logS, tq, g);
  }
}

// Slot holding frequency k after fft_dif: k's digits in stage order (the first
// stage's digit is the least significant of k) written most significant first,
// each digit's bits in place, then the remainder digit:
// slot = digit_reverse(k mod R^n) << last | k >> n log2 R  (R = 16 or 8).
__device__ __forceinline__ int slot_of(int k, int logC, const FftPlan& pl) {
  if (FL_FFT_R8 && pl.n8) {
    const int lo = 3 * pl.n8;
    unsigned x = __brev((unsigned)k & ((1u << lo) - 1u)) >> (32 - lo);  // bit-reversed: digits reversed, each inside out
    x = (x & 0x92492492u) | ((x & 0x49249249u) << 2) | ((x >> 2) & 0x49249249u);
    return (int)((x << pl.last) | ((unsigned)k >> lo));
  }
  const int lo = 4 * pl.n16;
  unsigned x = __brev((unsigned)k & ((1u << lo) - 1u));  // bit-reversed, nibbles internally reversed
  x = ((x & 0x33333333u) << 2) | ((x >> 2) & 0x33333333u);
  x = ((x & 0x55555555u) << 1) | ((x >> 1) & 0x55555555u);
  x = lo ? (x >> (32 - lo)) : 0u;
  return (int)((x << pl.last) | ((unsigned)k >> lo));
}

// ---------------------------------------------------------------------------
// composed-stencil description and the per-task window plan

struct Stencil {
  double c0, c1, c2;  // P(z) = c0 + c1 z + c2 z^2 (c2 = 0 for two taps)
  int span;           // taps - 1
  int hsmall = 0;     // chains: tallest kernel whose window fits the small ring (0: not set, see fft_ring)
};

struct ConvPlan {
  int64_t rlo;  // first kernel index kept in the window
  int64_t P;    // valid outputs per block
  int logN;     // real block size N = 2^logN
  double tau;   // |P(e^{i th})|^2 below tau -> |P|^h < 1e-24 -> bin zeroed
};

constexpr double LN_2_OVER_EPS = 50.656872045869936;  // ln(2 / 2e-22)

// Hoeffding window width Mw of W_h (rlo/rhi clamped to [0, M-1]).
__host__ __device__ inline int64_t window_width(const Stencil& st, int h, int64_t* rlo_out) {
  const int64_t M = (int64_t)h * st.span + 1;
  const double mass = st.c0 + st.c1 + st.c2;
  const double mu = (double)h * (st.c1 + 2.0 * st.c2) / mass;
  const double t = (double)st.span * sqrt(0.5 * (double)h * LN_2_OVER_EPS);
  int64_t rlo = (int64_t)floor(mu - t) - 1;
  int64_t rhi = (int64_t)ceil(mu + t) + 1;
  if (rlo < 0) rlo = 0;
  if (rhi > M - 1) rhi = M - 1;
  if (rlo_out) *rlo_out = rlo;
  return rhi - rlo + 1;
}

// Window + block plan for one task; uniform across the group (every thread computes it).
__device__ __forceinline__ ConvPlan plan_conv(const Stencil& st, int h, int64_t Lout, int logNmax) {
  ConvPlan p;
  int64_t rlo;
  const int64_t Mw = window_width(st, h, &rlo);
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
// values.  buf: smem_complex_slots(2^(logNmax-1)) double2; tq: quarter-wave
// twiddle table (shared or global).  Returns the executed fp64 flops (FFT
// convention 5 C log2 C per complex transform, two per block, plus 16 C for
// the split / spectrum / re-pack pass); -1 if the window exceeds the block.
__device__ double conv_fft(const double* __restrict__ x, int64_t L, double* __restrict__ y, int64_t Lout, int h,
                           const Stencil& st, double2* buf, int logNmax, const double2* tq, const Grp& g) {
  if (Lout <= 0) return 0.0;
  const ConvPlan pl = plan_conv(st, h, Lout, logNmax);
  if (pl.P < 1) return -1.0;
  const int logN = pl.logN;
  const int logC = logN - 1;
  const int C = 1 << logC;
  const int N = 1 << logN;
  const int tsh = TW_LOG - logN;  // W_N^k = twq(k << tsh)
  const double inv_c = 1.0 / (double)C;
  const int64_t rlo_modN = pl.rlo & (N - 1);
  const double rlo_sign = (pl.rlo & 1) ? -1.0 : 1.0;
  const int64_t nblk = (Lout + pl.P - 1) / pl.P;
  const FftPlan fp = fft_plan(logC, g.n);

  for (int64_t k0 = 0; k0 < Lout; k0 += pl.P) {
    FL_FFT_T(4);
    // -- load packed pairs z[n] = x[s+2n] + i x[s+2n+1]
    const int64_t s0 = k0 + pl.rlo;
#if FL_ASYNC_LOAD
    // asynchronous 8-byte copies global -> shared (zero-filled past L): every
    // load of the block is in flight at once and none holds a register (the
    // register-staged pass waited one L2 round trip per 4 elements per thread)
    for (int n = g.t; n < C; n += g.n) {
      const int64_t i0 = s0 + 2 * (int64_t)n;
      double* d = reinterpret_cast<double*>(buf + pidx(n));
      const unsigned da = (unsigned)__cvta_generic_to_shared(d);
      const int sa = (i0 < L) ? 8 : 0, sb = (i0 + 1 < L) ? 8 : 0;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(da), "l"(x + (sa ? i0 : 0)), "r"(sa) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(da + 8), "l"(x + (sb ? i0 + 1 : 0)), "r"(sb)
                   : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#else
#pragma unroll 4
    for (int n = g.t; n < C; n += g.n) {
      const int64_t i0 = s0 + 2 * (int64_t)n;
      const double a = (i0 < L) ? x[i0] : 0.0;
      const double b = (i0 + 1 < L) ? x[i0 + 1] : 0.0;
      buf[pidx(n)] = make_double2(a, b);
    }
#endif
    gsync(g);
    FL_FFT_T(0);
    fft_dif(buf, logC, tq, g, fp);
    FL_FFT_T(1);
    // -- split to the real spectrum, multiply, re-pack for the inverse (/C)
    // W_N^k and the window phase W_N^(k rlo) advance by fixed steps per iteration
    // (one table lookup each instead of conflicted strided lookups per bin)
    double2 Wk = twq(tq, (g.t & (N - 1)) << tsh);
    double2 ph = twq(tq, (int)(((int64_t)g.t * rlo_modN) & (N - 1)) << tsh);
    const double2 Wstep = twq(tq, (g.n & (N - 1)) << tsh);
    const double2 phstep = twq(tq, (int)(((int64_t)g.n * rlo_modN) & (N - 1)) << tsh);
#pragma unroll 1
    for (int k = g.t; k <= C / 2; k += g.n) {
      const int kc = (C - k) & (C - 1);
      const int pk = slot_of(k, logC, fp), pc = slot_of(kc, logC, fp);
#if FL_SPEC_SKIP
      {  // both spectrum values below the 1e-24 cut: the bin pair is zero, skip its loads and math
        const double2 omk = cconj(Wk), omc = make_double2(-Wk.x, -Wk.y);
        const double2 omk2 = cmul(omk, omk), omc2 = cmul(omc, omc);
        const double2 bk = make_double2(st.c0 + st.c1 * omk.x + st.c2 * omk2.x, st.c1 * omk.y + st.c2 * omk2.y);
        const double2 bc = make_double2(st.c0 + st.c1 * omc.x + st.c2 * omc2.x, st.c1 * omc.y + st.c2 * omc2.y);
        if (cnorm2(bk) < pl.tau && cnorm2(bc) < pl.tau) {
          buf[pidx(pk)] = make_double2(0.0, 0.0);
          if (k != 0 && k != C / 2) buf[pidx(pc)] = make_double2(0.0, 0.0);
          Wk = cmul(Wk, Wstep);
          ph = cmul(ph, phstep);
          continue;
        }
      }
#endif
      const double2 Zk = buf[pidx(pk)];
      const double2 Zc = buf[pidx(pc)];
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
      const double2 ph_c = cscale(cconj(ph), rlo_sign);
      const double2 Hk = spectrum(st, cconj(Wk), ph, h, pl.tau, inv_c);
      const double2 Hc = spectrum(st, make_double2(-Wk.x, -Wk.y), ph_c, h, pl.tau, inv_c);
      const double2 Yk = cmul(Xk, Hk);
      const double2 Yc = cmul(Xc, Hc);
      // A = Yk + conj(Yc), B = Yk - conj(Yc); Zp[k] = (A + i conj(Wk) B)/2, Zp[C-k] = conj((A - i conj(Wk) B)/2)
      const double2 A = make_double2(Yk.x + Yc.x, Yk.y - Yc.y);
      const double2 B = make_double2(Yk.x - Yc.x, Yk.y + Yc.y);
      const double2 cWB = cmul(cconj(Wk), B);
      const double2 iCWB = make_double2(-cWB.y, cWB.x);
      buf[pidx(pk)] = cscale(cadd(A, iCWB), 0.5);
      if (k != 0 && k != C / 2) buf[pidx(pc)] = cconj(cscale(csub(A, iCWB), 0.5));
      Wk = cmul(Wk, Wstep);
      ph = cmul(ph, phstep);
    }
    gsync(g);
    FL_FFT_T(2);
    fft_dit(buf, logC, tq, g, fp);
    FL_FFT_T(3);
    // -- store valid outputs: y[2n] = Re, y[2n+1] = Im
    const int64_t lim = (Lout - k0 < pl.P) ? (Lout - k0) : pl.P;
#pragma unroll 4
    for (int n = g.t; n < C; n += g.n) {
      const double2 v = buf[pidx(n)];
      const int64_t j = 2 * (int64_t)n;
      if (j < lim) y[k0 + j] = v.x;
      if (j + 1 < lim) y[k0 + j + 1] = v.y;
    }
    gsync(g);
    FL_FFT_T(5);
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
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (k < Lout) {
      const double* xk = sx + k;
      int r = sub;
#pragma unroll 2
      for (; r + 3 * G < M; r += 4 * G) {
        a0 = fma(sw[r], xk[r], a0);
        a1 = fma(sw[r + G], xk[r + G], a1);
        a2 = fma(sw[r + 2 * G], xk[r + 2 * G], a2);
        a3 = fma(sw[r + 3 * G], xk[r + 3 * G], a3);
      }
      for (; r < M; r += G) a0 = fma(sw[r], xk[r], a0);
    }
    double s = (a0 + a1) + (a2 + a3);
    for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (k < Lout && sub == 0) y[k] = s;
  }
  gsync(g);
  return 2.0 * (double)Lout * (double)M;
}

}  // namespace fl
