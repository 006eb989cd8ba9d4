// fl_put.cu -- American put on the anchored BSM grid: device divide-and-conquer
// (replaces bsm.fast_put_bsm and its recursion, bsm.py:402-713, and
// bsm.solve_bsm_trapezoid, bsm.py:504-582) and the O(T^2) projected march
// (replaces bsm.baseline_put_fd / _accel.put_march_window, bsm.py:273-338,
// _accel.py:163-200).
//
// Fast path: the persistent warp-specialised CTA of fl_sched.cuh.  Each chain
// warp prices one option at a time, pulled from a global queue in
// decreasing-cost order:
//   * the stage loop (bsm.py:639-665) and the _solve_q halving recursion
//     (bsm.py:443-501) run on the chain warp with an explicit stack;
//   * leaves (h <= PUT_LEAF: the reference's _strip_advance /
//     bsm_strip_sweep) run on the chain warp, in registers with shuffles;
//   * nodes with h <= FUSE_H run whole on the chain warp in shared memory
//     (mid jump, leaf, bottom jump, leaf: no round trip through L2);
//   * every longer linear jump (far / mid / bottom) is a worker task;
//   * the apex finish (bsm.py:679-713) is a worker task over shared memory.
// Row data live in a per-chain HBM arena, column-indexed, so the reference's
// concatenations (upper|mid, lower|bottom, near|far) are free.
//
// Work accounting: besides the executed flops, every chain adds the
// REFERENCE-ALGORITHMIC flops of its option (the reference's decomposition
// at its base_cutoff: 5 flops per projected cell of each reference strip,
// 5 N log2 N + 6 (N/2+1) per reference FFT jump of size N = next_pow2(L+M-1),
// SURVEY 8(d)).  That is the numerator of the reported roofline fraction.
#include <cstdint>

#include "fl_common.cuh"
#include "fl_conv.cuh"
#include "fl_kernels.h"
#include "fl_sched.cuh"
#include "fl_strip.cuh"
#include "host_params.h"

namespace fl {

#ifndef FL_PUT_LEAF
#define FL_PUT_LEAF 64
#endif
// leaf strip heights: the sliding 2h+2 frame (options with the exercise
// margin, PutParams::slide) and the full 4h+2 frame (the others; CPL 9 at 64)
constexpr int PUT_LEAF = FL_PUT_LEAF;
constexpr int PUT_LEAF_FULL = PUT_LEAF < 64 ? PUT_LEAF : 64;
constexpr int PUT_CPL = (4 * PUT_LEAF_FULL + 2 + 31) / 32;  // cells per lane in a full-frame leaf strip
constexpr int PUT_SLIDE_CPL = (2 * PUT_LEAF + 2 + 30) / 31;  // cells per lane (lane 0 is the ghost lane)
constexpr int PUT_SLIDE_H = (31 * PUT_SLIDE_CPL - 2) / 2;      // tallest strip the frame holds
template <int SL>
__host__ __device__ constexpr int put_leaf_h() { return SL == 1 ? PUT_LEAF : PUT_LEAF_FULL; }
#ifndef FL_LOW_H  // mid / bottom jumps of kernel height >= FL_LOW_H go to the chunked low-priority ring (0: none)
#define FL_LOW_H 4096
#endif
#ifndef FL_PUT_HS
#define FL_PUT_HS 256
#endif
// recursion subtrees of height <= PUT_HS run whole in the chain's shared memory
constexpr int PUT_HS = FL_PUT_HS;
constexpr int PUT_MARGIN = 2 * PUT_HS + 32;  // columns below the lowest boundary kept in the stage buffers
constexpr int PUT_MAX_DEPTH = 24;
// shared layout of a subtree: payoff (4 HS + 2) | input row (2 HS) | assembled rows of depth
// 0, 1, 2 (2 HS, HS, HS / 2)
constexpr int SUB_PAY = 0;
constexpr int SUB_IN = SUB_PAY + 4 * PUT_HS + 8;
constexpr int SUB_ASM0 = SUB_IN + 2 * PUT_HS + 8;
constexpr int SUB_ASM1 = SUB_ASM0 + 2 * PUT_HS + 8;
constexpr int SUB_ASM2 = SUB_ASM1 + PUT_HS + 8;
constexpr int SUB_END = SUB_ASM2 + PUT_HS / 2 + 8;
constexpr int SUB_DEPTH = 5;
static_assert(SUB_END <= CHAIN_SCRATCH, "subtree scratch");
static_assert(PUT_HS <= 8 * PUT_LEAF_FULL, "three asm levels cover a subtree");
static_assert(PUT_HS / 2 <= KT_H, "subtree correlations use the kernel table");
static_assert(2 * (2 * KT_H + 2) <= CHAIN_SCRATCH, "kernel-table scratch");

enum : int { TK_PUT_INIT = TK_USER + 0, TK_PUT_APEX = TK_USER + 1, TK_PUT_LOAD = TK_USER + 2 };

// reference-algorithmic cost model.  Exact integers, kept in
// 64-bit integer registers on the chain (fp64 conversions and dependent adds on
// the chain's critical path measured ~6 % of the headline run).
__device__ __forceinline__ uint64_t ref_jump_flops(int64_t L, int64_t M) {
  const uint64_t need = (uint64_t)(L + M - 1);
  const int lg = need <= 1 ? 0 : 64 - __clzll((long long)(need - 1));  // N = next_pow2(L+M-1) = 2^lg
  const uint64_t N = 1ull << lg;
  return 5ull * N * (uint64_t)lg + 3ull * N + 6ull;  // 5 N lg N + 6 (N/2 + 1)
}
// projected cells of a reference strip of width W swept `rows` times (shrinking cone)
__device__ __forceinline__ uint64_t ref_strip_flops(int64_t W, int64_t rows) {
  return 5ull * (uint64_t)(rows * W - rows * (rows + 1));
}

struct PutFrame {
  int64_t f, km;
  double* in_org;
  double* out_org;
  double* asm_org;
  int64_t arena;  // offset of this frame's assembled-row buffer in the frame arena
  int h, state;
};

// Column window of a chain's stage / payoff buffers.
struct PutLayout {
  int64_t colbase;  // lowest column held
  int64_t span;     // buffer length
};

__host__ __device__ inline PutLayout put_layout(int64_t n, int64_t ks) {
  PutLayout L;
  const int64_t lowest = (ks - n < -n ? ks - n : -n);
  L.colbase = lowest - PUT_MARGIN;
  L.span = (ks + n + 8) - L.colbase + 1;
  return L;
}

// trapezoid problem (solve_bsm_trapezoid): columns f-2h-1 .. f+W
__host__ __device__ inline PutLayout put_trap_layout(int64_t f, int64_t W, int64_t h) {
  PutLayout L;
  L.colbase = f - 2 * h - PUT_MARGIN;
  L.span = (f + W + 8) - L.colbase + 1;
  return L;
}

__host__ __device__ inline int64_t put_arena_doubles(int64_t span, int64_t n_rows) {
  return 3 * span + 2 * (2 * n_rows + 64 * PUT_MAX_DEPTH) + KTABLE_DOUBLES + 64;
}

// doubles needed per chain for a batch whose options have at most these sizes
int64_t put_ws_doubles(int64_t n_max, int64_t ks_pos_max) {
  const int64_t span = 2 * n_max + ks_pos_max + PUT_MARGIN + 16;
  return put_arena_doubles(span, n_max);
}

struct PutChainCtx {
  SchedShared* S;
  int c;
  Stencil st;
  const double* kc;  // composed weights W_1..W_DIRECT_H (slot m at kc + m*m)
  double* frames;     // two copies of the recursion-frame arena (frames, frames + fstride) ...
  int64_t fstride;
  uint32_t tog;       // ... alternated per depth, so consecutive nodes of one depth never
                      // share assembled-row memory (no false WAR dependencies between them)
  const double* pay_org;
  double* scratch;   // chain's shared scratch (CHAIN_SCRATCH doubles)
  double* wst;       // chain's weight stash (shared)
  int64_t ref_cut;   // the reference's base_cutoff (work accounting only)
  bool acct;           // count flops (accounting runs only)
  uint64_t flops;      // executed chain-side flops (lane-uniform)
  uint64_t ref_flops;  // reference-algorithmic flops (lane-uniform)
  unsigned long long* prof;
  bool pay_ready = false;  // the option's payoff table is written (see put_subtree)
  bool full = false;       // price on the full frame only (re-run after a fixed-frame miss)
};

// Reference cost of a recursion node of height h whose parent has height ph:
// the reference strips it whole if h <= cutoff (and its parent did not), else
// it issues the mid jump here and the bottom jump once km is known.
template <bool ACCT = true>
__device__ __forceinline__ void ref_node_enter(PutChainCtx& X, int h, int ph) {
  if (!ACCT || !X.acct) return;
  if (h > X.ref_cut) X.ref_flops += ref_jump_flops(2 * (int64_t)h, 2 * (int64_t)((h + 1) / 2) + 1);
  else if (ph > X.ref_cut) X.ref_flops += ref_strip_flops(4 * (int64_t)h + 2, h);
}
template <bool ACCT = true>
__device__ __forceinline__ void ref_node_bottom(PutChainCtx& X, int h, int64_t A) {
  if (!ACCT || !X.acct) return;
  if (h > X.ref_cut) X.ref_flops += ref_jump_flops(A, 2 * (int64_t)(h - (h + 1) / 2) + 1);
}


// Internal status (never reported): a fixed-frame leaf saw the exercise region
// reach its left margin; the option is priced again on the full frame.
constexpr int32_t FL_RETRY_FULL = 0x7f01;

// Leaf strip on the chain warp.  in_org / out_org / pay_org may address shared memory.
// SL: 1 the sliding / fixed frame (the caller guarantees P.slide, height <=
// PUT_SLIDE_H and hi == f + 2 height), 0 the full frame, -1 decided here.  The
// subtree walk is instantiated per strip kind so the hot walk carries one strip
// only (instruction-cache footprint).
template <bool ACCT = true, int SL = -1>
__device__ __forceinline__ int64_t put_leaf(PutChainCtx& X, const PutParams& P, const double* in_org,
                                            double* out_org, const double* pay_org, int64_t lo, int64_t hi,
                                            int64_t f, int height) {
  const long long t1 = clock64();
  long long tm[2] = {0, 0};
  FL_TR(*X.S, X.c, EV_LEAF_B, height);
  // the fixed frame when the option's exercise margin allows it (host flag PutParams::slide)
  const bool slide =
      SL == 1 || (SL < 0 && P.slide && !X.full && height <= PUT_SLIDE_H && hi == f + 2 * (int64_t)height);
  int64_t kb;
  if (slide) {
#if FL_STRIP_CLOCK  // tool builds: the strip loop's cycles alone, nothing else profiled
    kb = put_strip_fixed<PUT_SLIDE_CPL>(in_org, out_org, pay_org, f, height, P.cd, P.cm, P.cu, X.prof ? tm : nullptr);
    if (X.prof && lane_id() == 0) {
      atomicAdd(X.prof + PROF_STRIP_LOOP, (unsigned long long)tm[1]);
      atomicAdd(X.prof + PROF_STRIP_N, (unsigned long long)height);
    }
#else
    kb = put_strip_fixed<PUT_SLIDE_CPL>(in_org, out_org, pay_org, f, height, P.cd, P.cm, P.cu,
                                        FL_PROFP(X.prof) ? tm : nullptr);
#endif
    // the exercise region reached the frame's left margin: inside a subtree
    // (SL 1) the caller re-prices the option on the full frame; elsewhere the
    // full frame runs here
    if (SL != 1 && kb == FIXED_MISS)
      kb = put_strip_pipe<PUT_CPL>(in_org, out_org, pay_org, lo, hi, f, height, P.cd, P.cm, P.cu);
  } else {
    kb = put_strip_pipe<PUT_CPL>(in_org, out_org, pay_org, lo, hi, f, height, P.cd, P.cm, P.cu,
                                 FL_PROFP(X.prof) ? tm : nullptr);
  }
  FL_TR(*X.S, X.c, EV_LEAF_E, height);
  LCLK_ADD(X.prof, PROF_STRIP_CYC, clock64() - t1);
  if (FL_PROFP(X.prof) && lane_id() == 0) {
    prof_add(FL_PROFP(X.prof), PROF_STRIP_CYC, clock64() - t1);
    prof_add(FL_PROFP(X.prof), PROF_STRIP_N, height);
    prof_add(FL_PROFP(X.prof), PROF_STRIP_LOOP, tm[1]);
    prof_add(FL_PROFP(X.prof), PROF_LEAF_LOAD, tm[0] - t1);
  }
  if (ACCT && X.acct) X.flops += ref_strip_flops(hi - lo + 1, height);
  FL_TR(*X.S, X.c, EV_MARK, 1);
  return kb;
}


struct SubFrame {
  int64_t f, km;
  const double* in;
  double* out;
  double* asmo;
  int h, state, tk, tk0, q;
};

// A recursion subtree of height h0 <= PUT_HS done whole in shared memory
// (bsm.py:443-501 below this node): input cols f0+1..f0+2h0 of in_org, output
// cols kp+1..f0+h0 of out_org.  The input row and the payoff of cols
// f0-2h0-1..f0+2h0 are staged once; the chain walks the subtree running the
// leaf strips, while its helper warps run every mid / bottom correlation from
// shared memory (a node's mid overlaps its first child, its bottom its second).
// The explicit frame stack lives in shared memory (one copy per warp): frames
// in registers (a compile-time recursion) measured slower -- the live frames
// push the leaf strip into register spills.
// (instantiated with and without the flop accounting: the counting code in the
// walk costs ~5 % even when switched off at run time, so production runs use
// the ACCT = false instance and accounting runs the other)
template <bool ACCT, int SL>
__device__ int64_t put_subtree(PutChainCtx& X, const PutParams& P, int64_t f0, const double* in_org,
                               double* out_org, int h0, int ph0, int32_t* err) {
  const long long t0 = clock64();
  FL_TR(*X.S, X.c, EV_SUB_B, h0);
  double* s_pay = X.scratch + SUB_PAY;
  double* s_in = X.scratch + SUB_IN;
  const int64_t plo = f0 - 2 * (int64_t)h0 - 1;
  // once the option's payoff table is known written (the first subtree's input
  // wait covers the init task that writes it), the payoff columns and the
  // composed weights depend on nothing in flight: stage them first, so their
  // load latency overlaps the wait for the jump writing this subtree's input
  const bool early = X.pay_ready;
  if (early) {  // asynchronous copies, waited for after the input row's
    warp_stage_async(s_pay, X.pay_org + plo, 4 * h0 + 2);
    if (h0 > put_leaf_h<SL>()) stash_weights(*X.S, X.c, X.wst, X.kc, h0, put_leaf_h<SL>(), 2);
  }
  const double* pay_s = s_pay - plo;
  wait_conflicts(*X.S, X.c, U(in_org + f0 + 1), U(in_org + f0 + 2 * h0 + 1), 0, 0, U(out_org + f0 - h0),
                 U(out_org + f0 + h0 + 1));
  if (!early) {
    warp_stage_async(s_pay, X.pay_org + plo, 4 * h0 + 2);
    if (h0 > put_leaf_h<SL>()) stash_weights(*X.S, X.c, X.wst, X.kc, h0, put_leaf_h<SL>(), 2);
    X.pay_ready = true;
  }
  const long long t1 = clock64();
  FL_TR(*X.S, X.c, EV_STG_B, 0);
  warp_stage_async(s_in, in_org + f0 + 1, 2 * h0);
  warp_stage_wait();  // payoff, weights and input row: one round trip
  const long long t2 = clock64();
  FL_TR(*X.S, X.c, EV_STG_E, 0);
  long long twait = 0, tpost = 0;
  static_assert(sizeof(SubFrame) * SUB_DEPTH <= FRAME_SOLVE_OFF - FRAME_SUB_OFF, "subtree frames");
  SubFrame* stk = chain_frames<SubFrame>(X.scratch, FRAME_SUB_OFF);
  stk[0].f = f0; stk[0].h = h0; stk[0].in = s_in - (f0 + 1); stk[0].out = out_org; stk[0].state = 0;
  int sp = 1;
  int64_t ret = 0;
  // one helper post site and one wait site (the walk runs for every 256 rows:
  // its code footprint counts, see profiles/r01_experiments.md)
  while (sp > 0) {
    SubFrame& F = stk[sp - 1];
    const int h = F.h, h1 = (h + 1) / 2, h2 = h - h1;
    if (F.state == 0) {
      ref_node_enter(X, h, (sp >= 2) ? stk[sp - 2].h : ph0);
      if (h <= put_leaf_h<SL>()) {
        const int64_t kb = put_leaf<ACCT, SL>(X, P, F.in, F.out, pay_s, F.f - 2 * h - 1, F.f + 2 * h, F.f, h);
        if (kb == NONE_SEEN || kb < F.f - h || kb > F.f) {
          *err = (SL == 1 && kb == FIXED_MISS) ? FL_RETRY_FULL : FL_E_GEOMETRY | 1;
          return 0;
        }
        ret = kb;
        --sp;
        continue;
      }
      F.asmo = X.scratch + (sp == 1 ? SUB_ASM0 : sp == 2 ? SUB_ASM1 : SUB_ASM2) - (F.f - h1 + 1);
      F.q = (sp == 1) ? 1 : 0;  // the subtree root's jumps have the most slack: background ring
    } else {
      // a child finished: its boundary must stay within its height (state 1:
      // first child from f, state 2: second child from km); then the jump
      // posted before it (mid / bottom) must be complete
      const bool first = (F.state == 1);
      const int64_t fr = first ? F.f : F.km;
      const int hr = first ? h1 : h2;
      if (ret < fr - hr || ret > fr) { *err = FL_E_GEOMETRY | (first ? 2 : 3); return 0; }
      const long long tw = clock64();
      helper_wait_range(*X.S, X.c, F.q, F.tk0, F.tk);
      twait += clock64() - tw;
      if (!first) {
        --sp;
        continue;
      }
      F.km = ret;
    }
    // state 0: mid jump, cols f+h1+1 .. f+2h-h1 of row t+h1 from the 2h inputs
    // (overlaps the first child); state 1: bottom jump, cols km+h2+1 .. f+h of
    // row t+h from the assembled cols km+1 .. f+2h-h1 (overlaps the second child)
    const bool mid = (F.state == 0);
    const int64_t km = F.km;
    const int64_t A = F.f + 2 * (int64_t)h - h1 - km;
    if (!mid) ref_node_bottom<ACCT>(X, h, A);
    const int m = mid ? h1 : h2;
    const int Lj = mid ? 2 * (h - h1) : (int)(A - 2 * h2), Mj = 2 * m + 1;
    const double* xj = mid ? F.in + F.f + 1 : F.asmo + km + 1;
    double* yj = mid ? F.asmo + F.f + h1 + 1 : F.out + km + h2 + 1;
    const long long tp = clock64();
    F.tk = helper_post(*X.S, X.c, F.q, xj, yj, Lj, wslot(*X.S, X.c, X.wst, sp, m), Mj, &F.tk0);
    tpost += clock64() - tp;
    if (ACCT && X.acct) X.flops += 2ull * (uint64_t)(Lj * Mj);
    F.state = mid ? 1 : 2;
    SubFrame& C = stk[sp++];
    C.f = mid ? F.f : km;
    C.h = m;
    C.in = mid ? F.in : F.asmo;
    C.out = mid ? F.asmo : F.out;
    C.state = 0;
  }
  LCLK_ADD(X.prof, PROF_WAIT_CYC, t1 - t0);
  LCLK_ADD(X.prof, PROF_F_STAGE, t2 - t1);
  LCLK_ADD(X.prof, PROF_F_MID, twait);
  LCLK_ADD(X.prof, PROF_F_BOT, tpost);
  LCLK_ADD(X.prof, PROF_FUSE_CYC, clock64() - t1);
  LCLK_ADD(X.prof, PROF_FUSE_N, 1);
  if (FL_PROFP(X.prof) && lane_id() == 0) {
    prof_add(FL_PROFP(X.prof), PROF_WAIT_CYC, t1 - t0);
    prof_add(FL_PROFP(X.prof), PROF_F_STAGE, t2 - t1);
    prof_add(FL_PROFP(X.prof), PROF_F_MID, twait);
    prof_add(FL_PROFP(X.prof), PROF_F_BOT, tpost);
    prof_add(FL_PROFP(X.prof), PROF_FUSE_CYC, clock64() - t1);
    prof_add(FL_PROFP(X.prof), PROF_FUSE_N, 1);
  }
  FL_TR(*X.S, X.c, EV_SUB_E, h0);
  return ret;
}

__device__ __forceinline__ void put_conv(PutChainCtx& X, const double* x, int64_t L, double* y, int64_t Lout,
                                         int h) {
  // the jumps of tall nodes have slack to spare (a sibling subtree of their own
  // height): chunked on the low-priority ring, a latency-critical short jump
  // never queues behind a whole one
  chain_conv(*X.S, X.c, X.st, x, L, y, Lout, h, X.kc, FL_STRIP_CLOCK ? X.prof : FL_PROFP(X.prof),
             FL_LOW_H > 0 && h >= FL_LOW_H);
}

// _solve_q (bsm.py:443-501) as an explicit-stack loop on the chain warp.
template <bool ACCT>
__device__ int64_t put_solve_q(PutChainCtx& X, const PutParams& P, int64_t f0, double* in_org, double* out_org,
                               int h0, int32_t* err) {
  static_assert(FRAME_SOLVE_OFF + sizeof(PutFrame) * PUT_MAX_DEPTH <= CHAIN_FRAME_DOUBLES * sizeof(double),
                "recursion frames");
  PutFrame* stk = chain_frames<PutFrame>(X.scratch, FRAME_SOLVE_OFF);
  stk[0].f = f0; stk[0].h = h0; stk[0].in_org = in_org; stk[0].out_org = out_org;
  stk[0].arena = 0; stk[0].state = 0;
  int sp = 1;
  int64_t ret = 0;
  while (sp > 0) {
    PutFrame& F = stk[sp - 1];
    const int h = F.h;
    const int ph = (sp >= 2) ? stk[sp - 2].h : 0x7fffffff;
    FL_TR(*X.S, X.c, EV_NODE, h * 4 + F.state);
    if (F.state == 0) {
      if (h <= PUT_HS) {
        ret = (P.slide && !X.full && PUT_LEAF <= PUT_SLIDE_H)
                  ? put_subtree<ACCT, 1>(X, P, F.f, F.in_org, F.out_org, h, ph, err)
                  : put_subtree<ACCT, 0>(X, P, F.f, F.in_org, F.out_org, h, ph, err);
        if (*err) return 0;
        --sp;
        continue;
      }
      ref_node_enter<ACCT>(X, h, ph);
      const int h1 = (h + 1) / 2;
      const int d = sp - 1;
      X.tog ^= 1u << d;
      F.asm_org = X.frames + (((X.tog >> d) & 1u) ? X.fstride : 0) + F.arena - (F.f - h1 + 1);
      // mid: cols f+h1+1 .. f+2h-h1 of row t+h1 from the 2h inputs
      put_conv(X, F.in_org + F.f + 1, 2 * (int64_t)h, F.asm_org + F.f + h1 + 1, 2 * (int64_t)(h - h1), h1);
      F.state = 1;
      PutFrame& C = stk[sp];
      C.f = F.f; C.h = h1; C.in_org = F.in_org; C.out_org = F.asm_org;
      C.arena = F.arena + 2 * (int64_t)h + 8; C.state = 0;
      if (++sp >= PUT_MAX_DEPTH) { *err = FL_E_CAPACITY | 1; return 0; }
    } else if (F.state == 1) {
      const int h1 = (h + 1) / 2, h2 = h - h1;
      const int64_t km = ret;
      if (km < F.f - h1 || km > F.f) { *err = FL_E_GEOMETRY | 2; return 0; }
      F.km = km;
      const int64_t A = F.f + 2 * (int64_t)h - h1 - km;  // assembled cols km+1 .. f+2h-h1
      ref_node_bottom<ACCT>(X, h, A);
      // bottom: cols km+h2+1 .. f+h of row t+h
      put_conv(X, F.asm_org + km + 1, A, F.out_org + km + h2 + 1, A - 2 * (int64_t)h2, h2);
      F.state = 2;
      PutFrame& C = stk[sp];
      C.f = km; C.h = h2; C.in_org = F.asm_org; C.out_org = F.out_org;
      C.arena = F.arena + 2 * (int64_t)h + 8; C.state = 0;
      ++sp;
    } else {
      const int h2 = h - (h + 1) / 2;
      const int64_t kp = ret;
      if (kp < F.km - h2 || kp > F.km) { *err = FL_E_GEOMETRY | 3; return 0; }
      --sp;
    }
  }
  return ret;
}

// One stage (_advance_stage, bsm.py:557-582): far jump + boundary recursion,
// cur -> nxt over hh rows.  Returns the new boundary.
template <bool ACCT = true>
__device__ int64_t put_stage(PutChainCtx& X, const PutParams& P, int64_t f, int64_t red, int64_t hh,
                             double* cur_org, double* nxt_org, int32_t* err) {
  const int h = (int)hh;
  if (red > 2 * hh) {  // far: cols f+h+1 .. f+red-h stay linear
    X.ref_flops += ref_jump_flops(red, 2 * hh + 1);
    chain_conv(*X.S, X.c, X.st, cur_org + f + 1, red, nxt_org + f + h + 1, red - 2 * hh, h, X.kc,
               FL_STRIP_CLOCK ? X.prof : FL_PROFP(X.prof), true);
  }
  return put_solve_q<ACCT>(X, P, f, cur_org, nxt_org, h, err);
}

__device__ void put_record(const BatchOut& out, int o, int32_t& cnt, int64_t t, int64_t c) {
  if (lane_id() == 0 && out.bt != nullptr && cnt < out.cap) {
    out.bt[(int64_t)o * out.cap + cnt] = t;
    out.bc[(int64_t)o * out.cap + cnt] = c;
  }
  ++cnt;
}

// Arena: stage rows A | B | payoff table | recursion frames | kernel table.
__device__ PutChainCtx put_chain_setup(SchedShared& S, int c, const PutParams& P, const PutLayout& Lo,
                                       int64_t n_rows, double* arena, double* scratch, unsigned long long* prof,
                                       const double* init_src, int64_t init_col0, int64_t init_len, bool acct = true) {
  double* bufA = arena;
  double* pay = arena + 2 * Lo.span;
  double* frames = arena + 3 * Lo.span;
  const int64_t fstride = 2 * n_rows + 64 * PUT_MAX_DEPTH;
  double* kc = frames + 2 * fstride;
  Stencil st{P.cd, P.cm, P.cu, 2};
  st.hsmall = small_ring_hmax(st);
  build_kernel_table(kc, st, scratch);
  PutChainCtx X{&S,   c,       st,  kc, frames, fstride, 0u, pay - Lo.colbase, scratch, chain_wstash(scratch),
                (int64_t)P.cutoff, acct, 0ull, 0ull, prof};
  if (lane_id() < 4) S.wkey[c][lane_id()] = -1;  // new option: new weights
  __syncwarp();
  // payoff table 1 - e^{col ds} (bsm.py:232-244), row A zeroed, optionally
  // loaded with an initial segment (cols init_col0 .. +init_len)
  Task t;
  t.kind = TK_PUT_INIT;
  t.x = init_src; t.w = nullptr;
  t.y = bufA;
  t.L = Lo.span;
  t.i0 = Lo.colbase; t.i1 = init_col0 - Lo.colbase; t.i2 = init_len;
  t.d0 = P.ds;
  t.c0 = t.c1 = t.c2 = 0.0; t.h = 0; t.span = 0; t.Lout = 0;
  issue(S, c, RING_BIG, t, 0, 0, U(bufA), U(pay + Lo.span));
  return X;
}

// fast_put_bsm's stage loop (bsm.py:626-676) for option o on chain warp c.
// Returns the status; FL_RETRY_FULL leaves no output (the caller re-prices the
// option with full = true: full-frame leaves only).
template <bool ACCT>
__device__ int32_t put_chain_option(SchedShared& S, int c, const PutParams& P, int o, double* arena,
                                    double* scratch, const BatchOut& out, double* chain_flops, double* ref_flops,
                                    bool full = false) {
  const long long t_opt = clock64();
  const int64_t n = P.n, ks = P.ks;
  const PutLayout Lo = put_layout(n, ks);
  PutChainCtx X = put_chain_setup(S, c, P, Lo, n, arena, scratch, out.prof, nullptr, 0, 0, out.acct != 0);
  X.full = full;
  LCLK_ADD(out.prof, PROF_DEPWAIT_CYC, clock64() - t_opt);  // option setup (kernel table, init task issue)
  double* cur_org = arena - Lo.colbase;
  double* nxt_org = arena + Lo.span - Lo.colbase;
  int32_t err = 0, cnt = 0;
  int64_t m = 0, f = 0;
  double price = 0.0;
  put_record(out, o, cnt, 0, 0);
  for (;;) {
    const int64_t rem = n - m;
    const int64_t red = ks + rem - f;
    if (red < 0) { err = FL_E_GEOMETRY | 4; break; }
    if (red == 0) { price = P.K * (1.0 - exp((double)ks * P.ds)); break; }
    if (rem <= 2 * (int64_t)P.cutoff) {
      if (2 * rem + 2 > BIG_SLOTS) { err = FL_E_CAPACITY | 2; break; }
      Task t;
      t.kind = TK_PUT_APEX;
      t.x = cur_org; t.w = X.pay_org; t.y = nullptr;
      t.i0 = f; t.i1 = rem; t.i2 = ks;
      t.c0 = P.cd; t.c1 = P.cm; t.c2 = P.cu; t.h = 0; t.span = 2; t.L = 0; t.Lout = 0; t.d0 = 0.0;
      const int ring = (2 * rem + 2 <= MED_WSLOTS) ? RING_SMALL : RING_BIG;  // two rows of the apex in one worker buffer
      const int id = issue(S, c, ring, t, U(cur_org + ks - rem - 1), U(cur_org + ks + rem + 1), 0, 0);
      FL_TR(S, c, EV_TW_B, 0);
      warp_wait_done(S, id);
      FL_TR(S, c, EV_TW_E, 0);
      price = P.K * S.result[c];
      const int64_t lo = (f < ks - rem ? f : ks - rem) - 1;
      X.ref_flops += ref_strip_flops(ks + rem - lo + 1, rem);
      X.flops += 5ull * (uint64_t)(rem * rem + rem);
      break;
    }
    const int64_t hh = (rem / 2 < red / 2) ? rem / 2 : red / 2;
    if (hh < 1) {
      wait_conflicts(S, c, U(cur_org + f + 1), U(cur_org + f + 2), U(X.pay_org + f - 3), U(X.pay_org + f + 2),
                     U(nxt_org + f - 3), U(nxt_org + f + 2));
      X.ref_flops += ref_strip_flops(red + 4, 1);
      const int64_t kb = put_leaf(X, P, cur_org, nxt_org, X.pay_org, f - 3, f + 1, f, 1);
      if (kb == NONE_SEEN || kb < f - 1 || kb > f) { err = FL_E_GEOMETRY | 5; break; }
      f = kb;
      m += 1;
    } else {
      const int64_t kp = put_stage<ACCT>(X, P, f, red, hh, cur_org, nxt_org, &err);
      if (err) break;
      f = kp;
      m += hh;
    }
    put_record(out, o, cnt, m, f);
    if (out.snap) {  // record_rows (bsm.py:667-671): the handoff row's continuation segment
      wait_all_own(S, c);
      const int64_t len = ks + (n - m) - f;
      int64_t* used = out.snap_len + o;
      if (*used + len <= out.snap_cap) {
        double* dst = out.snap + (int64_t)o * out.snap_cap + *used;
        for (int64_t i = lane_id(); i < len; i += 32) dst[i] = nxt_org[f + 1 + i];
      }
      __syncwarp();
      if (lane_id() == 0) *used += len;  // the true length even when truncated
      __syncwarp();
    }
    double* t = cur_org;
    cur_org = nxt_org;
    nxt_org = t;
  }
  wait_all_own(S, c);  // the next option reuses this arena
  if (err == FL_RETRY_FULL) {
    if (out.snap && lane_id() == 0) out.snap_len[o] = 0;
    __syncwarp();
    return err;
  }
  if (lane_id() == 0) {
    out.price[o] = err ? 0.0 : price;
    out.status[o] = err;
    if (out.bcount) out.bcount[o] = err ? 0 : cnt;
    prof_add(out.prof, PROF_CHAIN_CYC, clock64() - t_opt);
  }
  LCLK_ADD(out.prof, PROF_CHAIN_CYC, clock64() - t_opt);
  *chain_flops += (double)X.flops;
  *ref_flops += (double)X.ref_flops;
  return err;
}

// put_chain_option with the full-frame re-run (at most one).
template <bool ACCT>
__device__ void put_chain_option_retry(SchedShared& S, int c, const PutParams& P, int o, double* arena,
                                       double* scratch, const BatchOut& out, double* chain_flops, double* ref_flops) {
  bool full = false;
  while (put_chain_option<ACCT>(S, c, P, o, arena, scratch, out, chain_flops, ref_flops, full) == FL_RETRY_FULL) {
    full = true;
    LCLK_ADD(out.prof, PROF_S_LEAF, 1);  // tool builds: options re-priced on the full frame
  }
}

// Worker-side execution of the put-specific tasks.  slots: capacity of sbuf in
// double2 (the apex uses it as two double arrays of `slots` entries).
__device__ double put_exec_task(SchedShared& S, const Task& t, double2* sbuf, int slots, int logN,
                                const double2* tq, const Grp& g) {
  if (t.kind == TK_PUT_INIT) {
    double* A = t.y;
    double* pay = t.y + 2 * t.L;
    for (int64_t i = g.t; i < t.L; i += g.n) {
      const int64_t k = i - t.i1;  // position in the initial segment
      A[i] = (t.x != nullptr && k >= 0 && k < t.i2) ? t.x[k] : 0.0;
      pay[i] = 1.0 - exp((double)(t.i0 + i) * t.d0);
    }
    return 0.0;
  }
  if (t.kind == TK_PUT_APEX) {
    // apex cone sweep (bsm._apex_finish) restricted to [ks-rem-1, ks+rem]
    const double* cur_org = t.x;
    const double* pay_org = t.w;
    const int64_t f = t.i0, rem = t.i1, ks = t.i2;
    const int64_t lo = ks - rem - 1, hi = ks + rem;
    const int W = (int)(hi - lo + 1);
    double* a = (double*)sbuf;
    double* b = a + slots;
    for (int i = g.t; i < W; i += g.n) {
      const int64_t col = lo + i;
      a[i] = (col <= f) ? pay_org[col] : cur_org[col];
      b[i] = a[i];
    }
    gsync(g);
    for (int s = 1; s <= rem; ++s) {
      for (int i = s + g.t; i <= W - 1 - s; i += g.n) {
        const double lin = fma(t.c0, a[i - 1], fma(t.c2, a[i + 1], t.c1 * a[i]));
        const double p = pay_org[lo + i];
        b[i] = lin > p ? lin : p;
      }
      gsync(g);
      double* tmp = a;
      a = b;
      b = tmp;
    }
    if (g.t == 0) S.result[t.chain] = a[ks - lo];
    return 0.0;
  }
  return exec_generic(t, sbuf, slots, logN, tq, g);
}

// ACCT selects the kernel instance: production launches run the walk without
// the per-node flop counting, accounting launches (fl_abi.cu) with it.  Two
// kernels rather than a run-time branch: one kernel holding both walks
// allocates registers for both and spills.
template <bool ACCT>
struct PutPricer {
  const PutParams* opts;
  const int32_t* order;
  BatchOut out;
  __device__ void chain(SchedShared& S, int c, int w, double* arena, double* scratch, double* flops) const {
    double ref = 0.0;
    const int o = order[w];
    put_chain_option_retry<ACCT>(S, c, opts[o], o, arena, scratch, out, flops, &ref);
    if (lane_id() == 0 && out.flops) atomicAdd(out.flops + 1, (unsigned long long)ref);
  }
  __device__ double exec(SchedShared& S, const Task& t, double2* sbuf, int slots, int logN, const double2* tq,
                         const Grp& g) const {
    return put_exec_task(S, t, sbuf, slots, logN, tq, g);
  }
};

template <bool ACCT>
__global__ void __launch_bounds__(SCHED_THREADS, 1)
put_fast_kernel(const PutParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork,
                int32_t* counter, double* __restrict__ ws, int64_t ws_stride, BatchOut out) {
  apply_dlist(out, order, nwork);
  const PutPricer<ACCT> pr{opts, order, out};
  sched_body(pr, nwork, counter, ws, ws_stride, out.flops, out.prof);
}

// ---------------------------------------------------------------------------
// solve_bsm_trapezoid (bsm.py:504-554): one stage of height h from a given
// row state (boundary f, continuation values on cols f+1 .. f+W).  Output:
// meta[0] = new boundary kp, meta[1] = status, values of cols kp+1 .. f+W-h
// into out[0 .. f+W-h-kp).

struct PutTrapPricer {
  PutParams P;  // cd, cm, cu, ds, cutoff used
  int64_t f, W, h;
  const double* seg;
  double* out;
  int64_t* meta;
  unsigned long long* flops;
  __device__ void chain(SchedShared& S, int c, int w, double* arena, double* scratch, double* fl) const {
    const PutLayout Lo = put_trap_layout(f, W, h);
    PutChainCtx X = put_chain_setup(S, c, P, Lo, 2 * h, arena, scratch, nullptr, seg, f + 1, W);
    double* cur_org = arena - Lo.colbase;
    double* nxt_org = arena + Lo.span - Lo.colbase;
    int32_t err = 0;
    int64_t kp = put_stage(X, P, f, W, h, cur_org, nxt_org, &err);
    wait_all_own(S, c);
    if (err == FL_RETRY_FULL) {  // a fixed-frame leaf lost its margin: full frame
      err = 0;
      X = put_chain_setup(S, c, P, Lo, 2 * h, arena, scratch, nullptr, seg, f + 1, W);
      X.full = true;
      kp = put_stage(X, P, f, W, h, cur_org, nxt_org, &err);
      wait_all_own(S, c);
    }
    const int64_t len = err ? 0 : (f + W - h) - kp;
    for (int64_t i = lane_id(); i < len; i += 32) out[i] = nxt_org[kp + 1 + i];
    if (lane_id() == 0) {
      meta[0] = err ? 0 : kp;
      meta[1] = err;
      if (flops) atomicAdd(flops + 1, (unsigned long long)X.ref_flops);
    }
    *fl += (double)X.flops;
  }
  __device__ double exec(SchedShared& S, const Task& t, double2* sbuf, int slots, int logN, const double2* tq,
                         const Grp& g) const {
    return put_exec_task(S, t, sbuf, slots, logN, tq, g);
  }
};

__global__ void __launch_bounds__(SCHED_THREADS, 1)
put_trap_kernel(PutTrapPricer pr, int32_t* counter, double* __restrict__ ws, int64_t ws_stride) {
  sched_body(pr, 1, counter, ws, ws_stride, pr.flops, nullptr);
}

// ---------------------------------------------------------------------------
// O(T^2) projected march over the shrinking window (baseline_put_fd).  Same
// unfused operation order as _accel.put_march_window (_accel.py:163-200), so
// prices and boundaries are bit-identical to the reference.

__global__ void __launch_bounds__(CTA_THREADS)
put_baseline_kernel(const PutParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork,
                    double* __restrict__ ws, int64_t ws_stride, BatchOut out) {
  __shared__ int s_red[CTA_THREADS / 32];
  apply_dlist(out, order, nwork);
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
  const int o = order[w];
  const PutParams P = opts[o];
  const int64_t n = P.n;
  const int64_t W = 2 * n + 1;
  const int64_t lo = P.ks - n;
  double* a = ws + (int64_t)blockIdx.x * ws_stride;
  double* b = a + W;
  double* pay = b + W;
  for (int64_t k = threadIdx.x; k < W; k += CTA_THREADS) {
    const double p = 1.0 - exp((double)(lo + k) * P.ds);
    pay[k] = p;
    a[k] = p > 0.0 ? p : 0.0;
    b[k] = a[k];
  }
  __syncthreads();
  const bool rec = out.bt != nullptr;
  if (rec && threadIdx.x == 0 && out.cap > 0) {
    out.bt[(int64_t)o * out.cap] = 0;
    out.bc[(int64_t)o * out.cap] = (P.ks + n < 0) ? P.ks + n : 0;
  }
  for (int64_t s = 1; s <= n; ++s) {
    int lg = -1;
    for (int64_t k = s + threadIdx.x; k <= W - 1 - s; k += CTA_THREADS) {
      // cm*cur + cu*right + cd*left, left to right, no contraction
      const double lin = __dadd_rn(__dadd_rn(__dmul_rn(P.cm, a[k]), __dmul_rn(P.cu, a[k + 1])),
                                   __dmul_rn(P.cd, a[k - 1]));
      const double p = pay[k];
      const bool red = lin > p;
      b[k] = red ? lin : p;
      if (!red) lg = (int)k;
    }
    if (rec) {
      lg = warp_max_i32(lg);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = lg;
    }
    __syncthreads();
    if (rec && threadIdx.x == 0 && s < out.cap) {
      int m = -1;
      for (int i = 0; i < CTA_THREADS / 32; ++i) m = s_red[i] > m ? s_red[i] : m;
      out.bt[(int64_t)o * out.cap + s] = s;
      out.bc[(int64_t)o * out.cap + s] = (m < 0) ? INT64_MIN : lo + m;
    }
    double* t = a;
    a = b;
    b = t;
  }
  if (threadIdx.x == 0) {
    out.price[o] = P.K * a[n];
    out.status[o] = 0;
    if (out.bcount) out.bcount[o] = (int32_t)(n + 1);
  }
  __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// launchers

int put_fast_smem_bytes() { return sched_smem_bytes(); }
int put_chains_per_cta() { return NCHAIN; }

static cudaError_t put_configure() {
  static std::atomic<unsigned long long> configured{0};
  return once_per_device(configured, [] {
    const int smem = sched_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(put_fast_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(put_fast_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(put_trap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return e;
  });
}

cudaError_t launch_put_fast(const PutParams* opts, const int32_t* order, int nwork, int32_t* counter, double* ws,
                            int64_t ws_stride, int grid, BatchOut out, cudaStream_t stream) {
  cudaError_t e = put_configure();
  if (e != cudaSuccess) return e;
  if (nwork <= 0) return cudaSuccess;
  e = cudaMemsetAsync(counter, 0, sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  if (out.acct)
    put_fast_kernel<true><<<grid, SCHED_THREADS, sched_smem_bytes(), stream>>>(opts, order, nwork, counter, ws,
                                                                               ws_stride, out);
  else
    put_fast_kernel<false><<<grid, SCHED_THREADS, sched_smem_bytes(), stream>>>(opts, order, nwork, counter, ws,
                                                                                ws_stride, out);
  return cudaGetLastError();
}

int64_t put_trap_ws_doubles(int64_t f, int64_t W, int64_t h) {
  return put_arena_doubles(put_trap_layout(f, W, h).span, 2 * h);
}

cudaError_t launch_put_trapezoid(const PutParams& P, int64_t f, int64_t W, int64_t h, const double* seg,
                                 double* out, int64_t* meta, int32_t* counter, double* ws, int64_t ws_stride,
                                 unsigned long long* flops, cudaStream_t stream) {
  cudaError_t e = put_configure();
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  const PutTrapPricer pr{P, f, W, h, seg, out, meta, flops};
  put_trap_kernel<<<1, SCHED_THREADS, sched_smem_bytes(), stream>>>(pr, counter, ws, ws_stride);
  return cudaGetLastError();
}

// baseline_put_fd with record_rows (bsm.py:296-322): one option, the O(T^2)
// march with snapshots of the valid window after the given steps.  Row t
// snapshot = window offsets t .. 2n-t (columns lo+t ..), packed in order.
__global__ void __launch_bounds__(CTA_THREADS)
put_march_rows_kernel(PutParams P, const int64_t* __restrict__ times, int ntimes, double* __restrict__ snap,
                      int64_t* __restrict__ last_green, double* __restrict__ price, double* __restrict__ ws) {
  __shared__ int s_red[CTA_THREADS / 32];
  const int64_t n = P.n;
  const int64_t W = 2 * n + 1;
  const int64_t lo = P.ks - n;
  double* a = ws;
  double* b = a + W;
  double* pay = b + W;
  for (int64_t k = threadIdx.x; k < W; k += CTA_THREADS) {
    const double p = 1.0 - exp((double)(lo + k) * P.ds);
    pay[k] = p;
    a[k] = p > 0.0 ? p : 0.0;
    b[k] = a[k];
  }
  __syncthreads();
  int ti = 0;
  int64_t soff = 0;
  for (int64_t s = 1; s <= n; ++s) {
    int lg = -1;
    for (int64_t k = s + threadIdx.x; k <= W - 1 - s; k += CTA_THREADS) {
      const double lin = __dadd_rn(__dadd_rn(__dmul_rn(P.cm, a[k]), __dmul_rn(P.cu, a[k + 1])),
                                   __dmul_rn(P.cd, a[k - 1]));
      const double p = pay[k];
      const bool red = lin > p;
      b[k] = red ? lin : p;
      if (!red) lg = (int)k;
    }
    lg = warp_max_i32(lg);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = lg;
    __syncthreads();
    if (threadIdx.x == 0) {
      int m = -1;
      for (int i = 0; i < CTA_THREADS / 32; ++i) m = s_red[i] > m ? s_red[i] : m;
      last_green[s] = (m < 0) ? INT64_MIN : lo + m;
    }
    double* t = a;
    a = b;
    b = t;
    while (ti < ntimes && times[ti] == s) {  // snapshot of the valid window of row s
      const int64_t len = W - 2 * s;
      for (int64_t k = threadIdx.x; k < len; k += CTA_THREADS) snap[soff + k] = a[s + k];
      soff += len;
      ++ti;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *price = P.K * a[n];
    last_green[0] = (P.ks + n < 0) ? P.ks + n : 0;
  }
}

cudaError_t launch_put_march_rows(const PutParams& P, const int64_t* times, int ntimes, double* snap,
                                  int64_t* last_green, double* price, double* ws, cudaStream_t stream) {
  put_march_rows_kernel<<<1, CTA_THREADS, 0, stream>>>(P, times, ntimes, snap, last_green, price, ws);
  return cudaGetLastError();
}

// O(T^2) baseline: the register-resident sweep (fl_sweep.cu) when the row
// fits its tile, else the global-memory march.  grid: CTAs (each loops over
// work items; the global march needs ws_stride doubles per CTA).
cudaError_t launch_put_baseline(const PutParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                                double* ws, int64_t ws_stride, BatchOut out, cudaStream_t stream) {
  if (nwork <= 0 || grid <= 0) return cudaSuccess;
  if (!out.dlist) {  // a few options (count known on the host): a cluster of SMs per option
    const cudaError_t e = launch_put_sweep_cluster(opts, order, nwork, n_max, out, stream);
    if (e != cudaErrorNotSupported) return e;
    (void)cudaGetLastError();
  }
  if (2 * n_max + 1 <= sweep_max_cells() && !sweep_disabled()) return launch_put_sweep(opts, order, nwork, n_max, grid, out, stream);
  put_baseline_kernel<<<grid, CTA_THREADS, 0, stream>>>(opts, order, nwork, ws, ws_stride, out);
  return cudaGetLastError();
}

}  // namespace fl
