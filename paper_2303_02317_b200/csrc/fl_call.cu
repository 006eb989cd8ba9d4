// fl_call.cu -- American call on the binomial lattice: device trapezoid
// decomposition (replaces american.fast_american_call and its recursion,
// american.py:201-530, and american.solve_trapezoid, american.py:298-358) and
// the O(T^2) projected induction (replaces binomial.baseline_american_call /
// _accel.american_call_backward, binomial.py:94-130, _accel.py:62-102).
//
// Same execution model as the put (fl_put.cu, fl_sched.cuh): a chain warp
// walks one option -- junction row, trapezoid loop, halving recursion -- and
// keeps the nonlinear leaves (binomial_strip_sweep, one column per lane,
// first green by warp min) and whole subtrees up to CALL_HS (in shared memory)
// to itself; the left / mid / bottom linear jumps are worker tasks, the
// junction row and the ceil(sqrt(T))-row residual strip are big-group tasks.
#include <cstdint>

#include "fl_common.cuh"
#include "fl_conv.cuh"
#include "fl_kernels.h"
#include "fl_sched.cuh"
#include "fl_strip.cuh"
#include "fl_callstrip.cuh"
#include "host_params.h"

namespace fl {

#ifndef FL_CALL_LEAF
#define FL_CALL_LEAF 128
#endif
constexpr int CALL_LEAF = FL_CALL_LEAF;  // leaf strip height (<= 64: call_leaf_v4<CALL_LEAF / 32>)
static_assert(CALL_LEAF == 32 || CALL_LEAF == 64 || CALL_LEAF == 128 || CALL_LEAF == 256,
              "leaf strips hold 32 * 2^k <= 256 columns");
#ifndef FL_CALL_LOW_H  // as FL_LOW_H (fl_put.cu) for the call's jumps; measured slower (C2 +2.7 %), off
#define FL_CALL_LOW_H 0
#endif
#ifndef FL_CALL_HS
#define FL_CALL_HS 256
#endif
constexpr int CALL_HS = FL_CALL_HS;  // recursion subtrees of height <= CALL_HS run whole in shared memory
constexpr int CALL_MAX_DEPTH = 28;
constexpr int CALL_RESID_CPT = 8;  // residual strip: cells per big-group thread (width <= 1024)
constexpr int CSUB_IN = 0, CSUB_ASM0 = CALL_HS + 8, CSUB_ASM1 = CSUB_ASM0 + CALL_HS + 8,
              CSUB_ASM2 = CSUB_ASM1 + CALL_HS / 2 + 8;
static_assert(CSUB_ASM2 + CALL_HS / 4 + 8 <= CHAIN_SCRATCH, "call subtree scratch");
static_assert(CALL_HS <= 8 * CALL_LEAF, "three asm levels cover a subtree");
static_assert(CALL_LEAF <= CALL_HS, "leaves inside the shared-memory subtrees");
static_assert(CALL_HS / 2 <= KT_H, "subtree correlations use the kernel table");

enum : int { TK_CALL_INIT = TK_USER + 4, TK_CALL_RESID = TK_USER + 5 };

__host__ __device__ inline int64_t call_arena_doubles(int64_t row_len, int64_t h_max) {
  return 2 * (row_len + 8) + 2 * (2 * h_max + 16 * CALL_MAX_DEPTH) + KTABLE_DOUBLES + 64;
}
int64_t call_ws_doubles(int64_t n_max) { return call_arena_doubles(n_max, n_max); }

__device__ __forceinline__ int64_t first_green_rec(int64_t i, int64_t j) {  // american.py:361-363
  return j >= i ? INT64_MIN : j + 1;
}

// reference-algorithmic cost model; the reference strip's cell
// count depends on the boundary path, estimated as 3/4 h^2 for h rows of width h
// (integer arithmetic on the chain: see fl_put.cu ref_jump_flops)
__device__ __forceinline__ uint64_t call_ref_jump(int64_t L, int64_t M) {
  const uint64_t need = (uint64_t)(L + M - 1);
  const int lg = need <= 1 ? 0 : 64 - __clzll((long long)(need - 1));
  const uint64_t N = 1ull << lg;
  return 5ull * N * (uint64_t)lg + 3ull * N + 6ull;
}

constexpr int CALL_TAB = CALL_LEAF + 8;
constexpr int CALL_E2 = CHAIN_SCRATCH - CALL_TAB;  // e2[k] = exp(2 k lu), k = 0..CALL_LEAF, in the chain scratch
constexpr int CALL_BT = CALL_E2 - CALL_TAB;        // a leaf's row bases (CALL_LEAF >= 128)
static_assert(CALL_BT >= CSUB_ASM2 + CALL_HS / 4 + 8, "e2 / base tables above the call subtree scratch");

struct CallFrame {
  int64_t i, j, jm;
  double* in_org;
  double* out_org;
  double* asm_org;
  int64_t arena;
  int h, state;
};

struct CallChainCtx {
  SchedShared* S;
  int c;
  Stencil st;
  const double* kc;
  double* frames;   // two copies of the frame arena, alternated per depth (see fl_put.cu)
  int64_t fstride;
  uint32_t tog;
  double* scratch;
  double* wst;  // weight stash (shared)
  int64_t ref_cut;
  bool acct;        // count flops (accounting runs only)
  uint64_t flops;   // executed chain-side flops
  uint64_t ref_q;   // reference-algorithmic flops x 4 (the 3/4 h^2 strip estimate stays exact)
  unsigned long long* prof;
};

__device__ __forceinline__ void call_ref_enter(CallChainCtx& X, int h, int ph) {
  if (!X.acct) return;
  if (h > X.ref_cut) X.ref_q += 4ull * call_ref_jump(h, (h + 1) / 2 + 1);
  else if (ph > X.ref_cut) X.ref_q += 15ull * (uint64_t)h * (uint64_t)h;  // 4 x 5 x 3/4 h^2
}
__device__ __forceinline__ void call_ref_bottom(CallChainCtx& X, int h, int64_t A) {
  if (!X.acct) return;
  const int h2 = h - (h + 1) / 2;
  if (h > X.ref_cut && A > h2) X.ref_q += 4ull * call_ref_jump(A, h2 + 1);
}

__device__ __forceinline__ int64_t call_leaf(CallChainCtx& X, const CallParams& P, const double* in_org,
                                             double* out_org, int64_t i, int64_t j, int h) {
  const long long t1 = clock64();
  double cells = 0.0;
  const int64_t jp = call_leaf_v4<CALL_LEAF / 32>(P, in_org, out_org, j - h + 1, i, j, h, &cells, X.scratch + CALL_E2,
                                                  X.scratch + CALL_BT);
  if (X.acct) X.flops += 5ull * (uint64_t)cells;
  LCLK_ADD(X.prof, PROF_STRIP_CYC, clock64() - t1);
  LCLK_ADD(X.prof, PROF_STRIP_N, h);
  if (FL_PROFP(X.prof) && lane_id() == 0) {
    prof_add(FL_PROFP(X.prof), PROF_STRIP_CYC, clock64() - t1);
    prof_add(FL_PROFP(X.prof), PROF_STRIP_N, h);
  }
  return jp;
}

struct CallSubFrame {
  int64_t i, j, jm;
  const double* in;
  double* out;
  double* asmo;
  int h, state, tk, tk0, q;
};

// A recursion subtree of height h0 <= CALL_HS done whole in shared memory
// (american.py:201-257 below this node): vals = in_org[j0-h0+1 .. j0] staged
// once; the chain runs the leaf strips while its helper warp runs every mid /
// bottom correlation (overlapping the node's first / second child).  Writes
// out_org[j0-h0+1 .. jp]; returns jp.
__device__ int64_t call_subtree(CallChainCtx& X, const CallParams& P, int64_t i0, int64_t j0, const double* in_org,
                                double* out_org, int h0, int ph0, int32_t* err) {
  const int64_t lo0 = j0 - h0 + 1;
  const long long t0 = clock64();
  // the composed weights depend on nothing in flight: stage them while the
  // jump writing this subtree's input row may still be running
  if (h0 > CALL_LEAF) stash_weights(*X.S, X.c, X.wst, X.kc, h0, CALL_LEAF, 1);
  wait_conflicts(*X.S, X.c, U(in_org + lo0), U(in_org + j0 + 1), 0, 0, U(out_org + lo0), U(out_org + j0 + 1));
  const long long t1 = clock64();
  double* s_in = X.scratch + CSUB_IN;
  warp_stage_async(s_in, in_org + lo0, h0);
  warp_stage_wait();  // weights and input row
  long long twait = 0;
  static_assert(sizeof(CallSubFrame) * 5 <= FRAME_SOLVE_OFF - FRAME_SUB_OFF, "subtree frames");
  CallSubFrame* stk = chain_frames<CallSubFrame>(X.scratch, FRAME_SUB_OFF);
  stk[0].i = i0; stk[0].j = j0; stk[0].h = h0; stk[0].in = s_in - lo0; stk[0].out = out_org; stk[0].state = 0;
  int sp = 1;
  int64_t ret = 0;
  // one helper post site and one wait site (as put_subtree)
  while (sp > 0) {
    CallSubFrame& F = stk[sp - 1];
    const int h = F.h, h1 = (h + 1) / 2, h2 = h - h1;
    const int64_t lo = F.j - h + 1;
    if (F.state == 0) {
      call_ref_enter(X, h, (sp >= 2) ? stk[sp - 2].h : ph0);
      if (h <= CALL_LEAF) {
        ret = call_leaf(X, P, F.in, F.out, F.i, F.j, h);
        --sp;
        continue;
      }
      F.asmo = X.scratch + (sp == 1 ? CSUB_ASM0 : sp == 2 ? CSUB_ASM1 : CSUB_ASM2) - lo;
      F.q = (sp == 1) ? 1 : 0;  // the subtree root's jumps have the most slack: background ring
    } else {
      // a child finished (state 1: first child from j, state 2: second from jm);
      // then the jump posted before it (mid / bottom, if any) must be complete
      const bool first = (F.state == 1);
      const int64_t jr = first ? F.j : F.jm;
      const int hr = first ? h1 : h2;
      if (ret < jr - hr || ret > jr) { *err = FL_E_GEOMETRY | (first ? 1 : 2); return 0; }
      if (first || F.tk >= 0) {
        const long long tw = clock64();
        helper_wait_range(*X.S, X.c, F.q, F.tk0, F.tk);
        twait += clock64() - tw;
      }
      if (!first) {
        --sp;
        continue;
      }
      F.jm = ret;
    }
    // state 0: mid (helper), cols lo .. j-h1 of row i-h1; state 1: bottom, cols
    // lo .. jm-h2 of row i-h from the assembled cols lo .. jm (if any)
    const bool mid = (F.state == 0);
    const int64_t A = F.jm - lo + 1;
    if (!mid) call_ref_bottom(X, h, A);
    const int m = mid ? h1 : h2;
    const int Lj = mid ? h2 : (int)(A - h2);
    F.tk = -1;
    if (mid || A > h2) {
      F.tk = helper_post(*X.S, X.c, F.q, (mid ? F.in : F.asmo) + lo, (mid ? F.asmo : F.out) + lo, Lj,
                         wslot(*X.S, X.c, X.wst, sp, m), m + 1, &F.tk0);
      if (X.acct) X.flops += 2ull * (uint64_t)((int64_t)Lj * (m + 1));
    }
    F.state = mid ? 1 : 2;
    CallSubFrame& C = stk[sp++];
    C.i = mid ? F.i : F.i - h1;
    C.j = mid ? F.j : F.jm;
    C.h = m;
    C.in = mid ? F.in : F.asmo;
    C.out = mid ? F.asmo : F.out;
    C.state = 0;
  }
  LCLK_ADD(X.prof, PROF_WAIT_CYC, t1 - t0);
  LCLK_ADD(X.prof, PROF_F_MID, twait);
  LCLK_ADD(X.prof, PROF_FUSE_CYC, clock64() - t1);
  LCLK_ADD(X.prof, PROF_FUSE_N, 1);
  if (FL_PROFP(X.prof) && lane_id() == 0) {
    prof_add(FL_PROFP(X.prof), PROF_WAIT_CYC, t1 - t0);
    prof_add(FL_PROFP(X.prof), PROF_F_MID, twait);
    prof_add(FL_PROFP(X.prof), PROF_FUSE_CYC, clock64() - t1);
    prof_add(FL_PROFP(X.prof), PROF_FUSE_N, 1);
  }
  return ret;
}

__device__ __forceinline__ void call_conv(CallChainCtx& X, const double* x, int64_t L, double* y, int64_t Lout,
                                          int h) {
  chain_conv(*X.S, X.c, X.st, x, L, y, Lout, h, X.kc, FL_STRIP_CLOCK ? X.prof : FL_PROFP(X.prof),
             FL_CALL_LOW_H > 0 && h >= FL_CALL_LOW_H);
}

// _solve (american.py:201-257) with an explicit stack on the chain warp.
// vals = in_org[j-h+1 .. j]; writes out_org[j-h+1 .. jp]; returns jp.
__device__ int64_t call_solve(CallChainCtx& X, const CallParams& P, int64_t i0, int64_t j0, int h0, double* in_org,
                              double* out_org, int32_t* err) {
  static_assert(FRAME_SOLVE_OFF + sizeof(CallFrame) * CALL_MAX_DEPTH <= CHAIN_FRAME_DOUBLES * sizeof(double),
                "recursion frames");
  CallFrame* stk = chain_frames<CallFrame>(X.scratch, FRAME_SOLVE_OFF);
  stk[0].i = i0; stk[0].j = j0; stk[0].h = h0; stk[0].in_org = in_org; stk[0].out_org = out_org;
  stk[0].arena = 0; stk[0].state = 0;
  int sp = 1;
  int64_t ret = 0;
  while (sp > 0) {
    CallFrame& F = stk[sp - 1];
    const int h = F.h;
    const int h1 = (h + 1) / 2, h2 = h - h1;
    const int ph = (sp >= 2) ? stk[sp - 2].h : 0x7fffffff;
    if (F.state == 0) {
      const int64_t lo = F.j - h + 1;
      if (h <= CALL_HS) {
        ret = call_subtree(X, P, F.i, F.j, F.in_org, F.out_org, h, ph, err);
        if (*err) return 0;
        --sp;
        continue;
      }
      call_ref_enter(X, h, ph);
      const int d = sp - 1;
      X.tog ^= 1u << d;
      F.asm_org = X.frames + (((X.tog >> d) & 1u) ? X.fstride : 0) + F.arena - lo;
      // mid: cols lo .. j-h1 of row i-h1
      call_conv(X, F.in_org + lo, h, F.asm_org + lo, h2, h1);
      F.state = 1;
      CallFrame& C = stk[sp];
      C.i = F.i; C.j = F.j; C.h = h1; C.in_org = F.in_org; C.out_org = F.asm_org;
      C.arena = F.arena + h + 8; C.state = 0;
      if (++sp >= CALL_MAX_DEPTH) { *err = FL_E_CAPACITY | 1; return 0; }
    } else if (F.state == 1) {
      const int64_t jm = ret;
      if (jm < F.j - h1 || jm > F.j) { *err = FL_E_GEOMETRY | 3; return 0; }
      F.jm = jm;
      const int64_t lo = F.j - h + 1;
      const int64_t A = jm - lo + 1;  // assembled cols lo .. jm
      call_ref_bottom(X, h, A);
      // bottom: cols lo .. jm-h2 of row i-h
      if (A > h2) call_conv(X, F.asm_org + lo, A, F.out_org + lo, A - h2, h2);
      F.state = 2;
      CallFrame& C = stk[sp];
      C.i = F.i - h1; C.j = jm; C.h = h2; C.in_org = F.asm_org; C.out_org = F.out_org;
      C.arena = F.arena + h + 8; C.state = 0;
      ++sp;
    } else {
      const int64_t jp = ret;
      if (jp < F.jm - h2 || jp > F.jm) { *err = FL_E_GEOMETRY | 4; return 0; }
      --sp;
    }
  }
  return ret;
}

__device__ void call_record(const BatchOut& out, int o, int32_t& cnt, int64_t t, int64_t c) {
  if (lane_id() == 0 && out.bt != nullptr && cnt < out.cap) {
    out.bt[(int64_t)o * out.cap + cnt] = t;
    out.bc[(int64_t)o * out.cap + cnt] = c;
  }
  ++cnt;
}

__device__ CallChainCtx call_chain_setup(SchedShared& S, int c, const CallParams& P, int64_t row_len, int64_t h_max,
                                         double* arena, double* scratch, unsigned long long* prof, bool acct = true) {
  double* frames = arena + 2 * (row_len + 8);
  const int64_t fstride = 2 * h_max + 16 * CALL_MAX_DEPTH;
  double* kc = frames + 2 * fstride;
  Stencil st{P.wd, P.wu, 0.0, 1};
  st.hsmall = small_ring_hmax(st);
  build_kernel_table(kc, st, scratch);
  __syncwarp();
  for (int k = lane_id(); k < CALL_TAB; k += 32) scratch[CALL_E2 + k] = exp(2.0 * (double)k * P.lu);  // call_leaf_v4
  __syncwarp();
  if (lane_id() < 4) S.wkey[c][lane_id()] = -1;  // new option: new weights
  __syncwarp();
  return CallChainCtx{&S, c, st, kc, frames, fstride, 0u, scratch, chain_wstash(scratch), (int64_t)P.cutoff,
                      acct, 0ull, 0ull, prof};
}

// The trapezoid loop from row i / boundary j down to the residual (american.py:486-498).
__device__ void call_trapezoids(CallChainCtx& X, const CallParams& P, int64_t& i, int64_t& j, int64_t first,
                                int64_t resid, double*& cur_org, double*& nxt_org, int32_t* err, const BatchOut* out,
                                int o, int32_t* cnt) {
  while (i > resid && j >= first) {
    const int64_t hh = (j - first + 1 < i - resid) ? j - first + 1 : i - resid;
    const int h = (int)hh;
    // left: cols first .. j-h of row i-h (american.py:341-344)
    const int64_t L = j - first + 1;
    if (L > hh) {
      X.ref_q += 4ull * call_ref_jump(L, hh + 1);
      chain_conv(*X.S, X.c, X.st, cur_org + first, L, nxt_org + first, L - hh, h, X.kc, FL_PROFP(X.prof), true);
    }
    const int64_t jp = call_solve(X, P, i, j, h, cur_org, nxt_org, err);
    if (*err) return;
    i -= hh;
    j = jp;
    if (out) call_record(*out, o, *cnt, i, first_green_rec(i, j));
    double* t = cur_org;
    cur_org = nxt_org;
    nxt_org = t;
  }
}

// fast_american_call (american.py:471-530) for option o on chain warp c.
__device__ void call_chain_option(SchedShared& S, int c, const CallParams& P, int o, double* arena,
                                  double* scratch, const BatchOut& out, double* chain_flops) {
  const long long t_opt = clock64();
  const int64_t n = P.n;
  CallChainCtx X = call_chain_setup(S, c, P, n, n, arena, scratch, out.prof, out.acct != 0);
  LCLK_ADD(out.prof, PROF_DEPWAIT_CYC, clock64() - t_opt);  // option setup (kernel table, e2 table)
  double* cur_org = arena;
  double* nxt_org = arena + (n + 8);
  int32_t err = 0, cnt = 0;
  call_record(out, o, cnt, n, first_green_rec(n, P.top_b));
  int64_t i = n - 1, j = P.junc_j;
  call_record(out, o, cnt, i, first_green_rec(i, j));
  {  // junction row T-1 (american.py:412-422) into row A
    Task t;
    t.kind = TK_CALL_INIT;
    t.x = nullptr; t.w = nullptr; t.y = cur_org;
    t.L = j + 1; t.Lout = 0;
    t.c0 = P.wd; t.c1 = P.wu; t.c2 = P.lu; t.d0 = P.S;
    t.i0 = n; t.i1 = P.top_b > 0 ? P.top_b : 0;
    t.i2 = __double_as_longlong(P.K);  // K travels as a bit pattern
    t.h = 0; t.span = 0;
    issue(S, c, RING_BIG, t, 0, 0, U(cur_org), U(cur_org + j + 1));
  }
  const int64_t resid = (int64_t)floor(sqrt((double)(n - 1))) + 1;  // isqrt(n-1)+1 (exact below 2^52)
  call_trapezoids(X, P, i, j, 0, resid, cur_org, nxt_org, &err, &out, o, &cnt);
  double price = 0.0;
  if (!err) {
    if (j < 0) {
      price = P.S - P.K;
    } else if (j + 2 > BIG_SLOTS || j + 1 > (int64_t)CALL_RESID_CPT * BIG_THREADS) {
      err = FL_E_CAPACITY | 2;
    } else {
      Task t;
      t.kind = TK_CALL_RESID;
      t.x = cur_org; t.y = nullptr; t.w = nullptr;
      t.L = 0; t.Lout = 0;
      t.c0 = P.wd; t.c1 = P.wu; t.c2 = P.lu; t.d0 = P.S;
      t.i0 = i; t.i1 = j; t.i2 = __double_as_longlong(P.K);
      t.h = 0; t.span = 0;
      const int id = issue(S, c, RING_BIG, t, U(cur_org), U(cur_org + j + 1), 0, 0);
      const long long tr = clock64();
      warp_wait_done(S, id);
      LCLK_ADD(out.prof, PROF_LEAF_LOAD, clock64() - tr);  // residual sweep wait
      const int64_t j0 = S.iresult[c];
      price = (j0 >= 0) ? S.result[c] : P.S - P.K;
      X.flops += 5ull * (uint64_t)S.result2[c];
      X.ref_q += 20ull * (uint64_t)S.result2[c];
      if (i > 0) call_record(out, o, cnt, 0, first_green_rec(0, j0));
    }
  }
  wait_all_own(S, c);
  if (lane_id() == 0) {
    out.price[o] = err ? 0.0 : price;
    out.status[o] = err;
    if (out.bcount) out.bcount[o] = err ? 0 : cnt;
    if (out.flops) atomicAdd(out.flops + 1, (unsigned long long)(X.ref_q / 4));
    prof_add(out.prof, PROF_CHAIN_CYC, clock64() - t_opt);
  }
  LCLK_ADD(out.prof, PROF_CHAIN_CYC, clock64() - t_opt);
  *chain_flops += (double)X.flops;
}

// Worker side of the call-specific tasks.
__device__ double call_exec_task(SchedShared& S, const Task& t, double2* sbuf, int slots, int logN,
                                 const double2* tq, const Grp& g) {
  if (t.kind == TK_CALL_INIT) {
    const double wd = t.c0, wu = t.c1, lu = t.c2, S0 = t.d0, K = __longlong_as_double(t.i2);
    const int64_t n = t.i0, start = t.i1;
    double* row = t.y;
    for (int64_t c = g.t; c < t.L; c += g.n) {
      double v = 0.0;
      if (t.x != nullptr) {
        v = t.x[c];
      } else if (c >= start) {
        double l0 = __dsub_rn(__dmul_rn(S0, exp(__dmul_rn(__dsub_rn(2.0 * (double)c, (double)n), lu))), K);
        double l1 = __dsub_rn(__dmul_rn(S0, exp(__dmul_rn(__dsub_rn(2.0 * (double)(c + 1), (double)n), lu))), K);
        l0 = l0 > 0.0 ? l0 : 0.0;
        l1 = l1 > 0.0 ? l1 : 0.0;
        v = __dadd_rn(__dmul_rn(wd, l0), __dmul_rn(wu, l1));
      }
      row[c] = v;
    }
    return 0.0;
  }
  if (t.kind == TK_CALL_RESID) {
    // residual strip over the whole run (american.py:499-521): lo = 0, height = i
    const double wd = t.c0, wu = t.c1, lu = t.c2, S0 = t.d0, K = __longlong_as_double(t.i2);
    const int64_t i = t.i0, j0 = t.i1;
    const int64_t W = j0 + 1;
    double* sv = (double*)sbuf;
    double* se2 = sv + (W + 1);
    int* s_fg = (int*)(se2 + (W + 1));
    for (int64_t c = g.t; c <= W; c += g.n) {
      sv[c] = (c < W) ? t.x[c] : 0.0;
      se2[c] = exp(2.0 * (double)c * lu);
    }
    gsync(g);
    int64_t j = j0;
    double cells = 0.0;
    for (int64_t s = 0; s < i; ++s) {
      if (j < 0) break;
      const int64_t parent = i - s, child = parent - 1;
      const int64_t top = j < child ? j : child;
      cells += (double)(top + 1);
      const double bc = __dmul_rn(S0, exp((double)(0 - child) * lu));
      const double bp = __dmul_rn(S0, exp((double)(0 - parent) * lu));
      if (g.t == 0) *s_fg = INT32_MAX;
      double nv[CALL_RESID_CPT];
      int k = 0;
      int myfg = INT32_MAX;
      for (int64_t c = g.t; c <= top && k < CALL_RESID_CPT; c += g.n, ++k) {
        const double vr = (c + 1 <= j) ? sv[c + 1] : __dsub_rn(__dmul_rn(bp, se2[c + 1]), K);
        const double lin = __dadd_rn(__dmul_rn(wd, sv[c]), __dmul_rn(wu, vr));
        const double grn = __dsub_rn(__dmul_rn(bc, se2[c]), K);
        if (lin >= grn) {
          nv[k] = lin;
        } else {
          nv[k] = grn;
          if (myfg == INT32_MAX) myfg = (int)c;
        }
      }
      myfg = warp_min_i32(myfg);
      gsync(g);
      if ((g.t & 31) == 0 && myfg != INT32_MAX) atomicMin(s_fg, myfg);
      k = 0;
      for (int64_t c = g.t; c <= top && k < CALL_RESID_CPT; c += g.n, ++k) sv[c] = nv[k];
      gsync(g);
      const int fg = *s_fg;
      j = (fg == INT32_MAX) ? top : (int64_t)fg - 1;
      gsync(g);
    }
    if (g.t == 0) {
      S.result[t.chain] = sv[0];
      S.iresult[t.chain] = j;
      S.result2[t.chain] = cells;
    }
    return 5.0 * cells;
  }
  return exec_generic(t, sbuf, slots, logN, tq, g);
}

struct CallPricer {
  static constexpr int kLayout = 6;  // one chain per SMSP (see warp_role)
  const CallParams* opts;
  const int32_t* order;
  BatchOut out;
  __device__ void chain(SchedShared& S, int c, int w, double* arena, double* scratch, double* flops) const {
    const int o = order[w];
    call_chain_option(S, c, opts[o], o, arena, scratch, out, flops);
  }
  __device__ double exec(SchedShared& S, const Task& t, double2* sbuf, int slots, int logN, const double2* tq,
                         const Grp& g) const {
    return call_exec_task(S, t, sbuf, slots, logN, tq, g);
  }
};

__global__ void __launch_bounds__(SCHED_THREADS, 1)
call_fast_kernel(const CallParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork,
                 int32_t* counter, double* __restrict__ ws, int64_t ws_stride, BatchOut out) {
  apply_dlist(out, order, nwork);
  const CallPricer pr{opts, order, out};
  sched_body(pr, nwork, counter, ws, ws_stride, out.flops, out.prof);
}

// ---------------------------------------------------------------------------
// solve_trapezoid (american.py:298-358): one trapezoid of height h from row i,
// run = red values of cols first .. j.  Output: meta[0] = new boundary jp,
// meta[1] = status, values of cols first .. jp of row i-h into out.

struct CallTrapPricer {
  CallParams P;
  int64_t i, j, first, h;
  const double* run;
  double* out;
  int64_t* meta;
  unsigned long long* flops;
  __device__ void chain(SchedShared& S, int c, int w, double* arena, double* scratch, double* fl) const {
    const int64_t width = j - first + 1;
    CallChainCtx X = call_chain_setup(S, c, P, width, h, arena, scratch, nullptr);
    double* cur_org = arena - first;
    double* nxt_org = arena + (width + 8) - first;
    {  // load the run
      Task t;
      t.kind = TK_CALL_INIT;
      t.x = run; t.w = nullptr; t.y = arena;
      t.L = width; t.Lout = 0;
      t.c0 = t.c1 = t.c2 = 0.0; t.d0 = 0.0;
      t.i0 = t.i1 = t.i2 = 0; t.h = 0; t.span = 0;
      issue(S, c, RING_BIG, t, 0, 0, U(arena), U(arena + width));
    }
    int32_t err = 0;
    int64_t ii = i, jj = j;
    // exactly one trapezoid: resid chosen so the loop runs once with height h
    const int64_t hh = h;
    const int64_t L = width;
    if (L > hh) {
      X.ref_q += 4ull * call_ref_jump(L, hh + 1);
      call_conv(X, cur_org + first, L, nxt_org + first, L - hh, (int)hh);
    }
    const int64_t jp = call_solve(X, P, ii, jj, (int)hh, cur_org, nxt_org, &err);
    wait_all_own(S, c);
    const int64_t len = err ? 0 : jp - first + 1;
    for (int64_t k = lane_id(); k < len; k += 32) out[k] = nxt_org[first + k];
    if (lane_id() == 0) {
      meta[0] = err ? 0 : jp;
      meta[1] = err;
      if (flops) atomicAdd(flops + 1, (unsigned long long)(X.ref_q / 4));
    }
    *fl += (double)X.flops;
  }
  __device__ double exec(SchedShared& S, const Task& t, double2* sbuf, int slots, int logN, const double2* tq,
                         const Grp& g) const {
    return call_exec_task(S, t, sbuf, slots, logN, tq, g);
  }
};

__global__ void __launch_bounds__(SCHED_THREADS, 1)
call_trap_kernel(CallTrapPricer pr, int32_t* counter, double* __restrict__ ws, int64_t ws_stride) {
  sched_body(pr, 1, counter, ws, ws_stride, pr.flops, nullptr);
}

// ---------------------------------------------------------------------------
// O(T^2) projected backward induction (american_call_backward, _accel.py:62-102).
// Unfused, left-to-right operation order as the reference: bit-identical.

__global__ void __launch_bounds__(CTA_THREADS)
call_baseline_kernel(const CallParams* __restrict__ opts, const int32_t* __restrict__ order, int nwork,
                     double* __restrict__ ws, int64_t ws_stride, BatchOut out) {
  __shared__ int s_fg;
  apply_dlist(out, order, nwork);
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
  const int o = order[w];
  const CallParams P = opts[o];
  const int64_t n = P.n;
  double* a = ws + (int64_t)blockIdx.x * ws_stride;
  double* b = a + (n + 2);
  double* u2 = b + (n + 2);
  const bool rec = out.bt != nullptr;
  if (threadIdx.x == 0) s_fg = INT32_MAX;
  __syncthreads();
  for (int64_t j = threadIdx.x; j <= n; j += CTA_THREADS) {
    const double u = exp(__dmul_rn(__dsub_rn(2.0 * (double)j, (double)n), P.lu));
    u2[j] = u;
    const double v = __dsub_rn(__dmul_rn(P.S, u), P.K);  // leaf_row
    a[j] = v > 0.0 ? v : 0.0;
    if (v > 0.0) atomicMin(&s_fg, (int)j);
  }
  __syncthreads();
  auto put_rec = [&](int64_t row, int fg) {
    if (rec && threadIdx.x == 0 && row < out.cap) {
      out.bt[(int64_t)o * out.cap + row] = row;
      out.bc[(int64_t)o * out.cap + row] = (fg == INT32_MAX) ? INT64_MIN : (int64_t)fg;
    }
  };
  put_rec(n, s_fg);
  __syncthreads();
  for (int64_t i = n - 1; i >= 0; --i) {
    if (threadIdx.x == 0) s_fg = INT32_MAX;
    __syncthreads();
    const double scale = __dmul_rn(P.S, exp((double)(n - i) * P.lu));
    int myfg = INT32_MAX;
    for (int64_t j = threadIdx.x; j <= i; j += CTA_THREADS) {
      const double lin = __dadd_rn(__dmul_rn(P.wd, a[j]), __dmul_rn(P.wu, a[j + 1]));
      const double grn = __dsub_rn(__dmul_rn(scale, u2[j]), P.K);
      if (lin >= grn) {
        b[j] = lin;
      } else {
        b[j] = grn;
        if (myfg == INT32_MAX) myfg = (int)j;
      }
    }
    if (rec) {
      myfg = warp_min_i32(myfg);
      if ((threadIdx.x & 31) == 0 && myfg != INT32_MAX) atomicMin(&s_fg, myfg);
    }
    __syncthreads();
    put_rec(i, s_fg);
    double* t = a;
    a = b;
    b = t;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out.price[o] = a[0];
    out.status[o] = 0;
    if (out.bcount) out.bcount[o] = (int32_t)(n + 1);
  }
  __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// launchers

static cudaError_t call_configure() {
  static std::atomic<unsigned long long> configured{0};
  return once_per_device(configured, [] {
    const int smem = sched_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(call_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(call_trap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return e;
  });
}

int call_chains_per_cta() { return NCHAIN; }

cudaError_t launch_call_fast(const CallParams* opts, const int32_t* order, int nwork, int32_t* counter, double* ws,
                             int64_t ws_stride, int grid, BatchOut out, cudaStream_t stream) {
  cudaError_t e = call_configure();
  if (e != cudaSuccess) return e;
  if (nwork <= 0) return cudaSuccess;
  e = cudaMemsetAsync(counter, 0, sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  call_fast_kernel<<<grid, SCHED_THREADS, sched_smem_bytes(), stream>>>(opts, order, nwork, counter, ws, ws_stride,
                                                                          out);
  return cudaGetLastError();
}

int64_t call_trap_ws_doubles(int64_t width, int64_t h) { return call_arena_doubles(width, h); }

cudaError_t launch_call_trapezoid(const CallParams& P, int64_t i, int64_t j, int64_t first, int64_t h,
                                  const double* run, double* out, int64_t* meta, int32_t* counter, double* ws,
                                  int64_t ws_stride, unsigned long long* flops, cudaStream_t stream) {
  cudaError_t e = call_configure();
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  const CallTrapPricer pr{P, i, j, first, h, run, out, meta, flops};
  call_trap_kernel<<<1, SCHED_THREADS, sched_smem_bytes(), stream>>>(pr, counter, ws, ws_stride);
  return cudaGetLastError();
}

// baseline_american_call(keep_grid=True) (binomial.py:133-158, numpy form):
// every row and its exercise mask retained, rows packed (row i at i(i+1)/2).
// Exercise value S exp((2j - i) lu) - K per cell (the grid variant's formula).
__global__ void __launch_bounds__(CTA_THREADS)
call_grid_kernel(CallParams P, double* __restrict__ rows, uint8_t* __restrict__ masks, int64_t* __restrict__ cols,
                 double* __restrict__ price, double* __restrict__ ws) {
  __shared__ int s_fg;
  const int64_t n = P.n;
  double* a = ws;
  double* b = a + (n + 2);
  if (threadIdx.x == 0) s_fg = INT32_MAX;
  __syncthreads();
  const int64_t base_n = n * (n + 1) / 2;
  for (int64_t j = threadIdx.x; j <= n; j += CTA_THREADS) {
    const double node = __dsub_rn(__dmul_rn(P.S, exp(__dmul_rn(__dsub_rn(2.0 * (double)j, (double)n), P.lu))), P.K);
    const double v = node > 0.0 ? node : 0.0;  // leaf_row
    a[j] = v;
    rows[base_n + j] = v;
    const bool g = v > 0.0;
    masks[base_n + j] = g;
    if (g) atomicMin(&s_fg, (int)j);
  }
  __syncthreads();
  if (threadIdx.x == 0) cols[n] = (s_fg == INT32_MAX) ? INT64_MIN : s_fg;
  for (int64_t i = n - 1; i >= 0; --i) {
    __syncthreads();
    if (threadIdx.x == 0) s_fg = INT32_MAX;
    __syncthreads();
    const int64_t base = i * (i + 1) / 2;
    for (int64_t j = threadIdx.x; j <= i; j += CTA_THREADS) {
      const double lin = __dadd_rn(__dmul_rn(P.wd, a[j]), __dmul_rn(P.wu, a[j + 1]));
      const double grn =
          __dsub_rn(__dmul_rn(P.S, exp(__dmul_rn(__dsub_rn(2.0 * (double)j, (double)i), P.lu))), P.K);
      const bool g = lin < grn;
      const double v = g ? grn : lin;
      b[j] = v;
      rows[base + j] = v;
      masks[base + j] = g;
      if (g) atomicMin(&s_fg, (int)j);
    }
    __syncthreads();
    if (threadIdx.x == 0) cols[i] = (s_fg == INT32_MAX) ? INT64_MIN : s_fg;
    double* t = a;
    a = b;
    b = t;
  }
  if (threadIdx.x == 0) *price = a[0];
}

cudaError_t launch_call_grid(const CallParams& P, double* rows, uint8_t* masks, int64_t* cols, double* price,
                             double* ws, cudaStream_t stream) {
  call_grid_kernel<<<1, CTA_THREADS, 0, stream>>>(P, rows, masks, cols, price, ws);
  return cudaGetLastError();
}

cudaError_t launch_call_baseline(const CallParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                                 double* ws, int64_t ws_stride, BatchOut out, cudaStream_t stream) {
  if (nwork <= 0 || grid <= 0) return cudaSuccess;
  if (n_max + 1 <= sweep_max_cells() && !sweep_disabled()) return launch_call_sweep(opts, order, nwork, n_max, grid, out, stream);
  call_baseline_kernel<<<grid, CTA_THREADS, 0, stream>>>(opts, order, nwork, ws, ws_stride, out);
  return cudaGetLastError();
}

}  // namespace fl
