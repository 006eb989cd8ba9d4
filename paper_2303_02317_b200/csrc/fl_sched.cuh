// fl_sched.cuh -- warp-specialised in-CTA scheduler for the divide-and-conquer
// pricers (the device replacement of the reference's recursion drivers and
// their 2-thread pool, american.py:168-198 / bsm.py:372-399).
//
// CTA layout (warp ids; the issue arbiter favours high ids):
//   warps [0, BIG_WARPS)               "big" group: one task at a time over
//                                      all its threads (named barrier 1)
//   warps [BIG_WARPS, +SMALL_WORKERS)  "small" workers: one warp per task
//   warps [CHAIN_WARP0, +NCHAIN)       chain warps: one option each
// A chain warp walks its option's halving recursion.  It keeps the sequential
// critical path to itself -- the nonlinear strips and, at the two lowest
// levels, whole recursion nodes fused in shared memory -- and ISSUES every
// longer linear jump as a task: into the small ring (one warp: direct dot
// products for kernels up to DIRECT_H, FFT blocks up to 1024 points) or the
// big ring (FFT blocks up to 8192 points).
//
// Tasks of a ring are claimed in issue order but run concurrently and finish
// out of order, so each task carries explicit dependencies: at issue time the
// chain compares the new task's read / write address ranges with those of its
// own unfinished tasks (RAW, WAR, WAW) and records the conflicting ones; a
// worker starts a task only when they are done.  Before touching memory
// itself the chain likewise waits for exactly the unfinished tasks it
// conflicts with, so jumps with slack overlap the strips.  Chains never share
// arena memory, so chains never wait on each other.
#pragma once

#include <cstdint>

#include "fl_common.cuh"
#include "fl_conv.cuh"

namespace fl {

// Warp layout (a warp's SM sub-partition, SMSP, is warp_id % 4):
//   warps 0-3    big FFT group: 8192-point blocks, consumes RING_BIG, then RING_LOW
//   warps 4-7    medium FFT group: 2048-point blocks, consumes RING_SMALL
//   warps 8-9    chain warps
//   warps 10-15  helper warps, three per chain: the chain's private
//                co-processors for the direct correlations of its shared-memory
//                subtrees, fed through a request ring (no deps scan)
// Groups execute one task at a time over 128 threads (named barriers 1, 2).
// (Isolating the chains on SMSPs of their own was measured: no gain.)
#ifndef FL_PROF  // 1: scheduler profile counters (FL_PROFILE=1 at run time); tool builds only --
#define FL_PROF 0  // the counting code enlarges the kernel and costs instruction-cache misses
#endif
#define FL_PROFP(p) (FL_PROF ? (p) : nullptr)
#ifndef FL_STRIP_CLOCK  // tool builds: a few clock64 intervals only (tools/strip_clock.py)
#define FL_STRIP_CLOCK 0
#endif
#if FL_STRIP_CLOCK
#define LCLK_ADD(p, slot, v) \
  do { if ((p) && (threadIdx.x & 31) == 0) atomicAdd((p) + (slot), (unsigned long long)(v)); } while (0)
#else
#define LCLK_ADD(p, slot, v) do { } while (0)
#endif
#ifndef FL_NHELP
#define FL_NHELP 2
#endif
#ifndef FL_PUBLISH_GPU_FENCE  // 1: GPU-scope fence before a task's done flag (measured 0.4-1 % slower)
#define FL_PUBLISH_GPU_FENCE 0
#endif
#ifndef FL_SOLO_HELP  // 1: with one item per CTA all four helpers serve chain 0 (layout 6)
#define FL_SOLO_HELP 1
#endif
constexpr int NCHAIN = 2;
constexpr int NHELP = FL_NHELP;  // helper warps per chain
constexpr int GROUP_WARPS = 4;
constexpr int GROUP_THREADS = 32 * GROUP_WARPS;
constexpr int BIG_WARPS = GROUP_WARPS;
constexpr int BIG_THREADS = GROUP_THREADS;
// layout 4 keeps two warp slots idle so the chains' SMSP holds nothing else
constexpr int IDLE_WARPS = 2;
constexpr int SCHED_WARPS = 2 * GROUP_WARPS + NCHAIN * (1 + NHELP) + IDLE_WARPS;
constexpr int SCHED_THREADS = 32 * SCHED_WARPS;
enum : int { ROLE_CHAIN = 0, ROLE_BIG = 1, ROLE_MED = 2, ROLE_HELPER = 3, ROLE_IDLE = 4 };
// Pricers choose the warp placement (Pricer::kLayout, default 4): layout 4
// puts both chains on SMSP 3 (the put's fixed strip runs best there, the FFT
// groups spread over SMSPs 0-2); layout 6 gives each chain an SMSP of its own
// with its helpers and one FFT group per remaining SMSP (the call's light
// 2-tap strip: C2 3.02 -> 2.88 ms; puts 14 % slower, profiles/r02_experiments.md).
template <class P>
struct LayoutOf {
  template <class Q>
  static constexpr int pick(decltype(Q::kLayout)*) { return Q::kLayout; }
  template <class Q>
  static constexpr int pick(...) { return 4; }
  static constexpr int value = pick<P>(nullptr);
};

template <int LAYOUT = 4>
__device__ __forceinline__ int warp_role(int w, int* rank) {
  // The chains' leaf strips exchange neighbours by shuffle every row, and a
  // shuffle waits behind every shared-memory access queued on its SMSP's MIO
  // path (measured, tools/strip_noise_bench.cu: 68 cycles/row alone, 148 with
  // three conflict-free shared-load warps on the same SMSP, 90 on the other
  // SMSPs).  So both chains share SMSP 3 with nothing else (warps 3, 7; 11 and
  // 15 idle), and the FFT groups and the helpers (two per chain) fill SMSPs 0-2.
  static_assert(NCHAIN == 2 && NHELP == 2 && SCHED_WARPS == 16, "layout 4 shape");
  if (LAYOUT == 6) {
    // each chain on an SMSP of its own with its two helpers (chain 0: SMSP 3,
    // chain 1: SMSP 2), the big group on SMSP 0, the medium group on SMSP 1
    constexpr int kR[16] = {ROLE_BIG, ROLE_MED, ROLE_CHAIN, ROLE_CHAIN, ROLE_BIG, ROLE_MED, ROLE_HELPER, ROLE_HELPER,
                            ROLE_BIG, ROLE_MED, ROLE_HELPER, ROLE_HELPER, ROLE_BIG, ROLE_MED, ROLE_IDLE, ROLE_IDLE};
    constexpr int kK[16] = {0, 0, 1, 0, 1, 1, NHELP + 0, 0, 2, 2, NHELP + 1, 1, 3, 3, 0, 0};
    *rank = kK[w];
    return kR[w];
  }
  if ((w & 3) == 3) {
    if (w < 8) { *rank = w >> 2; return ROLE_CHAIN; }
    *rank = 0;
    return ROLE_IDLE;
  }
  constexpr int kRole[12] = {ROLE_BIG, ROLE_BIG, ROLE_BIG, ROLE_BIG, ROLE_MED, ROLE_MED,
                             ROLE_MED, ROLE_MED, ROLE_HELPER, ROLE_HELPER, ROLE_HELPER, ROLE_HELPER};
  // slot = index among the non-chain warps: 0,1,2 | 4,5,6 | 8,9,10 | 12,13,14
  // big: warps 0,1,2,4; medium: 5,6,8,9; helpers: 10 (chain 0), 12 (chain 1), 13 (chain 0), 14 (chain 1)
  const int slot = (w >> 2) * 3 + (w & 3);
  constexpr int kRank[12] = {0, 1, 2, 3, 0, 1, 2, 3, 0, NHELP + 0, 1, NHELP + 1};
  *rank = kRank[slot];
  return kRole[slot];
  constexpr int C0 = 2 * GROUP_WARPS, H0 = C0 + NCHAIN;
  if (w >= H0) { *rank = w - H0; return ROLE_HELPER; }  // helper rank: chain = rank / NHELP
  if (w >= C0) { *rank = w - C0; return ROLE_CHAIN; }
  if (w < GROUP_WARPS) { *rank = w; return ROLE_BIG; }
  *rank = w - GROUP_WARPS;
  return ROLE_MED;
}

// Request ring between chain warp c and its helpers: direct correlations
// y[k] = sum_r w[r] x[k+r], k < Lout.  Requests posted together are
// independent (the chain waits for a request's inputs before posting it), so
// the helpers take them in posting order and finish them in any order; a
// ticket t is complete when done[t % HQ] >= t.
constexpr int HQ = 16;
struct HReq {
  const double* x;
  double* y;
  const double* w;
  int Lout, M;
};
struct Mailbox {
  HReq q[HQ];
  volatile int done[HQ];
  volatile int seq;  // last posted request
  int claim;         // last claimed request
  volatile int quit;
};

constexpr int NRINGS = 3;
#ifndef FL_QCAP
#define FL_QCAP 64
#endif
#ifndef FL_DIRECT_H  // kernels with h <= FL_DIRECT_H use direct dot products
#define FL_DIRECT_H 64
#endif
#ifndef FL_SMALL_MW  // FFT jumps with a window <= FL_SMALL_MW go to the medium group
#define FL_SMALL_MW 600
#endif
#ifndef FL_IDLE_NS  // longest back-off sleep of an idle worker poll
#define FL_IDLE_NS 2048
#endif
#ifndef FL_HELPER_NS  // longest back-off sleep of an idle helper poll
#define FL_HELPER_NS 512
#endif
constexpr int QCAP = FL_QCAP;  // per ring
constexpr int BIG_BAR = 1;
constexpr int MED_BAR = 2;
constexpr int DIRECT_H = FL_DIRECT_H;  // direct-correlation TASKS for kernels up to this height
#ifndef FL_KT_H  // composed weights W_1..W_KT_H are tabulated per option (subtree correlations)
#define FL_KT_H 128
#endif
constexpr int KT_H = FL_KT_H;
static_assert(KT_H >= DIRECT_H, "direct tasks read the table");
constexpr int BIG_LOGN = 13;                     // big-group FFT blocks <= 8192 real points
constexpr int SMALL_LOGN = 12;  // small-ring FFT blocks <= 4096 real points
constexpr int BIG_SLOTS = smem_complex_slots(1 << (BIG_LOGN - 1));
constexpr int MED_WSLOTS = smem_complex_slots(1 << (SMALL_LOGN - 1));  // one small-ring worker's buffer
constexpr int SMALL_SLOTS = MED_WSLOTS;  // the medium group's buffer
constexpr int NDEP = 6;

enum : int {
  TK_FFT = 0,
  TK_DIRECT = 1,
  TK_EXIT = 3,
  TK_USER = 8,  // pricer-specific tasks start here
};

// RING_LOW: big-group tasks with lots of slack (the stage-level far / left
// jumps), split into chunks and taken only when RING_BIG is empty, so the
// latency-critical mid / bottom jumps never queue behind them.
enum : int { RING_SMALL = 0, RING_BIG = 1, RING_LOW = 2 };
constexpr int64_t LOW_CHUNK = 8192;  // outputs per RING_LOW task

struct Task {
  const double* x;
  double* y;
  const double* w;
  int64_t L, Lout;
  double c0, c1, c2;
  int h, span, kind, chain;
  int64_t i0, i1, i2;
  double d0;
  int ndep;
  int dep[NDEP];     // (ring << 28) | index
  volatile int seq;  // == task index once published
};

struct Pend {  // a chain's record of one of its issued tasks
  int id;      // (ring << 28) | index
  uintptr_t rlo, rhi, wlo, whi;
};

constexpr int PEND_CAP = 64;

struct SchedShared {
  Task ring[NRINGS][QCAP];
  volatile int done[NRINGS][QCAP];  // index of the last finished task in the slot
  int reserve[NRINGS];
  int claim[NRINGS];
  Pend pend[NCHAIN][PEND_CAP];
  int npend[NCHAIN];
  int plo[NCHAIN];  // every pending entry below plo[c] is known finished (scan start)
  double result[NCHAIN];   // per-chain results of blocking tasks
  double result2[NCHAIN];
  int64_t iresult[NCHAIN];
  Mailbox mb[NCHAIN][2];  // per chain: [0] urgent requests, [1] background (subtree root)
  unsigned long long* prof;  // profile counters (null unless FL_PROFILE)
  int chains_left;
  int cw_ids[NCHAIN][8];   // per-chain conflict lists (shared, not per-lane local memory)
  int cw_raw[NCHAIN][8];
  int cw_deps[NCHAIN][NDEP];
  int wkey[NCHAIN][4];     // weight-stash keys per depth (-1: empty)
  int trace_c;  // chain pricing work item 0 (FL_TRACE builds)
  int trace_n;  // words of the trace written
};

// SchedShared lives at the start of dynamic shared memory (16-byte aligned size).
constexpr int SCHED_SHARED_DOUBLES = (int)((sizeof(SchedShared) + 15) / 16) * 2;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uintptr_t U(const void* p) { return reinterpret_cast<uintptr_t>(p); }

// profile counter slots (BatchOut::prof)
enum : int {
  PROF_FFT_CYC = 0, PROF_FFT_N, PROF_DIR_CYC, PROF_DIR_N, PROF_OTHER_CYC, PROF_OTHER_N, PROF_BIG_CYC, PROF_BIG_N,
  PROF_STRIP_CYC, PROF_STRIP_N, PROF_WAIT_CYC, PROF_FUSE_CYC, PROF_FUSE_N, PROF_KERNEL_CYC, PROF_IDLE_CYC,
  PROF_ISS_CYC, PROF_CHAIN_CYC, PROF_DEPWAIT_CYC,
  // detail (chain side)
  PROF_ISS_SCAN, PROF_ISS_STALL, PROF_ISS_SLOT, PROF_F_STAGE, PROF_F_MID, PROF_F_BOT, PROF_STRIP_LOOP,
  PROF_LEAF_LOAD,
  // conflict waits by cause: read-after-write / write-after-read-or-write, small / big ring
  PROF_W_RAW_S, PROF_W_RAW_B, PROF_W_WAR_S, PROF_W_WAR_B, PROF_W_N, PROF_W_SUML, PROF_W_SUMH, PROF_W_FFT,
  PROF_W_MAXL,
  PROF_HELP_CYC = 48, PROF_HELP_CYC_BG, PROF_HELP_FMA, PROF_S_LEAF,
  PROF_TIMELINE = 56,  // 3 words per work item follow the 56 counters (start ns, end ns, SM << 1 | chain)
};

__device__ __forceinline__ void prof_add(unsigned long long* prof, int slot, unsigned long long v) {
  if (FL_PROF && prof) atomicAdd(prof + slot, v);
}

// Event trace of the chain pricing work item 0 (FL_TRACE builds only; a tool,
// never on in the product): pairs (type << 32 | arg, clock64) after a counter.
#ifndef FL_TRACE
#define FL_TRACE 0
#endif
enum : int {
  EV_SUB_B = 1, EV_SUB_E, EV_LEAF_B, EV_LEAF_E, EV_HW_B, EV_HW_E, EV_POST_B, EV_POST_E, EV_CW_B, EV_CW_E,
  EV_IS_B, EV_IS_E, EV_STG_B, EV_STG_E, EV_NODE, EV_OPT_B, EV_OPT_E, EV_TW_B, EV_TW_E, EV_MARK
};
#if FL_TRACE
constexpr int TRACE_CAP = 1 << 21;
__device__ unsigned long long g_trace[TRACE_CAP];
#define FL_TR(S, c, ev, arg)                                                                      \
  do {                                                                                            \
    if ((S).trace_c == (c) && lane_id() == 0) {                                                   \
      const int i_ = (S).trace_n;                                                                 \
      if (i_ + 2 < TRACE_CAP) {                                                                   \
        (S).trace_n = i_ + 2;                                                                     \
        g_trace[i_ + 1] = ((unsigned long long)(ev) << 32) | (unsigned)(arg);                     \
        g_trace[i_ + 2] = (unsigned long long)clock64();                                          \
        g_trace[0] = (unsigned long long)(i_ + 2);                                                \
      }                                                                                           \
    }                                                                                             \
  } while (0)
#else
#define FL_TR(S, c, ev, arg) \
  do {                       \
  } while (0)
#endif

__device__ void sched_init(SchedShared& S) {
  for (int i = threadIdx.x; i < NRINGS * QCAP; i += blockDim.x) {
    const int r = i / QCAP, q = i % QCAP;
    S.ring[r][q].seq = -1;
    S.done[r][q] = q - QCAP;  // "previous generation finished"
  }
  if (threadIdx.x < NRINGS) {
    S.reserve[threadIdx.x] = 0;
    S.claim[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    S.chains_left = NCHAIN;
    S.trace_c = -1;
    S.trace_n = 0;
  }
  if (threadIdx.x < NCHAIN) {
    S.npend[threadIdx.x] = 0;
    S.plo[threadIdx.x] = 0;
    for (int q = 0; q < 2; ++q) {
      Mailbox& m = S.mb[threadIdx.x][q];
      m.seq = 0;
      m.claim = 0;
      m.quit = 0;
      for (int k = 0; k < HQ; ++k) m.done[k] = (k == 0) ? 0 : k - HQ;  // ticket t's slot predecessor t-HQ is done
    }
  }
}

__device__ __forceinline__ bool overlap(uintptr_t a0, uintptr_t a1, uintptr_t b0, uintptr_t b1) {
  return a0 < b1 && b0 < a1;
}

__device__ __forceinline__ bool task_done(const SchedShared& S, int id) {
  const int r = (int)((unsigned)id >> 28), idx = id & 0x0fffffff;
  return S.done[r][idx % QCAP] >= idx;
}

constexpr int HCHUNK = 64;  // outputs per helper request (large correlations are split)

// Chain side of request ring q of chain c (all lanes call): post a correlation
// as chunks of HCHUNK outputs with one publication; returns the last ticket and
// the first in *first (see helper_wait_range).
__device__ __forceinline__ int helper_post(SchedShared& S, int c, int q, const double* x, double* y, int Lout,
                                           const double* w, int M, int* first) {
  Mailbox& m = S.mb[c][q];
  const int t0 = m.seq + 1;
  *first = t0;
  if (Lout <= 0) return t0 - 1;
  FL_TR(S, c, EV_POST_B, Lout * 1024 + M);
  const int n = (Lout + HCHUNK - 1) / HCHUNK;  // <= HQ by construction (Lout <= 2 * PUT_HS)
  const int tl = t0 + n - 1;
  const int lane = lane_id();
  // the slots' previous occupants (t - HQ) must be finished
  while (__any_sync(0xffffffffu, lane < n && m.done[(t0 + lane) % HQ] < t0 + lane - HQ)) __nanosleep(16);
  __threadfence_block();  // every lane's writes to x (shared) ...
  if (lane < n) {
    HReq& r = m.q[(t0 + lane) % HQ];
    const int k0 = lane * HCHUNK;
    r.x = x + k0; r.y = y + k0; r.w = w; r.Lout = (Lout - k0 < HCHUNK) ? Lout - k0 : HCHUNK; r.M = M;
  }
  __syncwarp();           // ... and the requests are written before lane 0 publishes
  if (lane == 0) {
    __threadfence_block();
    m.seq = tl;
  }
  __syncwarp();
  FL_TR(S, c, EV_POST_E, q);
  return tl;
}

__device__ __forceinline__ void helper_wait_range(SchedShared& S, int c, int q, int first, int last) {
  FL_TR(S, c, EV_HW_B, q);
  for (int t = first; t <= last; ++t)
    while (__shfl_sync(0xffffffffu, S.mb[c][q].done[t % HQ], 0) < t) __nanosleep(8);
  __threadfence_block();
  FL_TR(S, c, EV_HW_E, last - first + 1);
}

// All lanes of the calling warp spin (warp-uniform, keeps the warp converged).
__device__ __forceinline__ void warp_wait_done(const SchedShared& S, int id) {
  while (!__shfl_sync(FULL, (int)task_done(S, id), 0)) __nanosleep(32);
  __threadfence_block();
}

// The chain's unfinished tasks conflicting with the given ranges, in issue
// order, into out[0..min(n,cap)); returns n.
__device__ int scan_conflicts(SchedShared& S, int c, uintptr_t r0, uintptr_t r1, uintptr_t r2, uintptr_t r3,
                              uintptr_t w0, uintptr_t w1, int* out, int cap, int* rawf = nullptr) {
  const int np = S.npend[c];
  int first = np > PEND_CAP ? np - PEND_CAP : 0;
  if (S.plo[c] > first) first = S.plo[c];
  int n = 0;
  bool prefix = true;  // entries below the first unfinished one need no more scans
  for (int base = first; base < np; base += 32) {  // warp-uniform trip count
    const int i = base + lane_id();
    bool hit = false, raw = false, live = false;
    int id = 0;
    if (i < np) {
      const Pend& p = S.pend[c][i % PEND_CAP];
      id = p.id;
      live = !task_done(S, id);
      raw = overlap(p.wlo, p.whi, r0, r1) || overlap(p.wlo, p.whi, r2, r3);
      const bool war = overlap(p.rlo, p.rhi, w0, w1) || overlap(p.wlo, p.whi, w0, w1);
      hit = (raw || war) && live;
    }
    if (prefix) {
      const unsigned lv = __ballot_sync(FULL, live);
      const int adv = lv ? __ffs(lv) - 1 : (np - base < 32 ? np - base : 32);
      if (lane_id() == 0) S.plo[c] = base + adv;
      __syncwarp();
      prefix = (lv == 0);
    }
    unsigned m = __ballot_sync(FULL, hit);
    const unsigned rm = __ballot_sync(FULL, raw);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      const int v = __shfl_sync(FULL, id, l);
      if (n < cap) {
        out[n] = v;
        if (rawf) rawf[n] = (rm >> l) & 1;
      }
      ++n;
    }
  }
  return n;
}

// Chain c waits for its unfinished tasks that conflict with a region it is
// about to read (r0/r1, r2/r3) and write (w0/w1).
__device__ void wait_conflicts(SchedShared& S, int c, uintptr_t r0, uintptr_t r1, uintptr_t r2, uintptr_t r3,
                               uintptr_t w0, uintptr_t w1) {
  int* ids = S.cw_ids[c];
  int* rawf = S.cw_raw[c];
  FL_TR(S, c, EV_CW_B, 0);
  for (;;) {
    const int n = scan_conflicts(S, c, r0, r1, r2, r3, w0, w1, ids, 8, rawf);
    if (n == 0) break;
    const int m = n < 8 ? n : 8;
    for (int i = 0; i < m; ++i) {
      const long long t0 = FL_PROFP(S.prof) ? clock64() : 0;
      if (FL_PROFP(S.prof) && lane_id() == 0 && rawf[i]) {
        const int rg = (int)((unsigned)ids[i] >> 28), ix = ids[i] & 0x0fffffff;
        const Task& tk = S.ring[rg][ix % QCAP];
        prof_add(FL_PROFP(S.prof), PROF_W_SUML, (unsigned long long)tk.L);
        prof_add(FL_PROFP(S.prof), PROF_W_SUMH, (unsigned long long)tk.h);
        prof_add(FL_PROFP(S.prof), PROF_W_FFT, tk.kind == TK_FFT ? 1ull : 0ull);
        if ((unsigned long long)tk.L > FL_PROFP(S.prof)[PROF_W_MAXL]) {  // debug: describe the longest waited task
          FL_PROFP(S.prof)[PROF_W_MAXL] = tk.L;
          FL_PROFP(S.prof)[PROF_W_MAXL + 1] = tk.Lout;
          FL_PROFP(S.prof)[PROF_W_MAXL + 2] = tk.h;
          FL_PROFP(S.prof)[PROF_W_MAXL + 3] = (unsigned long long)(tk.y - tk.x);
        }
        // histogram of waited-task h: slots +4 .. +8 for h <= 64, 128, 256, 512, larger
        const int hb = tk.h <= 64 ? 0 : tk.h <= 128 ? 1 : tk.h <= 256 ? 2 : tk.h <= 512 ? 3 : 4;
        prof_add(FL_PROFP(S.prof), PROF_W_MAXL + 4 + hb, 1);
        prof_add(FL_PROFP(S.prof), PROF_W_MAXL + 9 + hb, (unsigned long long)tk.L);
      }
      warp_wait_done(S, ids[i]);
      if (FL_PROFP(S.prof) && lane_id() == 0) {
        const int big = ((unsigned)ids[i] >> 28) == RING_BIG;
        prof_add(FL_PROFP(S.prof), (rawf[i] ? PROF_W_RAW_S : PROF_W_WAR_S) + big, clock64() - t0);
        prof_add(FL_PROFP(S.prof), PROF_W_N, 1);
      }
    }
    if (n <= 8) break;
  }
  __syncwarp();
  FL_TR(S, c, EV_CW_E, 0);
}

// Issue a task from chain warp `c` (all 32 lanes call).  Returns its id.
// rlo/rhi: read range; wlo/whi: write range.
#ifndef FL_ISSUE_CALL  // 1: issue() is a real call, 2: chain_conv() is (one copy of the code instead of 11)
#define FL_ISSUE_CALL 1
#endif
#if FL_ISSUE_CALL == 1
__noinline__
#endif
__device__ int issue(SchedShared& S, int c, int ring, const Task& t, uintptr_t rlo, uintptr_t rhi, uintptr_t wlo,
                     uintptr_t whi) {
  int* deps = S.cw_deps[c];
  int nd;
  FL_TR(S, c, EV_IS_B, ring);
  const long long t0 = FL_PROFP(S.prof) ? clock64() : 0;
  long long t1 = 0, t2 = 0;
  for (;;) {
    nd = scan_conflicts(S, c, rlo, rhi, 0, 0, wlo, whi, deps, NDEP);
    if (FL_PROFP(S.prof) && t1 == 0) t1 = clock64();
    if (nd <= NDEP) break;
    warp_wait_done(S, deps[0]);  // too many: retire the oldest conflict first
  }
#if FL_STRIP_CLOCK  // tool builds: issued tasks per ring and those with no dependency at issue
  if (S.prof && lane_id() == 0) {
    atomicAdd(S.prof + 48 + ring, 1ull);
    if (nd == 0) atomicAdd(S.prof + 52 + ring, 1ull);
  }
#endif
  // keep the pending list from overflowing: wait for the entry about to be overwritten
  {
    const int np = S.npend[c];
    if (np >= PEND_CAP) warp_wait_done(S, S.pend[c][np % PEND_CAP].id);
  }
  __threadfence_block();  // this lane's earlier global writes before the publish
  __syncwarp();
  int idx = 0;
  if (lane_id() == 0) idx = atomicAdd(&S.reserve[ring], 1);
  idx = __shfl_sync(FULL, idx, 0);
  if (FL_PROFP(S.prof)) t2 = clock64();
  // the slot's previous occupant must be finished
  while (!__shfl_sync(FULL, (int)(S.done[ring][idx % QCAP] >= idx - QCAP), 0)) __nanosleep(64);
  if (FL_PROFP(S.prof) && lane_id() == 0) {
    const long long t3 = clock64();
    prof_add(FL_PROFP(S.prof), PROF_ISS_SCAN, t1 - t0);
    prof_add(FL_PROFP(S.prof), PROF_ISS_STALL, t2 - t1);
    prof_add(FL_PROFP(S.prof), PROF_ISS_SLOT, t3 - t2);
  }
  const int id = (ring << 28) | (idx & 0x0fffffff);  // ring in bits 28..31
  if (lane_id() == 0) {
    Task& s = S.ring[ring][idx % QCAP];
    s.x = t.x; s.y = t.y; s.w = t.w; s.L = t.L; s.Lout = t.Lout;
    s.c0 = t.c0; s.c1 = t.c1; s.c2 = t.c2; s.h = t.h; s.span = t.span; s.kind = t.kind; s.chain = c;
    s.i0 = t.i0; s.i1 = t.i1; s.i2 = t.i2;
    s.d0 = t.d0;
#if FL_STRIP_CLOCK  // tool builds: the issue clock rides in d0 of FFT tasks (unused there)
    if (t.kind == TK_FFT) s.d0 = __longlong_as_double(clock64());
#endif
    s.ndep = nd;
    for (int i = 0; i < nd; ++i) s.dep[i] = deps[i];
    Pend& p = S.pend[c][S.npend[c] % PEND_CAP];
    p.id = id; p.rlo = rlo; p.rhi = rhi; p.wlo = wlo; p.whi = whi;
    S.npend[c] += 1;
    __threadfence_block();
    s.seq = idx;
  }
  __syncwarp();
  FL_TR(S, c, EV_IS_E, nd);
  return id;
}

// Chain c waits for all of its issued tasks.
__device__ void wait_all_own(SchedShared& S, int c) {
  const int np = S.npend[c];
  const int first = np > PEND_CAP ? np - PEND_CAP : 0;
  for (int i = first; i < np; ++i) warp_wait_done(S, S.pend[c][i % PEND_CAP].id);
}

// Which ring an FFT correlation goes to (uniform per task): the small ring when
// the kernel's Hoeffding window is at most FL_SMALL_MW columns.  The window
// grows with h, so a chain evaluates the rule once per option as a height
// threshold (small_ring_hmax into Stencil::hsmall: the window formula is a
// double sqrt plus conversions, ~400 cycles of the chain's serial time per
// issued jump otherwise).
__device__ __forceinline__ int fft_ring(const Stencil& st, int h) {
  if (st.hsmall > 0) return h <= st.hsmall ? RING_SMALL : RING_BIG;
  const int64_t Mw = window_width(st, h, nullptr);
  return (Mw <= FL_SMALL_MW) ? RING_SMALL : RING_BIG;
}
// Tallest kernel height sent to the small ring: bisection on the window width,
// then a walk to the exact edge (floor / ceil make the width jitter by a column).
__device__ __forceinline__ int small_ring_hmax(const Stencil& st) {
  int lo = 1, hi = 1 << 14;  // the width at 2^14 is > 1200 for any stencil
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (window_width(st, mid, nullptr) <= FL_SMALL_MW) lo = mid; else hi = mid - 1;
  }
  while (window_width(st, lo + 1, nullptr) <= FL_SMALL_MW) ++lo;
  while (lo > 1 && window_width(st, lo, nullptr) > FL_SMALL_MW) --lo;
  return lo;
}

// ---------------------------------------------------------------------------
// Direct dot products for short kernels: W_1..W_DIRECT_H per option (slot m at
// kc + m*m, m*span+1 doubles), built by repeated real-space convolution with
// the one-step stencil -- all terms nonnegative, ~m ulp relative accuracy
// (tighter than the reference's FFT power).

// Weight stash: the composed weights a shared-memory subtree's correlations
// use, copied from the per-option kernel table (HBM) into shared memory so the
// helpers' taps are shared-memory loads.  Subtree roots are <= 256 high, so
// the node heights at depth d (1..3) are two consecutive values <= 128 / 64 / 32;
// depth d holds W_key, W_key+1 (slots of WST_SZ[d] doubles at WST_OFF[d]).
constexpr int WST_SZ1 = 257, WST_SZ2 = 129, WST_SZ3 = 65;
constexpr int CHAIN_WSTASH = 2 * (WST_SZ1 + WST_SZ2 + WST_SZ3) + 2;
__device__ __forceinline__ int wst_off(int d) { return d == 1 ? 0 : d == 2 ? 2 * WST_SZ1 : 2 * (WST_SZ1 + WST_SZ2); }
__device__ __forceinline__ int wst_sz(int d) { return d == 1 ? WST_SZ1 : d == 2 ? WST_SZ2 : WST_SZ3; }

constexpr int64_t KTABLE_DOUBLES = (int64_t)(KT_H + 2) * (KT_H + 2) * 2;

// scratch: 2*(2*DIRECT_H+2) doubles of shared memory owned by the calling warp.
__device__ void build_kernel_table(double* kc, const Stencil& st, double* scratch) {
  const int lane = lane_id();
  const int span = st.span;
  double* a = scratch;
  double* b = scratch + (2 * KT_H + 2);
  for (int base = 0; base < 2 * KT_H + 2; base += 32) {
    const int i = base + lane;
    if (i < 2 * KT_H + 2) a[i] = (i == 0) ? st.c0 : (i == 1) ? st.c1 : (i == 2 && span == 2) ? st.c2 : 0.0;
  }
  __syncwarp();
  for (int m = 1; m <= KT_H; ++m) {
    const int M = m * span + 1;
    for (int base = 0; base < M; base += 32) {  // store W_m
      const int r = base + lane;
      if (r < M) kc[m * m + r] = a[r];
    }
    if (m == KT_H) break;
    const int M2 = M + span;
    for (int base = 0; base < M2; base += 32) {  // W_{m+1}[r] = sum_t c_t W_m[r-t]
      const int r = base + lane;
      if (r < M2) {
        double s = (r < M) ? st.c0 * a[r] : 0.0;
        if (r >= 1 && r - 1 < M) s = fma(st.c1, a[r - 1], s);
        if (span == 2 && r >= 2 && r - 2 < M) s = fma(st.c2, a[r - 2], s);
        b[r] = s;
      }
    }
    __syncwarp();
    double* t = a;
    a = b;
    b = t;
  }
  __syncwarp();
  __threadfence_block();
}

// Lout <= 64, register-blocked: lane (og = lane / 4, tg = lane % 4) accumulates
// the 8 consecutive outputs 8og .. 8og+7 over the tap quarter
// [tg Q, min(M, (tg+1) Q)), sliding a 12-value window of x through registers
// (4 new x and 4 weights per 4 taps: 32 DFMA per 8 shared loads), then the four
// quarters are summed by a transposed butterfly (6 shuffles; each lane ends
// owning 2 outputs).  Every load is guarded: reads stay inside x[0, Lout+M-1)
// and w[0, M).
__device__ __forceinline__ void conv_direct_blk(const double* __restrict__ x, double* __restrict__ y, int Lout,
                                                const double* __restrict__ w, int M) {
  const int lane = lane_id();
  const int tg = lane & 3, og = lane >> 2;
  const int Q = (M + 3) >> 2;
  const int s = tg * Q;
  const int e = (s + Q < M) ? s + Q : M;
  const int xlen = Lout + M - 1;
  const int xb = 8 * og;
  double acc[8], xw[12];
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    acc[b] = 0.0;
    const int i = xb + s + b;
    xw[b] = (i < xlen) ? x[i] : 0.0;
  }
  for (int r = s; r < e; r += 4) {
    double wv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = xb + r + 8 + j;
      xw[8 + j] = (i < xlen) ? x[i] : 0.0;
      wv[j] = (r + j < e) ? w[r + j] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[b] = fma(wv[j], xw[b + j], acc[b]);
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) xw[b] = xw[b + 4];
  }
  // quarters -> owner lanes: round 1 (xor 1) splits outputs 0-3 / 4-7, round 2 (xor 2) pairs
  const bool b0 = tg & 1, b1 = (tg >> 1) & 1;
  double k4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = b0 ? acc[i] : acc[i + 4];
    const double keep = b0 ? acc[i + 4] : acc[i];
    k4[i] = keep + __shfl_xor_sync(FULL, send, 1);
  }
  double k2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = b1 ? k4[i] : k4[i + 2];
    const double keep = b1 ? k4[i + 2] : k4[i];
    k2[i] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  const int k = xb + 4 * b0 + 2 * b1;
  if (k < Lout) y[k] = k2[0];
  if (k + 1 < Lout) y[k + 1] = k2[1];
}


// conv_direct_blk with the weights held in registers: w normally lives in HBM
// (the per-option kernel table), where one L2 round trip per 4 taps dominated.
// Lane (og, tg) loads the 9 weights w[s + 9 og + i] of its tap quarter up front
// (one round trip per 72 taps), and at tap s + 9c + i takes the weight from
// lane (c, tg) by shuffle.  Taps past the quarter carry weight 0.
__device__ __forceinline__ void conv_direct_reg(const double* __restrict__ x, double* __restrict__ y, int Lout,
                                                const double* __restrict__ w, int M) {
  constexpr int R = 9;  // weights per lane per round (8 lanes x 9 = 72 taps of a quarter)
  const int lane = lane_id();
  const int tg = lane & 3, og = lane >> 2;
  const int Q = (M + 3) >> 2;
  const int s = tg * Q;
  const int e = (s + Q < M) ? s + Q : M;
  const int xlen = Lout + M - 1;
  const int xb = 8 * og;
  double acc[8], xw[8 + R - 1];
#pragma unroll
  for (int b = 0; b < 8; ++b) acc[b] = 0.0;
#pragma unroll
  for (int b = 0; b < 7; ++b) {
    const int i = xb + s + b;
    xw[b] = (i < xlen) ? x[i] : 0.0;
  }
  for (int r0 = s; r0 < s + Q; r0 += 8 * R) {
    double wr[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = r0 + R * og + i;
      wr[i] = (r < e) ? w[r] : 0.0;
    }
    const int nblk = (s + Q - r0 + R - 1) / R < 8 ? (s + Q - r0 + R - 1) / R : 8;
    for (int c = 0; c < nblk; ++c) {
      const int rb = r0 + R * c;  // first tap of this block; window holds x[xb + rb .. xb + rb + 6]
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int ix = xb + rb + 7 + i;
        xw[7 + i] = (ix < xlen) ? x[ix] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const double wv = __shfl_sync(FULL, wr[i], (c << 2) | tg);
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[b] = fma(wv, xw[b + i], acc[b]);
      }
#pragma unroll
      for (int b = 0; b < 7; ++b) xw[b] = xw[b + R];
    }
  }
  const bool b0 = tg & 1, b1 = (tg >> 1) & 1;
  double k4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = b0 ? acc[i] : acc[i + 4];
    const double keep = b0 ? acc[i + 4] : acc[i];
    k4[i] = keep + __shfl_xor_sync(FULL, send, 1);
  }
  double k2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = b1 ? k4[i] : k4[i + 2];
    const double keep = b1 ? k4[i + 2] : k4[i];
    k2[i] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  const int k = xb + 4 * b0 + 2 * b1;
  if (k < Lout) y[k] = k2[0];
  if (k + 1 < Lout) y[k + 1] = k2[1];
}

__device__ double warp_conv_direct(const double* __restrict__ x, double* __restrict__ y, int64_t Lout,
                                   const double* __restrict__ w, int M) {
  for (int64_t k0 = 0; k0 < Lout; k0 += 64)
    conv_direct_blk(x + k0, y + k0, (Lout - k0 < 64) ? (int)(Lout - k0) : 64, w, M);
  __syncwarp();
  return 2.0 * (double)Lout * (double)M;
}

// Stage n doubles from global into warp-owned shared memory (all loads in
// flight), zero-filling up to n_total (warp_conv_direct reads 3 past its window).
// Loads are batched 8 per lane into registers before the stores, so a stage of
// up to 256 values costs one memory round trip (a load / store interleave
// would serialise on possible aliasing).
template <int NB>
__device__ __forceinline__ void warp_stage_nb(double* __restrict__ dst, const double* __restrict__ src, int n,
                                              int n_total) {
  if (n_total < n) n_total = n;
  const int lane = lane_id();
  for (int base = 0; base < n_total; base += 32 * NB) {
    double v[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int i = base + 32 * k + lane;
      v[k] = (i < n) ? src[i] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int i = base + 32 * k + lane;
      if (i < n_total) dst[i] = v[k];
    }
  }
  __syncwarp();
}
__device__ __forceinline__ void warp_stage(double* dst, const double* src, int n, int n_total = -1) {
  warp_stage_nb<8>(dst, src, n, n_total);
}

#ifndef FL_STAGE_UNROLL
#define FL_STAGE_UNROLL 1
#endif
constexpr int kStageUnroll = FL_STAGE_UNROLL;
// Asynchronous warp_stage: 8-byte cp.async copies global -> shared (zero-fill
// from n to n_total), no register staging and every copy in flight at once.
// The data may be read only after warp_stage_wait().
__device__ __forceinline__ void warp_stage_async(double* dst, const double* src, int n, int n_total = -1) {
  if (n_total < n) n_total = n;
  // not unrolled: the callers' lengths are compile-time constants, and a fully
  // unrolled copy (33 iterations at a 256-row subtree) is ~40 KB of straight-line
  // code in the persistent kernel (instruction-cache footprint)
#pragma unroll kStageUnroll
  for (int i = lane_id(); i < n_total; i += 32) {
    const unsigned da = (unsigned)__cvta_generic_to_shared(dst + i);
    const int sz = (i < n) ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(da), "l"(src + (sz ? i : 0)), "r"(sz)
                 : "memory");
  }
}
__device__ __forceinline__ void warp_stage_wait() {
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
}

// A linear jump issued by chain c: a direct-dot-product task (h <= DIRECT_H)
// or an FFT task, on the small or big ring.
#if FL_ISSUE_CALL == 2
__noinline__
#endif
__device__ void chain_conv(SchedShared& S, int c, const Stencil& st, const double* x, int64_t L, double* y,
                           int64_t Lout, int h, const double* kc, unsigned long long* prof, bool low = false) {
  if (Lout <= 0) return;
  Task t;
  t.c0 = st.c0; t.c1 = st.c1; t.c2 = st.c2; t.span = st.span; t.h = h;
  t.i0 = t.i1 = t.i2 = 0;
  t.d0 = 0.0;
  t.x = x; t.L = L; t.y = y; t.Lout = Lout;
  const long long t0 = clock64();
  if (h <= DIRECT_H && L <= 1024) {
    t.kind = TK_DIRECT;
    t.w = kc + (int64_t)h * h;
    issue(S, c, RING_SMALL, t, U(x), U(x + L), U(y), U(y + Lout));
  } else {
    t.kind = TK_FFT;
    t.w = nullptr;
    const int ring = fft_ring(st, h);
    if (low && ring == RING_BIG) {
      const int64_t span = L - Lout;  // taps - 1
      for (int64_t k0 = 0; k0 < Lout; k0 += LOW_CHUNK) {
        const int64_t n = (Lout - k0 < LOW_CHUNK) ? Lout - k0 : LOW_CHUNK;
        t.x = x + k0; t.L = n + span; t.y = y + k0; t.Lout = n;
        issue(S, c, RING_LOW, t, U(t.x), U(t.x + t.L), U(t.y), U(t.y + n));
      }
    } else {
      issue(S, c, ring, t, U(x), U(x + L), U(y), U(y + Lout));
    }
  }
  if (prof && lane_id() == 0) prof_add(prof, PROF_ISS_CYC, clock64() - t0);
  LCLK_ADD(prof, PROF_ISS_CYC, clock64() - t0);
}

// Worker side: wait until slot `idx` of `ring` is published and its deps are done
// (warp-uniform; called by one warp).
__device__ __forceinline__ void worker_wait_ready(SchedShared& S, int ring, int idx) {
  Task& s = S.ring[ring][idx % QCAP];
  // idle poll with exponential backoff: spinning warps steal issue slots and
  // shared-memory (MIO) bandwidth from the chains' shuffles
  unsigned ns = 16;
  while (__shfl_sync(FULL, s.seq, 0) != idx) {
    __nanosleep(ns);
    ns = ns < FL_IDLE_NS ? 2 * ns : ns;
  }
  __threadfence_block();
  const int nd = s.ndep;
  for (int i = 0; i < nd; ++i) warp_wait_done(S, s.dep[i]);
}

__device__ __forceinline__ Task load_task(const Task& s) {
  Task t;
  t.x = s.x; t.y = s.y; t.w = s.w; t.L = s.L; t.Lout = s.Lout;
  t.c0 = s.c0; t.c1 = s.c1; t.c2 = s.c2; t.h = s.h; t.span = s.span; t.kind = s.kind;
  t.chain = s.chain; t.i0 = s.i0; t.i1 = s.i1; t.i2 = s.i2;
  t.d0 = s.d0;
  t.ndep = 0;
  return t;
}

__device__ __forceinline__ void publish_done(SchedShared& S, int ring, int idx) {
#if FL_PUBLISH_GPU_FENCE
  __threadfence();
#else
  // every consumer of a task's outputs (the chains, their helpers, later tasks'
  // workers) is a warp of this CTA, and the host reads only after the kernel
  // ends: a CTA-scope fence orders the outputs before the done flag (a GPU-scope
  // fence waits for the L2 acknowledgement of every store, on the group's
  // critical path between two tasks)
  __threadfence_block();
#endif
  S.done[ring][idx % QCAP] = idx;
}

// Make the composed weights of every correlation of a shared-memory subtree
// rooted at height h0 resident in the chain's stash (asynchronous copies: the
// caller's warp_stage_wait() precedes any use): each internal node at
// depth d-1 correlates with W_m of its children's heights m (depth d), two
// consecutive values per depth.  Slots are reused while they cover the
// subtree (consecutive subtrees mostly share heights).
__device__ void stash_weights(SchedShared& S, int c, double* wst, const double* kc, int h0, int leaf, int span) {
  for (int d = 1; d <= 3; ++d) {
    const int pmax = (h0 + (1 << (d - 1)) - 1) >> (d - 1);  // tallest node at depth d-1
    if (pmax <= leaf) break;                                // depth d-1 is all leaves
    const int lo = h0 >> d, hi = (h0 + (1 << d) - 1) >> d;
    const int key = S.wkey[c][d];
    if (key >= 0 && lo >= key && hi <= key + 1) continue;
    for (int j = 0; j < 2; ++j) {
      const int m = lo + j;
      if (m > KT_H) break;
      warp_stage_async(wst + wst_off(d) + j * wst_sz(d), kc + (int64_t)m * m, m * span + 1);
    }
    if (lane_id() == 0) S.wkey[c][d] = lo;
    __syncwarp();
  }
}
__device__ __forceinline__ const double* wslot(const SchedShared& S, int c, const double* wst, int d, int m) {
  return wst + wst_off(d) + (m - S.wkey[c][d]) * wst_sz(d);
}

// Execute a generic task on a worker group; returns executed flops (or < 0 on error).
// sbuf: the group's shared buffer (slots double2).
__device__ double exec_generic(const Task& t, double2* sbuf, int slots, int logNmax, const double2* tq,
                               const Grp& g) {
  const Stencil st{t.c0, t.c1, t.c2, t.span};
  if (t.kind == TK_FFT) return conv_fft(t.x, t.L, t.y, t.Lout, t.h, st, sbuf, logNmax, tq, g);
  // TK_DIRECT: the group's first warp, x and weights staged in shared memory
  if (g.t >= 32) return 0.0;
  const int M = t.h * t.span + 1;
  double* sx = (double*)sbuf;
  double* sw = sx + 2 * slots - M - 8;
  warp_stage(sw, t.w, M);
  double fl = 0.0;
  const int64_t chunk = 2 * slots - 2 * M - 16;  // x values per staged chunk (+4 zero pad fits)
  for (int64_t k0 = 0; k0 < t.Lout; k0 += chunk - M + 1) {
    const int64_t nk = (t.Lout - k0 < chunk - M + 1) ? (t.Lout - k0) : (chunk - M + 1);
    warp_stage(sx, t.x + k0, (int)(nk + M - 1), (int)(nk + M + 3));
    fl += warp_conv_direct(sx, t.y + k0, nk, sw, M);
  }
  return fl;
}

// ---------------------------------------------------------------------------
// The persistent kernel body shared by the pricers.
//
// Pricer interface:
//   __device__ void chain(SchedShared& S, int c, int w, double* arena, double* scratch, double* flops) const;
//       price work item w on chain warp c (all 32 lanes call; scratch: CHAIN_SCRATCH
//       doubles of shared memory owned by the warp, arena: the chain's HBM workspace)
//   __device__ double exec(SchedShared& S, const Task& t, double2* sbuf, int slots, int logN,
//                          const double2* tq, const Grp& g) const;
//       execute one task (pricer-specific kinds, else exec_generic)

constexpr int CHAIN_SCRATCH = 2480;  // doubles of shared-memory scratch per chain warp
// The chain's recursion frame stacks live in shared memory after the scratch:
// one copy per warp (a per-thread local-memory stack is 32 copies that the FFT
// groups' streaming evicts from L1, costing an L2 round trip per frame access).
constexpr int CHAIN_FRAME_DOUBLES = 288;
constexpr int FRAME_SUB_OFF = 0;      // bytes: subtree walk (put_subtree / call_subtree)
constexpr int FRAME_SOLVE_OFF = 384;  // bytes: the halving recursion above the subtrees
constexpr int CHAIN_SMEM = CHAIN_SCRATCH + CHAIN_FRAME_DOUBLES + CHAIN_WSTASH;
__device__ __forceinline__ double* chain_wstash(double* scratch) { return scratch + CHAIN_SCRATCH + CHAIN_FRAME_DOUBLES; }
template <class F>
__device__ __forceinline__ F* chain_frames(double* scratch, int off_bytes) {
  return reinterpret_cast<F*>(reinterpret_cast<char*>(scratch + CHAIN_SCRATCH) + off_bytes);
}

__host__ __device__ constexpr int sched_smem_bytes() {
  return (SCHED_SHARED_DOUBLES + NCHAIN * CHAIN_SMEM) * (int)sizeof(double) +
         (TWQ + BIG_SLOTS + SMALL_SLOTS) * (int)sizeof(double2);
}

template <class Pricer>
__device__ __forceinline__ void sched_body(const Pricer& pr, int nwork, int32_t* counter, double* ws,
                                           int64_t ws_stride, unsigned long long* flops_out,
                                           unsigned long long* prof) {
  extern __shared__ double2 sdyn_raw[];
  // dynamic shared memory: scheduler state | chain scratch | twiddles | FFT buffers
  SchedShared& S = *reinterpret_cast<SchedShared*>(sdyn_raw);
  double* chain_scratch = reinterpret_cast<double*>(sdyn_raw) + SCHED_SHARED_DOUBLES;
  double2* tq = reinterpret_cast<double2*>(chain_scratch + NCHAIN * CHAIN_SMEM);  // quarter-wave twiddles
  double2* bigbuf = tq + TWQ;              // big-group FFT buffer
  double2* medbuf = bigbuf + BIG_SLOTS;   // medium-group FFT buffer
  __shared__ int s_idx[2], s_ring[2];
  for (int i = threadIdx.x; i < TWQ; i += blockDim.x) tq[i] = fl_tw[i];
  sched_init(S);
  if (threadIdx.x == 0) S.prof = prof;
  __syncthreads();
  int rank = 0;
  const int role = warp_role<LayoutOf<Pricer>::value>(threadIdx.x >> 5, &rank);
  if (role == ROLE_IDLE) return;
  if (role == ROLE_HELPER) {
    // ---- helper warp of chain rank / NHELP: correlations from the chain's
    // request rings, urgent ring first (claims by CAS: never commit to an
    // unposted ticket while the other ring has work)
    // a batch that runs one item per CTA (chain 0 only, see below) gives chain 0
    // the idle chain's helpers as well -- on layout 6 only (calls at 128 options:
    // 2.17 -> 2.07 ms; on layout 4 the two extra pollers cost the puts 1 %)
    const int cc = (FL_SOLO_HELP && LayoutOf<Pricer>::value == 6 && nwork <= (int)gridDim.x) ? 0 : rank / NHELP;
    double flops = 0.0;
    unsigned ns = 8;
    for (;;) {
      int q = -1, t = 0;
      if (lane_id() == 0) {
        for (int k = 0; k < 2 && q < 0; ++k) {
          Mailbox& mm = S.mb[cc][k];
          const int cl = *(volatile int*)&mm.claim;
          if (cl < mm.seq && atomicCAS(&mm.claim, cl, cl + 1) == cl) { q = k; t = cl + 1; }
        }
      }
      q = __shfl_sync(FULL, q, 0);
      if (q < 0) {
        if (__shfl_sync(FULL, S.mb[cc][0].quit, 0)) break;
        __nanosleep(ns);
        ns = ns < FL_HELPER_NS ? 2 * ns : ns;
        continue;
      }
      ns = 8;
      t = __shfl_sync(FULL, t, 0);
      Mailbox& m = S.mb[cc][q];
      __threadfence_block();
      const volatile HReq& r = m.q[t % HQ];
      const double* x = r.x;
      double* y = r.y;
      const double* w = r.w;
      const int Lout = r.Lout, M = r.M;
      const long long th = clock64();
      flops += warp_conv_direct(x, y, Lout, w, M);
      __threadfence_block();
      __syncwarp();
      if (lane_id() == 0) {
        m.done[t % HQ] = t;
        prof_add(prof, PROF_HELP_CYC + q, clock64() - th);
        prof_add(prof, PROF_HELP_FMA, (unsigned long long)Lout * M);
      }
    }
    if (lane_id() == 0 && flops_out) atomicAdd(flops_out, (unsigned long long)flops);
    return;
  }
  if (role == ROLE_CHAIN) {
    // ---- chain warps
    const int c = rank;
    double* arena = ws + ((int64_t)blockIdx.x * NCHAIN + c) * ws_stride;
    double chain_flops = 0.0;
    // A batch with no more items than CTAs runs one item per CTA on chain 0
    // (an option alone on an SM runs ~1.5x faster than a co-resident pair);
    // otherwise chains claim items dynamically in decreasing-cost order.
    const bool solo = nwork <= (int)gridDim.x;
    bool taken = false;
    for (;;) {
      int w = 0;
      if (solo) {
        if (taken || c != 0) break;
        w = (int)blockIdx.x;
        taken = true;
      } else {
        if (lane_id() == 0) w = atomicAdd(counter, 1);
        w = __shfl_sync(FULL, w, 0);
      }
      if (w >= nwork) break;
      unsigned long long ts = 0;
      if (FL_PROFP(prof)) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
#if FL_TRACE
      if (lane_id() == 0) S.trace_c = (w == 0) ? c : (S.trace_c == c ? -1 : S.trace_c);
      __syncwarp();
#endif
      FL_TR(S, c, EV_OPT_B, w);
      pr.chain(S, c, w, arena, chain_scratch + c * CHAIN_SMEM, &chain_flops);
      FL_TR(S, c, EV_OPT_E, w);
      if (FL_PROFP(prof) && lane_id() == 0) {  // timeline of work item w: start / end ns, SM and chain
        unsigned long long te, sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(te));
        asm volatile("{ .reg .u32 r; mov.u32 r, %%smid; cvt.u64.u32 %0, r; }" : "=l"(sm));
        unsigned long long* tl = prof + PROF_TIMELINE + 3 * (int64_t)w;
        tl[0] = ts; tl[1] = te; tl[2] = (sm << 1) | (unsigned long long)c;
      }
    }
    if (lane_id() == 0) {  // release this chain's helper (all its requests were waited for)
      __threadfence_block();
      S.mb[c][0].quit = 1;
    }
    if (lane_id() == 0 && flops_out) atomicAdd(flops_out, (unsigned long long)chain_flops);
    int last = 0;
    if (lane_id() == 0) last = (atomicSub(&S.chains_left, 1) == 1);
    last = __shfl_sync(FULL, last, 0);
    if (last) {
      // last chain out: one EXIT for each group
      Task t;
      t.kind = TK_EXIT;
      t.x = nullptr; t.y = nullptr; t.w = nullptr; t.L = t.Lout = 0;
      t.c0 = t.c1 = t.c2 = 0.0; t.h = 0; t.span = 0;
      t.i0 = t.i1 = t.i2 = 0; t.d0 = 0.0;
      issue(S, c, RING_SMALL, t, 0, 0, 0, 0);
      issue(S, c, RING_BIG, t, 0, 0, 0, 0);
    }
    return;
  }
  // ---- FFT groups: one task at a time over 128 threads; each group is the
  // only consumer of its rings (the big group: RING_BIG, then RING_LOW; the
  // medium group: RING_SMALL), so claims need no atomics
  double flops = 0.0;
  const long long t_start = clock64();
  const int gi = (role == ROLE_BIG) ? 0 : 1;
  const Grp g{rank * 32 + lane_id(), GROUP_THREADS, gi == 0 ? BIG_BAR : MED_BAR};
  double2* buf = gi == 0 ? bigbuf : medbuf;
  const int slots = gi == 0 ? BIG_SLOTS : SMALL_SLOTS;
  const int logN = gi == 0 ? BIG_LOGN : SMALL_LOGN;
  // claim order: the big group RING_BIG, RING_LOW, then the medium group's
  // RING_SMALL (idle big-group time absorbs small-ring queueing);
  // the medium group RING_SMALL only
  const int r_hi = gi == 0 ? RING_BIG : RING_SMALL;
  const int r_2 = gi == 0 ? RING_LOW : -1;
  const int r_3 = gi == 0 ? RING_SMALL : -1;
  constexpr int NCLAIM = 3;
  for (;;) {
    const long long t0 = clock64();
    if (rank == 0) {
      int ring = -1, idx = 0;
      unsigned ns = 16;
      for (;;) {
        // take the head of RING_hi if it is published and its dependencies are
        // done, else the head of RING_lo if so: never commit to a task that
        // waits on a task queued behind it in this group's own rings (the
        // earliest-issued head always becomes ready, so this cannot deadlock)
        int r = -1, i = 0;
        if (lane_id() == 0) {
          for (int k = 0; k < NCLAIM && r < 0; ++k) {
            const int rr = k == 0 ? r_hi : k == 1 ? r_2 : r_3;
            if (rr < 0) continue;
            const int ii = *(volatile int*)&S.claim[rr];
            if (ii >= *(volatile int*)&S.reserve[rr]) continue;
            const Task& sl = S.ring[rr][ii % QCAP];
            if (sl.seq != ii) continue;  // reserved, not yet published
            __threadfence_block();
            if (rr == RING_SMALL && gi == 0 && sl.kind == TK_EXIT) continue;  // the medium group's own exit
            bool ready = true;
            for (int d = 0; d < sl.ndep; ++d) ready = ready && task_done(S, sl.dep[d]);
            if (!ready) continue;
            if (rr == RING_SMALL) {  // two consumers: claim by CAS
              if (atomicCAS(&S.claim[rr], ii, ii + 1) == ii) { r = rr; i = ii; }
            } else {
              r = rr;
              i = ii;
              S.claim[rr] = ii + 1;
            }
          }
        }
        r = __shfl_sync(FULL, r, 0);
        if (r >= 0) { ring = r; idx = __shfl_sync(FULL, i, 0); break; }
        __nanosleep(ns);
        ns = ns < FL_IDLE_NS ? 2 * ns : ns;
      }
      worker_wait_ready(S, ring, idx);
      if (lane_id() == 0) { s_idx[gi] = idx; s_ring[gi] = ring; }
    }
    gsync(g);
    const int idx = s_idx[gi], tring = s_ring[gi];
    const Task t = load_task(S.ring[tring][idx % QCAP]);
    const long long t1 = clock64();
    if (g.t == 0) prof_add(prof, PROF_IDLE_CYC, t1 - t0);
    if (t.kind == TK_EXIT) break;
#if FL_STRIP_CLOCK  // tool builds: queue delay (issue -> claim) and service time per ring
    const long long tq0 = t.kind == TK_FFT ? __double_as_longlong(t.d0) : t1;
#endif
    // a stolen small-ring task runs with the medium group's block plan (same
    // arithmetic whichever group executes it)
    const bool stolen = (gi == 0 && tring == RING_SMALL);
    const double fl = pr.exec(S, t, buf, stolen ? SMALL_SLOTS : slots, stolen ? SMALL_LOGN : logN, tq, g);
    flops += fl > 0 ? fl : 0.0;
    gsync(g);
#if FL_STRIP_CLOCK
    if (g.t == 0 && prof && t.kind == TK_FFT) {
      const int sl = 36 + 4 * tring;  // per ring: queue, service, count, stolen count
      atomicAdd(prof + sl, (unsigned long long)(t1 - tq0));
      atomicAdd(prof + sl + 1, (unsigned long long)(clock64() - t1));
      atomicAdd(prof + sl + 2, 1ull);
      if (gi == 0 && tring == RING_SMALL) atomicAdd(prof + sl + 3, 1ull);
    }
#endif
    if (g.t == 0) {
      publish_done(S, tring, idx);
      if (FL_PROFP(prof)) {
        const int ps = gi == 0 ? PROF_BIG_CYC
                               : (t.kind == TK_FFT) ? PROF_FFT_CYC : (t.kind == TK_DIRECT) ? PROF_DIR_CYC : PROF_OTHER_CYC;
        prof_add(prof, ps, clock64() - t1);
        prof_add(prof, ps + 1, 1);
      }
    }
  }
  if (g.t == 0) {
    if (flops_out) atomicAdd(flops_out, (unsigned long long)flops);
    prof_add(prof, PROF_KERNEL_CYC, clock64() - t_start);
  }
}

}  // namespace fl
