// fl_sched.cuh -- warp-specialised in-CTA scheduler for the divide-and-conquer
// pricers (the device replacement of the reference's recursion drivers and
// their 2-thread pool, american.py:168-198 / bsm.py:372-399).
//
// A CTA holds NCHAIN "chain" warps and a group of worker warps.  Each chain
// warp owns one option at a time and walks its halving recursion: it runs
// the nonlinear strips itself (the sequential critical path) and ISSUES every
// linear jump (valid-mode correlation with a composed stencil) as a task into
// a shared FIFO ring.  The worker group drains the ring in order, all worker
// threads cooperating on one task (FFT or direct executor, fl_conv.cuh).
//
// Ordering: tasks execute in issue order, so task->task dependencies (RAW /
// WAR / WAW through the option's HBM arena) hold by construction.  A chain
// touching memory itself (a strip) first waits for those of its own pending
// tasks whose read / write address ranges conflict with the strip's -- and
// only those, so linear jumps with slack run concurrently with the strips.
// Chains never share arena memory, so chains never wait on each other.
#pragma once

#include <cstdint>

#include "fl_common.cuh"
#include "fl_conv.cuh"

namespace fl {

constexpr int NCHAIN = 2;
constexpr int NWORKER_WARPS = 8;
constexpr int WORKERS = 32 * NWORKER_WARPS;
constexpr int SCHED_THREADS = 32 * (NCHAIN + NWORKER_WARPS);
constexpr int QCAP = 64;
constexpr int WORKER_BAR = 1;
constexpr int DIRECT_H = 64;  // kernels with h <= DIRECT_H use the direct executor
constexpr int SCHED_LOGN_MAX = 13;
constexpr int SCHED_SLOTS = smem_complex_slots(1 << (SCHED_LOGN_MAX - 1));

enum : int {
  TK_FFT = 0,
  TK_DIRECT = 1,
  TK_KBUILD = 2,
  TK_EXIT = 3,
  TK_USER = 8,  // pricer-specific tasks start here
};

struct Task {
  const double* x;
  double* y;
  const double* w;
  int64_t L, Lout;
  double c0, c1, c2;
  int h, span, kind, chain;
  int64_t i0, i1, i2, i3;
  double d0, d1, d2, d3, d4;
  volatile int seq;  // == task index once published
};

struct Pend {  // a chain's record of one of its issued tasks (address ranges)
  int idx;
  uintptr_t rlo, rhi, wlo, whi;
};

struct SchedShared {
  Task ring[QCAP];
  Pend pend[NCHAIN][QCAP];
  int npend[NCHAIN];
  double result[NCHAIN];
  int reserve;
  volatile int done;
  int chains_left;
  int64_t kcache_epoch[NCHAIN];
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// profile counter slots (BatchOut::prof)
enum : int {
  PROF_FFT_CYC = 0, PROF_FFT_N, PROF_DIR_CYC, PROF_DIR_N, PROF_KB_CYC, PROF_KB_N, PROF_OTHER_CYC, PROF_OTHER_N,
  PROF_STRIP_CYC, PROF_STRIP_N, PROF_WAIT_CYC, PROF_WAIT_N, PROF_ISSUE_CYC, PROF_KERNEL_CYC, PROF_IDLE_CYC,
  PROF_FFT_LOUT, PROF_DIR_LOUT, PROF_CHAIN_CYC, PROF_QFULL_CYC, PROF_DIVERGED,
};

__device__ __forceinline__ void prof_add(unsigned long long* prof, int slot, unsigned long long v) {
  if (prof) atomicAdd(prof + slot, v);
}

__device__ void sched_init(SchedShared& S) {
  for (int i = threadIdx.x; i < QCAP; i += blockDim.x) S.ring[i].seq = -1;
  if (threadIdx.x == 0) {
    S.reserve = 0;
    S.done = 0;
    S.chains_left = NCHAIN;
  }
  if (threadIdx.x < NCHAIN) S.npend[threadIdx.x] = 0;
}

__device__ __forceinline__ bool overlap(uintptr_t a0, uintptr_t a1, uintptr_t b0, uintptr_t b1) {
  return a0 < b1 && b0 < a1;
}

// Issue a task from chain warp `c` (all 32 lanes call).  rd / wr: byte ranges
// the task reads / writes (for the chain's own conflict checks).  Returns the
// task index.
__device__ int issue(SchedShared& S, int c, const Task& t, uintptr_t rlo, uintptr_t rhi, uintptr_t wlo,
                     uintptr_t whi) {
  __threadfence_block();  // this lane's earlier global writes before the publish
  __syncwarp();
  int idx = 0;
  if (lane_id() == 0) idx = atomicAdd(&S.reserve, 1);
  idx = __shfl_sync(FULL, idx, 0);
  // warp-uniform spin (a lane-0-only loop would leave the warp split)
  while (idx - __shfl_sync(FULL, S.done, 0) >= QCAP) __nanosleep(64);
  if (lane_id() == 0) {
    Task& s = S.ring[idx % QCAP];
    s.x = t.x; s.y = t.y; s.w = t.w; s.L = t.L; s.Lout = t.Lout;
    s.c0 = t.c0; s.c1 = t.c1; s.c2 = t.c2; s.h = t.h; s.span = t.span; s.kind = t.kind; s.chain = c;
    s.i0 = t.i0; s.i1 = t.i1; s.i2 = t.i2; s.i3 = t.i3;
    s.d0 = t.d0; s.d1 = t.d1; s.d2 = t.d2; s.d3 = t.d3; s.d4 = t.d4;
    Pend& p = S.pend[c][S.npend[c] % QCAP];
    p.idx = idx; p.rlo = rlo; p.rhi = rhi; p.wlo = wlo; p.whi = whi;
    S.npend[c] += 1;
    __threadfence_block();
    s.seq = idx;
  }
  __syncwarp();
  return idx;
}

// Chain waits until task `idx` (and so every earlier task) has completed.
__device__ __forceinline__ void wait_task(SchedShared& S, int idx) {
  while (__shfl_sync(FULL, S.done, 0) <= idx) __nanosleep(32);  // warp-uniform spin
  __threadfence_block();
}

// Chain c waits for its pending tasks that conflict with a region it is about
// to read (r0/r1, r2/r3) and write (w0/w1).
__device__ void wait_conflicts(SchedShared& S, int c, uintptr_t r0, uintptr_t r1, uintptr_t r2, uintptr_t r3,
                               uintptr_t w0, uintptr_t w1) {
  const int done = S.done;
  const int np = S.npend[c];
  int need = -1;
  const int first = np > QCAP ? np - QCAP : 0;
  // warp-uniform trip count: keeps the chain warp converged (a lane-dependent
  // loop bound here splits the warp and sends later shuffles down the slow
  // collective path)
  for (int base = first; base < np; base += 32) {
    const int i = base + lane_id();
    if (i < np) {
      const Pend& p = S.pend[c][i % QCAP];
      const bool live = p.idx >= done;
      const bool raw = overlap(p.wlo, p.whi, r0, r1) || overlap(p.wlo, p.whi, r2, r3);
      const bool war = overlap(p.rlo, p.rhi, w0, w1) || overlap(p.wlo, p.whi, w0, w1);
      if (live && (raw || war) && p.idx > need) need = p.idx;
    }
  }
  need = __reduce_max_sync(FULL, need);
  if (need >= 0) wait_task(S, need);
  __syncwarp();
}

// Chain c waits for all of its issued tasks.
__device__ void wait_all_own(SchedShared& S, int c) {
  const int np = S.npend[c];
  if (np == 0) return;
  const int last = S.pend[c][(np - 1) % QCAP].idx;
  wait_task(S, last);
}

__device__ __forceinline__ uintptr_t U(const void* p) { return reinterpret_cast<uintptr_t>(p); }

// Issue y[0..Lout) = valid correlation of x[0..L) with W_h (chooses the executor;
// builds the direct weights on first use).  kc: this chain's kernel cache
// (slot h at kc + h*h, (h*span+1) doubles); kbuilt: per-h flags in smem;
// delta: zero buffer with 1.0 at index DIRECT_H*2+1.
__device__ void issue_conv(SchedShared& S, int c, const Stencil& st, const double* x, int64_t L, double* y,
                           int64_t Lout, int h, double* kc, unsigned char* kbuilt, const double* delta) {
  if (Lout <= 0) return;
  Task t;
  t.c0 = st.c0; t.c1 = st.c1; t.c2 = st.c2; t.span = st.span; t.h = h;
  if (h <= DIRECT_H && L <= 4096) {
    const int M = h * st.span + 1;
    double* w = kc + (int64_t)h * h;
    if (!kbuilt[h]) {
      Task b = t;
      b.kind = TK_KBUILD;
      b.x = delta + (2 * DIRECT_H + 1) - (M - 1);
      b.L = 2 * (int64_t)M - 1;
      b.y = w;
      b.Lout = M;
      issue(S, c, b, U(b.x), U(b.x + b.L), U(w), U(w + M));
      if (lane_id() == 0) kbuilt[h] = 1;
      __syncwarp();
    }
    t.kind = TK_DIRECT;
    t.w = w;
  } else {
    t.kind = TK_FFT;
    t.w = nullptr;
  }
  t.x = x; t.L = L; t.y = y; t.Lout = Lout;
  issue(S, c, t, U(x), U(x + L), U(y), U(y + Lout));
}

// Execute a generic task on the worker group; returns executed flops (or < 0 on error).
__device__ double exec_generic(const Task& t, double2* sbuf, const Grp& g) {
  const Stencil st{t.c0, t.c1, t.c2, t.span};
  if (t.kind == TK_FFT || t.kind == TK_KBUILD)
    return conv_fft(t.x, t.L, t.y, t.Lout, t.h, st, sbuf, SCHED_LOGN_MAX, g);
  // TK_DIRECT
  return conv_direct(t.x, t.L, t.y, t.Lout, t.w, t.h * t.span + 1, (double*)sbuf, g);
}

}  // namespace fl
