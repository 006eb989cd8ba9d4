// fl_abi.cu -- the C ABI (include/fftlattice_b200.h): host-side parameter
// derivation (host_params.h), device buffer management, kernel dispatch and
// result merging.  The reference's pricing entry points (binomial.py:80/161,
// american.py:428, bsm.py:273/585) map onto fl_price_batch per option kind.
#include <algorithm>
#include <iterator>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fftlattice_b200.h"
#include "fl_kernels.h"
#include "host_params.h"

namespace {

// mixed batches: chain slots of a B200 (148 SMs x 2 chains) and the fill ratio
// (a kind's summed cost / (slots x its largest cost)) from which the two kinds run
// as two kernels instead of one mixed kernel
constexpr double kChainSlots = 2.0 * 148.0;
constexpr double kSplitFill = 1.1;

thread_local std::string g_last_error;

int fail(const std::string& msg) {
  g_last_error = msg;
  return 1;
}

#define FL_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t sz = want < 256 ? 256 : want;
    cudaError_t e = cudaMalloc(&p, sz);
    if (e == cudaSuccess) bytes = sz;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct HostPinned {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
};

// Grow-only pinned host array (params are staged here, then copied H2D).
template <class T>
struct PinnedVec {
  T* p = nullptr;
  size_t cap = 0, n = 0;
  cudaError_t resize(size_t want) {
    if (want > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      const size_t c = want < 64 ? 64 : want;
      cudaError_t e = cudaMallocHost((void**)&p, c * sizeof(T));
      if (e != cudaSuccess) return e;
      cap = c;
    }
    n = want;
    return cudaSuccess;
  }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
  T* data() { return p; }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = n = 0;
  }
};

std::mutex g_init_mu;
bool g_tw_ready[64] = {false};

cudaError_t ensure_device_init(int dev, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!g_tw_ready[dev]) {
    fl::init_twiddles(stream);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    g_tw_ready[dev] = true;
  }
  return cudaSuccess;
}

inline double cost_put(int64_t n) {
  const double l = std::log2((double)std::max<int64_t>(n, 2));
  return 24.8 * (double)n * l * l;
}
inline double cost_call(int64_t n) {
  const double l = std::log2((double)std::max<int64_t>(n, 2));
  return 10.0 * (double)n * l * l;
}

void sort_by_cost(std::vector<int32_t>& ord, const std::vector<double>& cost) {
  std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
}

}  // namespace

struct fl_batch {
  int dev = 0;
  int64_t n = 0;
  int method = FL_METHOD_FAST;
  int32_t cap = 0;
  int launches = 0;
  // host-side
  std::vector<int8_t> kind;
  std::vector<int32_t> hstatus;  // host-decided status (errors)
  std::vector<int32_t> mode;
  PinnedVec<fl::PutParams> put;
  PinnedVec<fl::CallParams> call;
  PinnedVec<fl::EuroParams> euro;
  PinnedVec<int32_t> orders;
  DevBuf d_stats;
  size_t h2d_bytes = 0, d2h_bytes = 0;
  // flop accounting: production runs skip the chains' per-node counting; the
  // counts come from one untimed accounting run of the same batch (same kernel,
  // same inputs, deterministic), made on the first stats / ref-flops query
  bool acct_mode = false, acct_valid = false;
  double acct_exec = 0.0, acct_ref = 0.0;
  bool need_put = false, need_call = false, need_euro = false;
  std::vector<double> cost;
  std::vector<int32_t> o_put_fast, o_put_base, o_call_fast, o_call_base, o_euro_fast, o_euro_base;
  std::vector<int32_t> o_mixed;  // puts and calls together (both kinds present): e >= 0 put, e < 0 call -e-1
  size_t off_mixed = 0;
  int grid_mixed = 0;
  int64_t ws_mixed_stride = 0;
  int64_t snap_cap = 0;  // fast-put record_rows capture (fl_put_fast_rows only)
  DevBuf d_snap, d_snaplen;
  // device-side
  DevBuf d_put, d_call, d_euro, d_orders, d_price, d_status, d_bt, d_bc, d_bcount, d_counter;
  DevBuf d_ws_put, d_ws_call, d_ws_base;
  int64_t ws_put_stride = 0, ws_call_stride = 0, ws_base_stride = 0;
  int64_t n_put_base = 0, n_call_base = 0, n_euro_base = 0;  // widest baseline row per list
  int grid_put = 0, grid_call = 0;
  size_t off_put_fast = 0, off_put_base = 0, off_call_fast = 0, off_call_base = 0, off_euro_fast = 0,
         off_euro_base = 0;

  void release() {
    for (DevBuf* b : {&d_put, &d_call, &d_euro, &d_orders, &d_price, &d_status, &d_bt, &d_bc, &d_bcount, &d_counter,
                      &d_ws_put, &d_ws_call, &d_ws_base, &d_stats, &d_snap, &d_snaplen})
      b->release();
    put.release();
    call.release();
    euro.release();
    orders.release();
  }
};

namespace {

// Host-side derivation + dispatch lists.  Pure host work (libm), no CUDA.
int plan_host(fl_batch* b, int64_t n, const int8_t* kind, const double* S, const double* K, const double* R,
               const double* Y, const double* V, const double* E, const int64_t* T, double lam, int64_t call_cutoff,
               int64_t put_cutoff, int method, int32_t cap, const double* bparams = nullptr) {
  b->n = n;
  b->method = method;
  b->cap = cap;
  b->kind.assign(kind, kind + n);
  b->hstatus.assign(n, 0);
  b->mode.assign(n, fl::MODE_ERROR);
  FL_CUDA(b->put.resize(n));
  FL_CUDA(b->call.resize(n));
  FL_CUDA(b->euro.resize(n));
  b->cost.assign(n, 0.0);
  for (auto* v : {&b->o_put_fast, &b->o_put_base, &b->o_call_fast, &b->o_call_base, &b->o_euro_fast, &b->o_euro_base})
    v->clear();
  // FL_FULL_STRIPS=1 (tests only): disable the sliding-frame put leaf strips, so
  // the full-frame fallback is exercised on well-conditioned options too
  const char* fs = std::getenv("FL_FULL_STRIPS");
  const bool full_strips = fs && fs[0] == '1';
  for (int64_t i = 0; i < n; ++i) {
    const fl::SpecIn s{S[i], K[i], R[i], Y[i], V[i], E[i], T[i]};
    const int32_t o = (int32_t)i;
    int32_t st = 0;
    // caller-supplied lattice constants (n x 4: weight_down, weight_up,
    // log_up, step_years; a NaN weight_down row derives them from the spec)
    fl::Binom ovr_b{};
    const fl::Binom* ovr = nullptr;
    if (bparams && !std::isnan(bparams[4 * i])) {
      ovr_b.wd = bparams[4 * i]; ovr_b.wu = bparams[4 * i + 1]; ovr_b.lu = bparams[4 * i + 2];
      ovr_b.dt = bparams[4 * i + 3];
      ovr = &ovr_b;
    }
    switch (kind[i]) {
      case FL_KIND_EURO: {
        st = fl::prep_euro(s, b->euro[i], ovr);
        if (!st) {
          b->mode[i] = (method == FL_METHOD_FAST) ? fl::MODE_FAST : fl::MODE_BASELINE;
          (method == FL_METHOD_FAST ? b->o_euro_fast : b->o_euro_base).push_back(o);
        }
        break;
      }
      case FL_KIND_CALL: {
        if (method == FL_METHOD_FAST) {
          st = fl::prep_call(s, call_cutoff, b->call[i], b->euro[i], ovr);
          if (!st) {
            b->mode[i] = b->call[i].mode;
            if (b->mode[i] == fl::MODE_FAST) b->o_call_fast.push_back(o);
            else if (b->mode[i] == fl::MODE_BASELINE) b->o_call_base.push_back(o);
            else if (b->mode[i] == fl::MODE_EURO) b->o_euro_fast.push_back(o);
          }
        } else {
          fl::Binom bn;
          st = fl::binomial_or_override(s, ovr, bn);
          if (!st) {
            fl::CallParams& c = b->call[i];
            c.S = s.S; c.K = s.K; c.wd = bn.wd; c.wu = bn.wu; c.lu = bn.lu; c.n = s.T;
            c.top_b = -1; c.junc_j = -1; c.cutoff = (int32_t)call_cutoff; c.mode = fl::MODE_BASELINE; c.price = 0;
            b->mode[i] = fl::MODE_BASELINE;
            b->o_call_base.push_back(o);
          }
        }
        b->cost[i] = cost_call(s.T);
        break;
      }
      case FL_KIND_PUT: {
        st = fl::prep_put(s, lam, put_cutoff, b->put[i]);
        if (full_strips) b->put[i].slide = 0;  // test knob: every leaf on the full 4h+2 frame
        if (method == FL_METHOD_BASELINE) {
          // baseline_put_fd: discretization errors only, no cutoff / intrinsic dispatch
          if (!st || (st == (FL_E_VALIDATION | FL_F_CUTOFF))) {
            st = 0;
            b->put[i].mode = fl::MODE_BASELINE;
          }
        }
        if (!st) {
          b->mode[i] = b->put[i].mode;
          if (b->mode[i] == fl::MODE_FAST) b->o_put_fast.push_back(o);
          else if (b->mode[i] == fl::MODE_BASELINE) b->o_put_base.push_back(o);
        }
        b->cost[i] = cost_put(s.T);
        break;
      }
      default:
        st = FL_E_VALIDATION;
    }
    b->hstatus[i] = st;
    if (st) b->mode[i] = fl::MODE_ERROR;
  }
  sort_by_cost(b->o_put_fast, b->cost);
  sort_by_cost(b->o_call_fast, b->cost);
  b->o_mixed.clear();
  // Both kinds present: one kernel over one cost-ordered queue (the kinds share
  // every SM) -- unless each kind alone keeps every chain slot of the GPU busy for
  // longer than its longest option (cost model): then each kind runs on its own,
  // smaller kernel (its own warp layout, register allocation and instruction
  // footprint) back to back, the tail of the first being a few short options.
  // Measured on C5 mixes: break-even at a fill ratio of 0.9 (3072 options), 12 %
  // faster at 1.18 (4096), 8.6 % at 18.5 (65 536); far slower below 0.6
  // (profiles/r02_experiments.md).  FL_SPLIT_KINDS=0 / 1 forces either dispatch.
  auto fill = [&](const std::vector<int32_t>& ord) {
    double sum = 0.0, mx = 0.0;
    for (int32_t e : ord) { sum += b->cost[e]; mx = std::max(mx, b->cost[e]); }
    return mx > 0.0 ? sum / (kChainSlots * mx) : 0.0;
  };
  const char* split_env = std::getenv("FL_SPLIT_KINDS");
  const bool split = split_env ? split_env[0] == '1'
                               : (fill(b->o_put_fast) >= kSplitFill && fill(b->o_call_fast) >= kSplitFill);
  if (!b->o_put_fast.empty() && !b->o_call_fast.empty() && !split) {
    std::merge(b->o_put_fast.begin(), b->o_put_fast.end(), b->o_call_fast.begin(), b->o_call_fast.end(),
               std::back_inserter(b->o_mixed), [&](int32_t a, int32_t c) { return b->cost[a] > b->cost[c]; });
    for (int32_t& e : b->o_mixed)
      if (b->kind[e] == FL_KIND_CALL) e = -e - 1;
  }
  b->need_put = !b->o_put_fast.empty() || !b->o_put_base.empty();
  b->need_call = !b->o_call_fast.empty() || !b->o_call_base.empty();
  b->need_euro = !b->o_euro_fast.empty() || !b->o_euro_base.empty();
  return 0;
}

// CTAs for a fast batch of n items: one per item while they fit on the SMs
// (each runs alone, sched_body's solo mode), else NCHAIN items per CTA.
static int grid_for(int n, int nc, int nsm) { return n <= nsm ? n : std::min((n + nc - 1) / nc, nsm); }

int upload(fl_batch* b, cudaStream_t stream) {
  const int64_t n = b->n;
  FL_CUDA(cudaGetDevice(&b->dev));
  FL_CUDA(ensure_device_init(b->dev, stream));
  int nsm = 0;
  FL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, b->dev));
  if (b->need_put) FL_CUDA(b->d_put.ensure(sizeof(fl::PutParams) * n));
  if (b->need_call) FL_CUDA(b->d_call.ensure(sizeof(fl::CallParams) * n));
  if (b->need_euro) FL_CUDA(b->d_euro.ensure(sizeof(fl::EuroParams) * n));
  FL_CUDA(b->d_stats.ensure((64 + 3 * n) * sizeof(unsigned long long)));  // counters | timeline
  // orders packed into one buffer
  size_t off = 0;
  auto place = [&](const std::vector<int32_t>& v, size_t& o) { o = off; off += v.size(); };
  place(b->o_put_fast, b->off_put_fast);
  place(b->o_put_base, b->off_put_base);
  place(b->o_call_fast, b->off_call_fast);
  place(b->o_call_base, b->off_call_base);
  place(b->o_euro_fast, b->off_euro_fast);
  place(b->o_euro_base, b->off_euro_base);
  place(b->o_mixed, b->off_mixed);
  FL_CUDA(b->d_orders.ensure(sizeof(int32_t) * (off + 1)));
  FL_CUDA(b->d_price.ensure(sizeof(double) * n));
  FL_CUDA(b->d_status.ensure(sizeof(int32_t) * n));
  FL_CUDA(b->d_bcount.ensure(sizeof(int32_t) * n));
  if (b->cap > 0) {
    FL_CUDA(b->d_bt.ensure(sizeof(int64_t) * n * b->cap));
    FL_CUDA(b->d_bc.ensure(sizeof(int64_t) * n * b->cap));
  }
  FL_CUDA(b->d_counter.ensure(64));
  // workspaces
  int64_t nmax_put = 0, ksmax = 0, nmax_call = 0, nmax_base = 0;
  for (int32_t o : b->o_put_fast) {
    nmax_put = std::max(nmax_put, b->put[o].n);
    ksmax = std::max<int64_t>(ksmax, std::max<int64_t>(b->put[o].ks, 0));
  }
  for (int32_t o : b->o_call_fast) nmax_call = std::max(nmax_call, b->call[o].n);
  b->n_put_base = b->n_call_base = b->n_euro_base = 0;
  for (int32_t o : b->o_put_base) b->n_put_base = std::max(b->n_put_base, b->put[o].n);
  for (int32_t o : b->o_call_base) b->n_call_base = std::max(b->n_call_base, b->call[o].n);
  for (int32_t o : b->o_euro_base) b->n_euro_base = std::max(b->n_euro_base, b->euro[o].n);
  // the global-memory fallback march needs a workspace row set per CTA; the
  // register-resident sweeps (fl_sweep.cu) need none
  const int64_t cells_max = fl::sweep_disabled() ? 0 : fl::sweep_max_cells();
  if (2 * b->n_put_base + 1 > cells_max) nmax_base = std::max(nmax_base, b->n_put_base * 2 + 2);
  if (b->n_call_base + 1 > cells_max) nmax_base = std::max(nmax_base, b->n_call_base + 2);
  if (b->n_euro_base + 1 > cells_max) nmax_base = std::max(nmax_base, b->n_euro_base + 2);
  if (!b->o_put_fast.empty()) {
    b->ws_put_stride = fl::put_ws_doubles(nmax_put, ksmax);
    const int nc = fl::put_chains_per_cta();
    b->grid_put = grid_for((int)b->o_put_fast.size(), nc, nsm);
    FL_CUDA(b->d_ws_put.ensure(sizeof(double) * b->ws_put_stride * b->grid_put * nc));
  }
  if (!b->o_call_fast.empty()) {
    b->ws_call_stride = fl::call_ws_doubles(nmax_call);
    const int nc = fl::call_chains_per_cta();
    b->grid_call = grid_for((int)b->o_call_fast.size(), nc, nsm);
    FL_CUDA(b->d_ws_call.ensure(sizeof(double) * b->ws_call_stride * b->grid_call * nc));
  }
  if (!b->o_mixed.empty()) {
    b->ws_mixed_stride = std::max(b->ws_put_stride, b->ws_call_stride);
    const int nc = fl::put_chains_per_cta();
    b->grid_mixed = grid_for((int)b->o_mixed.size(), nc, nsm);
    FL_CUDA(b->d_ws_put.ensure(sizeof(double) * b->ws_mixed_stride * b->grid_mixed * nc));
  }
  const int64_t nbase = (int64_t)std::max({b->o_put_base.size(), b->o_call_base.size(), b->o_euro_base.size()});
  if (nbase > 0 && nmax_base > 0) {
    b->ws_base_stride = 3 * nmax_base + 16;
    FL_CUDA(b->d_ws_base.ensure(sizeof(double) * b->ws_base_stride * nbase));
  }
  // H2D (pinned staging)
  FL_CUDA(b->orders.resize(off + 1));
  int32_t* orders = b->orders.data();
  orders[off] = 0;
  auto copy_in = [&](const std::vector<int32_t>& v, size_t o) { std::copy(v.begin(), v.end(), orders + o); };
  copy_in(b->o_put_fast, b->off_put_fast);
  copy_in(b->o_put_base, b->off_put_base);
  copy_in(b->o_call_fast, b->off_call_fast);
  copy_in(b->o_call_base, b->off_call_base);
  copy_in(b->o_euro_fast, b->off_euro_fast);
  copy_in(b->o_euro_base, b->off_euro_base);
  copy_in(b->o_mixed, b->off_mixed);
  b->h2d_bytes = sizeof(int32_t) * (off + 1);
  if (b->need_put) {
    FL_CUDA(cudaMemcpyAsync(b->d_put.p, b->put.data(), sizeof(fl::PutParams) * n, cudaMemcpyHostToDevice, stream));
    b->h2d_bytes += sizeof(fl::PutParams) * n;
  }
  if (b->need_call) {
    FL_CUDA(cudaMemcpyAsync(b->d_call.p, b->call.data(), sizeof(fl::CallParams) * n, cudaMemcpyHostToDevice, stream));
    b->h2d_bytes += sizeof(fl::CallParams) * n;
  }
  if (b->need_euro) {
    FL_CUDA(cudaMemcpyAsync(b->d_euro.p, b->euro.data(), sizeof(fl::EuroParams) * n, cudaMemcpyHostToDevice, stream));
    b->h2d_bytes += sizeof(fl::EuroParams) * n;
  }
  FL_CUDA(cudaMemcpyAsync(b->d_orders.p, orders, sizeof(int32_t) * (off + 1), cudaMemcpyHostToDevice, stream));
  return 0;
}

fl::BatchOut make_out(fl_batch* b) {
  fl::BatchOut o;
  o.price = b->d_price.as<double>();
  o.status = b->d_status.as<int32_t>();
  o.bt = b->cap > 0 ? b->d_bt.as<int64_t>() : nullptr;
  o.bc = b->cap > 0 ? b->d_bc.as<int64_t>() : nullptr;
  o.bcount = b->d_bcount.as<int32_t>();
  o.cap = b->cap;
  o.flops = b->d_stats.as<unsigned long long>();
  o.prof = std::getenv("FL_PROFILE") ? b->d_stats.as<unsigned long long>() + 8 : nullptr;
  o.acct = (b->acct_mode || std::getenv("FL_ACCT")) ? 1 : 0;
  if (b->snap_cap > 0) {
    o.snap = b->d_snap.as<double>();
    o.snap_cap = b->snap_cap;
    o.snap_len = b->d_snaplen.as<int64_t>();
  }
  return o;
}

int run(fl_batch* b, cudaStream_t stream) {
  const fl::BatchOut out = make_out(b);
  const int32_t* ord = b->d_orders.as<int32_t>();
  int32_t* counter = b->d_counter.as<int32_t>();
  b->launches = 0;
  FL_CUDA(cudaMemsetAsync(b->d_stats.p, 0, 64 * sizeof(unsigned long long), stream));
  if (!b->o_mixed.empty()) {
    FL_CUDA(fl::launch_american_fast(b->d_put.as<fl::PutParams>(), b->d_call.as<fl::CallParams>(),
                                     ord + b->off_mixed, (int)b->o_mixed.size(), counter, b->d_ws_put.as<double>(),
                                     b->ws_mixed_stride, b->grid_mixed, out, stream));
    ++b->launches;
  } else if (!b->o_put_fast.empty()) {
    FL_CUDA(fl::launch_put_fast(b->d_put.as<fl::PutParams>(), ord + b->off_put_fast, (int)b->o_put_fast.size(),
                                counter, b->d_ws_put.as<double>(), b->ws_put_stride, b->grid_put, out, stream));
    ++b->launches;
  }
  if (b->o_mixed.empty() && !b->o_call_fast.empty()) {
    FL_CUDA(fl::launch_call_fast(b->d_call.as<fl::CallParams>(), ord + b->off_call_fast,
                                 (int)b->o_call_fast.size(), counter + 8, b->d_ws_call.as<double>(),
                                 b->ws_call_stride, b->grid_call, out, stream));
    ++b->launches;
  }
  if (!b->o_euro_fast.empty()) {
    FL_CUDA(fl::launch_euro_fast(b->d_euro.as<fl::EuroParams>(), ord + b->off_euro_fast, (int)b->o_euro_fast.size(),
                                 (int)b->o_euro_fast.size(), out, stream));
    ++b->launches;
  }
  if (!b->o_put_base.empty()) {
    const int nb = (int)b->o_put_base.size();
    FL_CUDA(fl::launch_put_baseline(b->d_put.as<fl::PutParams>(), ord + b->off_put_base, nb, b->n_put_base, nb,
                                    b->d_ws_base.as<double>(), b->ws_base_stride, out, stream));
    ++b->launches;
  }
  if (!b->o_call_base.empty()) {
    const int nb = (int)b->o_call_base.size();
    FL_CUDA(fl::launch_call_baseline(b->d_call.as<fl::CallParams>(), ord + b->off_call_base, nb, b->n_call_base, nb,
                                     b->d_ws_base.as<double>(), b->ws_base_stride, out, stream));
    ++b->launches;
  }
  if (!b->o_euro_base.empty()) {
    const int nb = (int)b->o_euro_base.size();
    FL_CUDA(fl::launch_euro_baseline(b->d_euro.as<fl::EuroParams>(), ord + b->off_euro_base, nb, b->n_euro_base, nb,
                                     b->d_ws_base.as<double>(), b->ws_base_stride, out, stream));
    ++b->launches;
  }
  return 0;
}

inline int64_t fg_rec(int64_t i, int64_t j) { return j >= i ? INT64_MIN : j + 1; }

int fetch(fl_batch* b, double* price, int32_t* status, int64_t* bt, int64_t* bc, int32_t* bcount,
          cudaStream_t stream) {
  const int64_t n = b->n;
  const int32_t cap = b->cap;
  FL_CUDA(cudaMemcpyAsync(price, b->d_price.p, sizeof(double) * n, cudaMemcpyDeviceToHost, stream));
  FL_CUDA(cudaMemcpyAsync(status, b->d_status.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, stream));
  std::vector<int32_t> cnt(n, 0);
  FL_CUDA(cudaMemcpyAsync(cnt.data(), b->d_bcount.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, stream));
  const bool want_b = cap > 0 && bt && bc && bcount;
  if (want_b) {
    FL_CUDA(cudaMemcpyAsync(bt, b->d_bt.p, sizeof(int64_t) * n * cap, cudaMemcpyDeviceToHost, stream));
    FL_CUDA(cudaMemcpyAsync(bc, b->d_bc.p, sizeof(int64_t) * n * cap, cudaMemcpyDeviceToHost, stream));
  }
  FL_CUDA(cudaStreamSynchronize(stream));
  b->d2h_bytes = (sizeof(double) + 2 * sizeof(int32_t)) * n + (want_b ? 2 * sizeof(int64_t) * n * cap : 0);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t m = b->mode[i];
    int32_t c = cnt[i];
    auto rec = [&](int32_t k, int64_t t, int64_t col) {
      if (want_b && k < cap) {
        bt[i * cap + k] = t;
        bc[i * cap + k] = col;
      }
    };
    if (m == fl::MODE_ERROR) {
      status[i] = b->hstatus[i];
      price[i] = std::nan("");
      c = 0;
    } else if (b->kind[i] == FL_KIND_PUT && m == fl::MODE_INTRINSIC) {
      status[i] = 0;
      price[i] = b->put[i].price;
      rec(0, 0, std::min<int64_t>(0, b->put[i].ks + b->put[i].n));
      c = 1;
    } else if (b->kind[i] == FL_KIND_CALL && m == fl::MODE_INTRINSIC) {
      const fl::CallParams& p = b->call[i];
      status[i] = 0;
      price[i] = p.price;
      rec(0, p.n - 1, fg_rec(p.n - 1, p.junc_j));  // ascending order: T-1, T
      rec(1, p.n, fg_rec(p.n, p.top_b));
      c = 2;
    } else if (b->kind[i] == FL_KIND_CALL && m == fl::MODE_EURO) {
      const fl::CallParams& p = b->call[i];
      rec(0, p.n, p.top_b == p.n ? INT64_MIN : fg_rec(p.n, p.top_b));
      c = 1;
    } else if (b->kind[i] == FL_KIND_CALL && m == fl::MODE_FAST && want_b && status[i] == 0) {
      // device records run T, T-1, ..., 0: reverse into ascending order
      const int32_t k = std::min(c, cap);
      std::reverse(bt + i * cap, bt + i * cap + k);
      std::reverse(bc + i * cap + 0, bc + i * cap + k);
    }
    if (bcount) bcount[i] = c;
  }
  return 0;
}

}  // namespace

extern "C" {

int fl_version(void) { return 100; }

const char* fl_last_error(void) { return g_last_error.c_str(); }

int fl_batch_prepare(fl_batch** out, int64_t n, const int8_t* kind, const double* S, const double* K,
                     const double* R, const double* Y, const double* V, const double* E, const int64_t* T,
                     double lam, int64_t call_cutoff, int64_t put_cutoff, int method, int32_t bnd_cap,
                     void* stream) {
  if (!out) return fail("fl_batch_prepare: null out");
  if (n < 0) return fail("fl_batch_prepare: negative n");
  fl_batch* b = new fl_batch();
  int rc = plan_host(b, n, kind, S, K, R, Y, V, E, T, lam, call_cutoff, put_cutoff, method, bnd_cap);
  if (!rc) rc = upload(b, (cudaStream_t)stream);
  if (!rc && cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) rc = fail("fl_batch_prepare: sync failed");
  if (rc) {
    b->release();
    delete b;
    return rc;
  }
  *out = b;
  return 0;
}

int fl_batch_run(fl_batch* b, void* stream) {
  if (!b) return fail("fl_batch_run: null batch");
  return run(b, (cudaStream_t)stream);
}

int fl_batch_fetch(fl_batch* b, double* price, int32_t* status, int64_t* bnd_times, int64_t* bnd_cols,
                   int32_t* bnd_count, void* stream) {
  if (!b) return fail("fl_batch_fetch: null batch");
  return fetch(b, price, status, bnd_times, bnd_cols, bnd_count, (cudaStream_t)stream);
}

int fl_batch_launches(const fl_batch* b) { return b ? b->launches : 0; }

// One untimed accounting run of the batch (once per prepared batch).
static int ensure_accounting(fl_batch* b, cudaStream_t stream) {
  if (b->acct_valid) return 0;
  b->acct_mode = true;
  const int rc = run(b, stream);
  b->acct_mode = false;
  if (rc) return rc;
  unsigned long long f[2] = {0, 0};
  FL_CUDA(cudaMemcpyAsync(f, b->d_stats.p, sizeof(f), cudaMemcpyDeviceToHost, stream));
  FL_CUDA(cudaStreamSynchronize(stream));
  b->acct_exec = (double)f[0];
  b->acct_ref = (double)f[1];
  b->acct_valid = true;
  return 0;
}

int fl_batch_stats(fl_batch* b, double* fp64_flops, int64_t* h2d_bytes, int64_t* d2h_bytes, void* stream) {
  if (!b) return fail("fl_batch_stats: null batch");
  if (fp64_flops) {
    if (const int rc = ensure_accounting(b, (cudaStream_t)stream)) return rc;
    *fp64_flops = b->acct_exec;
  }
  if (h2d_bytes) *h2d_bytes = (int64_t)b->h2d_bytes;
  if (d2h_bytes) *d2h_bytes = (int64_t)b->d2h_bytes;
  return 0;
}

int fl_inspect(int64_t n, const int8_t* kind, const double* S, const double* K, const double* R, const double* Y,
               const double* V, const double* E, const int64_t* T, double lam, int64_t call_cutoff,
               int64_t put_cutoff, int32_t* status, int32_t* mode, double* dparams, int64_t* iparams) {
  if (n < 0 || !kind || !S || !K || !R || !Y || !V || !E || !T || !status || !mode || !dparams || !iparams)
    return fail("fl_inspect: null pointer");
  for (int64_t i = 0; i < n; ++i) {
    const fl::SpecIn s{S[i], K[i], R[i], Y[i], V[i], E[i], T[i]};
    double* d = dparams + 4 * i;
    int64_t* q = iparams + 2 * i;
    d[0] = d[1] = d[2] = d[3] = 0.0;
    q[0] = q[1] = 0;
    int32_t st = 0, md = fl::MODE_ERROR;
    if (kind[i] == FL_KIND_EURO) {
      fl::EuroParams e;
      st = fl::prep_euro(s, e);
      if (!st) { md = fl::MODE_FAST; d[0] = e.wd; d[1] = e.wu; d[2] = e.bg; d[3] = e.lu; }
    } else if (kind[i] == FL_KIND_CALL) {
      fl::CallParams c;
      fl::EuroParams e;
      st = fl::prep_call(s, call_cutoff, c, e);
      if (!st) { md = c.mode; d[0] = c.wd; d[1] = c.wu; d[2] = c.lu; d[3] = c.price; q[0] = c.top_b; q[1] = c.junc_j; }
    } else if (kind[i] == FL_KIND_PUT) {
      fl::PutParams p;
      st = fl::prep_put(s, lam, put_cutoff, p);
      if (!st) { md = p.mode; d[0] = p.cd; d[1] = p.cm; d[2] = p.cu; d[3] = p.ds; q[0] = p.ks; q[1] = p.slide; }
    } else {
      st = FL_E_VALIDATION;
    }
    status[i] = st;
    mode[i] = st ? fl::MODE_ERROR : md;
  }
  return 0;
}

int fl_batch_ref_flops(fl_batch* b, double* ref_flops, void* stream) {
  if (!b) return fail("fl_batch_ref_flops: null batch");
  if (const int rc = ensure_accounting(b, (cudaStream_t)stream)) return rc;
  if (ref_flops) *ref_flops = b->acct_ref;
  return 0;
}

// Shared driver of the single-problem trapezoid entry points: device buffers
// for one input row, one output row and one chain arena, freed on return.
struct TrapBufs {
  DevBuf in, out, meta, counter, ws, stats;
  ~TrapBufs() {
    for (DevBuf* b : {&in, &out, &meta, &counter, &ws, &stats}) b->release();
  }
};

int fl_put_trapezoid(double cd, double cm, double cu, double ds, int64_t base_cutoff, int64_t f, const double* seg,
                     int64_t W, int64_t h, double* out_seg, int64_t* kp, int32_t* status, void* stream) {
  if (!seg || !out_seg || !kp || !status) return fail("fl_put_trapezoid: null pointer");
  if (h < 1 || W < 2 * h) return fail("fl_put_trapezoid: need h >= 1 and W >= 2h");
  if (h > (int64_t)1 << 30) return fail("fl_put_trapezoid: h too large");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  FL_CUDA(ensure_device_init(dev, st));
  TrapBufs B;
  const int64_t stride = fl::put_trap_ws_doubles(f, W, h);
  FL_CUDA(B.in.ensure(sizeof(double) * W));
  FL_CUDA(B.out.ensure(sizeof(double) * (W + h)));
  FL_CUDA(B.meta.ensure(2 * sizeof(int64_t)));
  FL_CUDA(B.counter.ensure(64));
  FL_CUDA(B.ws.ensure(sizeof(double) * stride * fl::put_chains_per_cta()));
  FL_CUDA(B.stats.ensure(2 * sizeof(unsigned long long)));
  FL_CUDA(cudaMemcpyAsync(B.in.p, seg, sizeof(double) * W, cudaMemcpyHostToDevice, st));
  fl::PutParams P{};
  P.cd = cd; P.cm = cm; P.cu = cu; P.ds = ds; P.cutoff = (int32_t)std::min<int64_t>(base_cutoff, 1 << 30);
  P.n = h; P.mode = fl::MODE_FAST;
  FL_CUDA(fl::launch_put_trapezoid(P, f, W, h, B.in.as<double>(), B.out.as<double>(), B.meta.as<int64_t>(),
                                   B.counter.as<int32_t>(), B.ws.as<double>(), stride, nullptr, st));
  int64_t meta[2] = {0, 0};
  FL_CUDA(cudaMemcpyAsync(meta, B.meta.p, sizeof(meta), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  *kp = meta[0];
  *status = (int32_t)meta[1];
  if (meta[1] == 0) {
    const int64_t len = (f + W - h) - meta[0];
    if (len < 0 || len > W + h) return fail("fl_put_trapezoid: inconsistent output length");
    FL_CUDA(cudaMemcpy(out_seg, B.out.p, sizeof(double) * len, cudaMemcpyDeviceToHost));
  }
  return 0;
}

int fl_call_trapezoid(double S, double K, double wd, double wu, double lu, int64_t base_cutoff, int64_t i, int64_t j,
                      int64_t first, const double* run, int64_t h, double* out_run, int64_t* jp, int32_t* status,
                      void* stream) {
  if (!run || !out_run || !jp || !status) return fail("fl_call_trapezoid: null pointer");
  const int64_t width = j - first + 1;
  if (h < 1 || width < h || h > i) return fail("fl_call_trapezoid: need 1 <= h <= min(run width, i)");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  FL_CUDA(ensure_device_init(dev, st));
  TrapBufs B;
  const int64_t stride = fl::call_trap_ws_doubles(width, h);
  FL_CUDA(B.in.ensure(sizeof(double) * width));
  FL_CUDA(B.out.ensure(sizeof(double) * width));
  FL_CUDA(B.meta.ensure(2 * sizeof(int64_t)));
  FL_CUDA(B.counter.ensure(64));
  FL_CUDA(B.ws.ensure(sizeof(double) * stride * fl::call_chains_per_cta()));
  FL_CUDA(cudaMemcpyAsync(B.in.p, run, sizeof(double) * width, cudaMemcpyHostToDevice, st));
  fl::CallParams P{};
  P.S = S; P.K = K; P.wd = wd; P.wu = wu; P.lu = lu; P.n = i;
  P.cutoff = (int32_t)std::min<int64_t>(base_cutoff, 1 << 30);
  P.mode = fl::MODE_FAST;
  FL_CUDA(fl::launch_call_trapezoid(P, i, j, first, h, B.in.as<double>(), B.out.as<double>(), B.meta.as<int64_t>(),
                                    B.counter.as<int32_t>(), B.ws.as<double>(), stride, nullptr, st));
  int64_t meta[2] = {0, 0};
  FL_CUDA(cudaMemcpyAsync(meta, B.meta.p, sizeof(meta), cudaMemcpyDeviceToHost, st));
  FL_CUDA(cudaStreamSynchronize(st));
  *jp = meta[0];
  *status = (int32_t)meta[1];
  if (meta[1] == 0) {
    const int64_t len = meta[0] - first + 1;
    if (len < 0 || len > width) return fail("fl_call_trapezoid: inconsistent output length");
    if (len > 0) FL_CUDA(cudaMemcpy(out_run, B.out.p, sizeof(double) * len, cudaMemcpyDeviceToHost));
  }
  return 0;
}

int fl_call_grid(double S, double K, double wd, double wu, double lu, int64_t n, double* rows, uint8_t* masks,
                 int64_t* cols, double* price, void* stream) {
  if (!rows || !masks || !cols || !price) return fail("fl_call_grid: null pointer");
  if (n < 1 || n > (1 << 15)) return fail("fl_call_grid: steps must be in [1, 32768] for a retained grid");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t cells = (n + 1) * (n + 2) / 2;
  DevBuf d_rows, d_masks, d_cols, d_price, d_ws;
  FL_CUDA(d_rows.ensure(sizeof(double) * cells));
  FL_CUDA(d_masks.ensure(cells));
  FL_CUDA(d_cols.ensure(sizeof(int64_t) * (n + 1)));
  FL_CUDA(d_price.ensure(sizeof(double)));
  FL_CUDA(d_ws.ensure(sizeof(double) * 2 * (n + 2)));
  fl::CallParams P{};
  P.S = S; P.K = K; P.wd = wd; P.wu = wu; P.lu = lu; P.n = n; P.mode = fl::MODE_BASELINE;
  cudaError_t e = fl::launch_call_grid(P, d_rows.as<double>(), d_masks.as<uint8_t>(), d_cols.as<int64_t>(),
                                       d_price.as<double>(), d_ws.as<double>(), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(rows, d_rows.p, sizeof(double) * cells, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(masks, d_masks.p, cells, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(cols, d_cols.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(price, d_price.p, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (DevBuf* b : {&d_rows, &d_masks, &d_cols, &d_price, &d_ws}) b->release();
  if (e != cudaSuccess) return fail(std::string("fl_call_grid: ") + cudaGetErrorString(e));
  return 0;
}

int fl_put_march_rows(double cd, double cm, double cu, double ds, double K, int64_t ks, int64_t n,
                      const int64_t* times, int ntimes, double* snap, int64_t snap_cap, int64_t* last_green,
                      double* price, void* stream) {
  if (!last_green || !price || (ntimes > 0 && (!times || !snap))) return fail("fl_put_march_rows: null pointer");
  if (n < 1) return fail("fl_put_march_rows: steps must be >= 1");
  int64_t need = 0;
  for (int i = 0; i < ntimes; ++i) {
    if (times[i] < 1 || times[i] > n || (i > 0 && times[i] <= times[i - 1]))
      return fail("fl_put_march_rows: times must be increasing in [1, steps]");
    need += 2 * n + 1 - 2 * times[i];
  }
  if (need > snap_cap) return fail("fl_put_march_rows: snapshot buffer too small");
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf d_times, d_snap, d_lg, d_price, d_ws;
  FL_CUDA(d_times.ensure(sizeof(int64_t) * (ntimes + 1)));
  FL_CUDA(d_snap.ensure(sizeof(double) * (need + 1)));
  FL_CUDA(d_lg.ensure(sizeof(int64_t) * (n + 1)));
  FL_CUDA(d_price.ensure(sizeof(double)));
  FL_CUDA(d_ws.ensure(sizeof(double) * 3 * (2 * n + 1)));
  if (ntimes > 0) FL_CUDA(cudaMemcpyAsync(d_times.p, times, sizeof(int64_t) * ntimes, cudaMemcpyHostToDevice, st));
  fl::PutParams P{};
  P.K = K; P.cd = cd; P.cm = cm; P.cu = cu; P.ds = ds; P.ks = ks; P.n = n; P.mode = fl::MODE_BASELINE;
  cudaError_t e = fl::launch_put_march_rows(P, d_times.as<int64_t>(), ntimes, d_snap.as<double>(),
                                            d_lg.as<int64_t>(), d_price.as<double>(), d_ws.as<double>(), st);
  if (e == cudaSuccess && need > 0)
    e = cudaMemcpyAsync(snap, d_snap.p, sizeof(double) * need, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(last_green, d_lg.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(price, d_price.p, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (DevBuf* b : {&d_times, &d_snap, &d_lg, &d_price, &d_ws}) b->release();
  if (e != cudaSuccess) return fail(std::string("fl_put_march_rows: ") + cudaGetErrorString(e));
  return 0;
}

int fl_put_fast_rows(double S, double K, double R, double V, double E, int64_t T, double lam, int64_t base_cutoff,
                     double* snap, int64_t snap_cap, int64_t* snap_len, double* price, int32_t* status,
                     int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap, void* stream) {
  if (!snap || !snap_len || !price || !status) return fail("fl_put_fast_rows: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  fl_batch b;
  const int8_t kind = FL_KIND_PUT;
  const double Y = 0.0;
  int rc = plan_host(&b, 1, &kind, &S, &K, &R, &Y, &V, &E, &T, lam, 256, base_cutoff, FL_METHOD_FAST, bnd_cap);
  if (rc) { b.release(); return rc; }
  b.snap_cap = snap_cap;
  cudaError_t e = b.d_snap.ensure(sizeof(double) * (snap_cap + 1));
  if (e == cudaSuccess) e = b.d_snaplen.ensure(sizeof(int64_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(b.d_snaplen.p, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) { b.release(); return fail(std::string("fl_put_fast_rows: ") + cudaGetErrorString(e)); }
  rc = upload(&b, st);
  if (!rc) rc = run(&b, st);
  if (!rc) rc = fetch(&b, price, status, bnd_times, bnd_cols, bnd_count, st);
  if (!rc) {
    e = cudaMemcpy(snap_len, b.d_snaplen.p, sizeof(int64_t), cudaMemcpyDeviceToHost);
    const int64_t got = std::min<int64_t>(*snap_len, snap_cap);
    if (e == cudaSuccess && got > 0) e = cudaMemcpy(snap, b.d_snap.p, sizeof(double) * got, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = fail(std::string("fl_put_fast_rows: ") + cudaGetErrorString(e));
  }
  b.release();
  return rc;
}

int fl_euro_approx(int64_t n, const double* S, const double* K, const double* R, const double* Y, const double* V,
                   const double* E, const int64_t* T, int method, double* price, int32_t* status, void* stream) {
  if (n < 0 || !S || !K || !R || !Y || !V || !E || !T || !price || !status) return fail("fl_euro_approx: null pointer");
  if (method != FL_METHOD_GAUSS && method != FL_METHOD_CLOSED) return fail("fl_euro_approx: unknown method");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  FL_CUDA(ensure_device_init(dev, st));
  std::vector<fl::EuroApprox> ok;
  std::vector<int64_t> idx;
  for (int64_t i = 0; i < n; ++i) {
    fl::EuroApprox a{};
    const fl::SpecIn s{S[i], K[i], R[i], Y[i], V[i], E[i], T[i]};
    status[i] = fl::prep_euro_approx(s, method, a);
    price[i] = 0.0;
    if (!status[i]) { ok.push_back(a); idx.push_back(i); }
  }
  if (ok.empty()) return 0;
  const int m = (int)ok.size();
  DevBuf d_opts, d_price;
  FL_CUDA(d_opts.ensure(sizeof(fl::EuroApprox) * m));
  FL_CUDA(d_price.ensure(sizeof(double) * m));
  std::vector<double> out(m);
  cudaError_t e = cudaMemcpyAsync(d_opts.p, ok.data(), sizeof(fl::EuroApprox) * m, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = fl::launch_euro_approx(d_opts.as<fl::EuroApprox>(), m, method, d_price.as<double>(), st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out.data(), d_price.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  d_opts.release();
  d_price.release();
  if (e != cudaSuccess) return fail(std::string("fl_euro_approx: ") + cudaGetErrorString(e));
  for (int k = 0; k < m; ++k) price[idx[k]] = out[k];
  return 0;
}

int fl_fft(const double* in, int64_t n, int inverse, double* out, void* stream) {
  if (!in || !out) return fail("fl_fft: null pointer");
  if (n < 1 || (n & (n - 1)) != 0) return fail("fl_fft: length must be a power of two");
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf a, b;
  FL_CUDA(a.ensure(sizeof(double2) * n));
  FL_CUDA(b.ensure(sizeof(double2) * n));
  FL_CUDA(cudaMemcpyAsync(a.p, in, sizeof(double2) * n, cudaMemcpyHostToDevice, st));
  double2* r = nullptr;
  cudaError_t e = fl::fft_pow2(a.as<double2>(), b.as<double2>(), n, inverse ? 1 : -1, &r, st);
  if (e == cudaSuccess && inverse) e = fl::launch_cscale(r, n, 1.0 / (double)n, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, r, sizeof(double2) * n, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  a.release();
  b.release();
  if (e != cudaSuccess) return fail(std::string("fl_fft: ") + cudaGetErrorString(e));
  return 0;
}

int fl_convolve(const double* x, int64_t nx, const double* y, int64_t ny, double* out, void* stream) {
  if (!x || !y || !out) return fail("fl_convolve: null pointer");
  if (nx < 1 || ny < 1) return fail("fl_convolve: empty input");
  const int64_t out_len = nx + ny - 1;
  int64_t n = 1;
  while (n < out_len) n <<= 1;
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf a, b, t;
  FL_CUDA(a.ensure(sizeof(double2) * n));
  FL_CUDA(b.ensure(sizeof(double2) * n));
  FL_CUDA(t.ensure(sizeof(double2) * n));
  FL_CUDA(cudaMemsetAsync(a.p, 0, sizeof(double2) * n, st));
  FL_CUDA(cudaMemsetAsync(b.p, 0, sizeof(double2) * n, st));
  FL_CUDA(cudaMemcpyAsync(a.p, x, sizeof(double2) * nx, cudaMemcpyHostToDevice, st));
  FL_CUDA(cudaMemcpyAsync(b.p, y, sizeof(double2) * ny, cudaMemcpyHostToDevice, st));
  double2 *fa = nullptr, *fb = nullptr, *r = nullptr;
  cudaError_t e = fl::fft_pow2(a.as<double2>(), t.as<double2>(), n, -1, &fa, st);
  // fa is a or t; transform b using the other scratch
  double2* scratch = (fa == a.as<double2>()) ? t.as<double2>() : a.as<double2>();
  if (e == cudaSuccess) e = fl::fft_pow2(b.as<double2>(), scratch, n, -1, &fb, st);
  if (e == cudaSuccess) e = fl::launch_cmul(fa, fb, n, 1.0, st);
  double2* other = (fa == a.as<double2>()) ? ((fb == t.as<double2>()) ? b.as<double2>() : t.as<double2>())
                                           : ((fb == a.as<double2>()) ? b.as<double2>() : a.as<double2>());
  if (e == cudaSuccess) e = fl::fft_pow2(fa, other, n, 1, &r, st);
  if (e == cudaSuccess) e = fl::launch_cscale(r, n, 1.0 / (double)n, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, r, sizeof(double2) * out_len, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  a.release();
  b.release();
  t.release();
  if (e != cudaSuccess) return fail(std::string("fl_convolve: ") + cudaGetErrorString(e));
  return 0;
}

int fl_kernel_power(const double* w, int64_t L, int64_t h, double* out, void* stream) {
  // generic kernel_power (fft.py:203-260): the spectrum of the zero-padded
  // kernel raised to the h-th power, inverted (any taps, any finite weights);
  // a one-tap kernel is its weight to the h-th power.  Writes h (L-1) + 1
  // weights.
  if (!w || !out) return fail("fl_kernel_power: null pointer");
  if (L < 1 || h < 1) return fail("fl_kernel_power: need L >= 1 and h >= 1");
  const int64_t out_len = h * (L - 1) + 1;
  int64_t n = 1;
  while (n < out_len) n <<= 1;
  if (n > ((int64_t)1 << 27)) return fail("fl_kernel_power: composed kernel too long");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  DevBuf a, t;
  FL_CUDA(a.ensure(sizeof(double2) * n));
  FL_CUDA(t.ensure(sizeof(double2) * n));
  std::vector<double2> hw(L);
  for (int64_t i = 0; i < L; ++i) hw[i] = make_double2(w[i], 0.0);
  cudaError_t e = cudaMemsetAsync(a.p, 0, sizeof(double2) * n, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(a.p, hw.data(), sizeof(double2) * L, cudaMemcpyHostToDevice, st);
  double2 *f = nullptr, *r = nullptr;
  if (n == 1) {
    if (e == cudaSuccess) e = fl::launch_cpow(a.as<double2>(), 1, h, 1.0, st);
    r = a.as<double2>();
  } else {
    if (e == cudaSuccess) e = fl::fft_pow2(a.as<double2>(), t.as<double2>(), n, -1, &f, st);
    if (e == cudaSuccess) e = fl::launch_cpow(f, n, h, 1.0 / (double)n, st);
    double2* other = (f == a.as<double2>()) ? t.as<double2>() : a.as<double2>();
    if (e == cudaSuccess) e = fl::fft_pow2(f, other, n, 1, &r, st);
  }
  std::vector<double2> ho(out_len);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ho.data(), r, sizeof(double2) * out_len, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  a.release();
  t.release();
  if (e != cudaSuccess) return fail(std::string("fl_kernel_power: ") + cudaGetErrorString(e));
  for (int64_t i = 0; i < out_len; ++i) out[i] = ho[i].x;
  return 0;
}

int64_t fl_batch_device_bytes(const fl_batch* b) {
  if (!b) {
    fail("fl_batch_device_bytes: null batch");
    return -1;
  }
  int64_t t = 0;
  for (const DevBuf* d : {&b->d_stats, &b->d_snap, &b->d_snaplen, &b->d_put, &b->d_call, &b->d_euro, &b->d_orders,
                          &b->d_price, &b->d_status, &b->d_bt, &b->d_bc, &b->d_bcount, &b->d_counter, &b->d_ws_put,
                          &b->d_ws_call, &b->d_ws_base})
    t += (int64_t)d->bytes;
  return t;
}

int fl_batch_profile(fl_batch* b, uint64_t* counters56, void* stream) {
  if (!b) return fail("fl_batch_profile: null batch");
  if (!FL_PROF && !FL_STRIP_CLOCK)
    return fail("fl_batch_profile: library built without profile counters (build with FL_NVCC_FLAGS=-DFL_PROF=1)");
  FL_CUDA(cudaMemcpyAsync(counters56, b->d_stats.as<unsigned long long>() + 8, 56 * sizeof(uint64_t),
                          cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  FL_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

int fl_batch_timeline(fl_batch* b, uint64_t* out3n, void* stream) {
  if (!b || !out3n) return fail("fl_batch_timeline: null argument");
  if (!FL_PROF) return fail("fl_batch_timeline: library built without profile counters (build with FL_NVCC_FLAGS=-DFL_PROF=1)");
  FL_CUDA(cudaMemcpyAsync(out3n, b->d_stats.as<unsigned long long>() + 64, 3 * b->n * sizeof(uint64_t),
                          cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  FL_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

#if FL_TRACE
// Tool-only (FL_TRACE builds): copy the chain event trace of the last run and reset it.
int fl_trace_read(uint64_t* out, int64_t cap) {
  FL_CUDA(cudaDeviceSynchronize());
  FL_CUDA(cudaMemcpyFromSymbol(out, fl::g_trace, (size_t)cap * sizeof(uint64_t)));
  static const unsigned long long zero = 0;
  FL_CUDA(cudaMemcpyToSymbol(fl::g_trace, &zero, sizeof(zero)));
  return 0;
}
#endif

int fl_probe_fp64(double* tflops, void* stream) {
  if (!tflops) return fail("fl_probe_fp64: null output");
  FL_CUDA(fl::probe_fp64(tflops, (cudaStream_t)stream));
  return 0;
}

int fl_probe_transcendentals(double* exp_per_s, double* log_per_s, void* stream) {
  if (!exp_per_s || !log_per_s) return fail("fl_probe_transcendentals: null output");
  FL_CUDA(fl::probe_transcendentals(exp_per_s, log_per_s, (cudaStream_t)stream));
  return 0;
}

void fl_batch_free(fl_batch* b) {
  if (!b) return;
  b->release();
  delete b;
}

}  // extern "C"

namespace {

// One cached batch per (thread, device): device buffers grow and are reused
// across calls; released when the thread exits or on fl_release_cache().
struct BatchCache {
  fl_batch* b[64] = {nullptr};
  void release_all() {
    for (fl_batch*& p : b)
      if (p) {
        p->release();
        delete p;
        p = nullptr;
      }
  }
  ~BatchCache() { release_all(); }
};
thread_local BatchCache t_cache;

int price_with(fl_batch* b, int64_t n, const int8_t* kind, const double* S, const double* K, const double* R,
               const double* Y, const double* V, const double* E, const int64_t* T, double lam, int64_t call_cutoff,
               int64_t put_cutoff, int method, double* price, int32_t* status, int64_t* bnd_times,
               int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap, cudaStream_t stream,
               const double* bparams = nullptr) {
  int rc = plan_host(b, n, kind, S, K, R, Y, V, E, T, lam, call_cutoff, put_cutoff, method, bnd_cap, bparams);
  if (rc) return rc;
  rc = upload(b, stream);
  if (rc) return rc;
  rc = run(b, stream);
  if (rc) return rc;
  return fetch(b, price, status, bnd_times, bnd_cols, bnd_count, stream);
}

// Process-wide per-device batches for the multi-device entry (its worker
// threads are short-lived; the buffers persist per device, one user at a time).
std::mutex g_dev_mu[64];
fl_batch* g_dev_batch[64] = {nullptr};

}  // namespace

extern "C" {

int fl_price_batch_ex(int64_t n, const int8_t* kind, const double* S, const double* K, const double* R,
                      const double* Y, const double* V, const double* E, const int64_t* T, const double* bparams,
                      double lam, int64_t call_cutoff, int64_t put_cutoff, int method, double* price,
                      int32_t* status, int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap,
                      void* stream) {
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail("fl_price_batch: device index out of range");
  if (!t_cache.b[dev]) t_cache.b[dev] = new fl_batch();
  return price_with(t_cache.b[dev], n, kind, S, K, R, Y, V, E, T, lam, call_cutoff, put_cutoff, method, price,
                    status, bnd_times, bnd_cols, bnd_count, bnd_cap, (cudaStream_t)stream, bparams);
}

int fl_price_batch(int64_t n, const int8_t* kind, const double* S, const double* K, const double* R,
                   const double* Y, const double* V, const double* E, const int64_t* T, double lam,
                   int64_t call_cutoff, int64_t put_cutoff, int method, double* price, int32_t* status,
                   int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap, void* stream) {
  return fl_price_batch_ex(n, kind, S, K, R, Y, V, E, T, nullptr, lam, call_cutoff, put_cutoff, method, price,
                           status, bnd_times, bnd_cols, bnd_count, bnd_cap, stream);
}

void fl_release_cache(void) { t_cache.release_all(); }

int fl_shard_plan(int64_t n, const int8_t* kind, const int64_t* T, int nshard, int32_t* owner) {
  if (nshard < 1 || !owner) return fail("fl_shard_plan: nshard must be >= 1");
  // longest-processing-time greedy over the survey's cost model (shard.py)
  std::vector<double> cost(n);
  for (int64_t i = 0; i < n; ++i)
    cost[i] = kind[i] == FL_KIND_PUT ? cost_put(T[i]) : kind[i] == FL_KIND_CALL ? cost_call(T[i]) : 8.0 * (double)T[i];
  std::vector<int64_t> ord(n);
  for (int64_t i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
  std::vector<double> load(nshard, 0.0);
  for (int64_t i : ord) {
    const int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    owner[i] = r;
    load[r] += cost[i];
  }
  return 0;
}

int fl_price_batch_multi(int ndev, const int* devices, int64_t n, const int8_t* kind, const double* S,
                         const double* K, const double* R, const double* Y, const double* V, const double* E,
                         const int64_t* T, double lam, int64_t call_cutoff, int64_t put_cutoff, int method,
                         double* price, int32_t* status, int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count,
                         int32_t bnd_cap) {
  if (ndev < 1 || !devices) return fail("fl_price_batch_multi: need at least one device");
  int ndev_vis = 0;
  FL_CUDA(cudaGetDeviceCount(&ndev_vis));
  for (int d = 0; d < ndev; ++d)
    if (devices[d] < 0 || devices[d] >= ndev_vis || devices[d] >= 64)
      return fail("fl_price_batch_multi: invalid device " + std::to_string(devices[d]));
  std::vector<int32_t> owner(n);
  if (const int rc = fl_shard_plan(n, kind, T, ndev, owner.data())) return rc;
  const bool want_b = bnd_cap > 0 && bnd_times && bnd_cols && bnd_count;
  std::vector<std::string> err(ndev);
  std::vector<std::thread> th;
  for (int d = 0; d < ndev; ++d) {
    th.emplace_back([&, d] {
      std::vector<int64_t> idx;
      for (int64_t i = 0; i < n; ++i)
        if (owner[i] == d) idx.push_back(i);
      const int64_t m = (int64_t)idx.size();
      if (m == 0) return;
      const int dev = devices[d];
      if (cudaSetDevice(dev) != cudaSuccess) {
        err[d] = "cudaSetDevice failed";
        return;
      }
      // gather this shard's inputs (contiguous), price on the device's own
      // stream, scatter the results back: option i's arithmetic does not
      // depend on its shard, so results equal the single-device call's
      std::vector<int8_t> k(m);
      std::vector<double> s(m), kk(m), r(m), y(m), v(m), e(m), p(m);
      std::vector<int64_t> t(m), bt(want_b ? m * bnd_cap : 0), bc(want_b ? m * bnd_cap : 0);
      std::vector<int32_t> st(m), cnt(want_b ? m : 0);
      for (int64_t j = 0; j < m; ++j) {
        const int64_t i = idx[j];
        k[j] = kind[i]; s[j] = S[i]; kk[j] = K[i]; r[j] = R[i]; y[j] = Y[i]; v[j] = V[i]; e[j] = E[i]; t[j] = T[i];
      }
      cudaStream_t stream = nullptr;
      if (cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking) != cudaSuccess) {
        err[d] = "cudaStreamCreate failed";
        return;
      }
      int rc = 0;
      {
        std::lock_guard<std::mutex> lk(g_dev_mu[dev]);
        if (!g_dev_batch[dev]) g_dev_batch[dev] = new fl_batch();
        rc = price_with(g_dev_batch[dev], m, k.data(), s.data(), kk.data(), r.data(), y.data(), v.data(), e.data(),
                        t.data(), lam, call_cutoff, put_cutoff, method, p.data(), st.data(),
                        want_b ? bt.data() : nullptr, want_b ? bc.data() : nullptr, want_b ? cnt.data() : nullptr,
                        want_b ? bnd_cap : 0, stream);
      }
      cudaStreamDestroy(stream);
      if (rc) {
        err[d] = "device " + std::to_string(dev) + ": " + g_last_error;
        return;
      }
      for (int64_t j = 0; j < m; ++j) {
        const int64_t i = idx[j];
        price[i] = p[j];
        status[i] = st[j];
        if (want_b) {
          bnd_count[i] = cnt[j];
          std::copy(bt.begin() + j * bnd_cap, bt.begin() + (j + 1) * bnd_cap, bnd_times + i * bnd_cap);
          std::copy(bc.begin() + j * bnd_cap, bc.begin() + (j + 1) * bnd_cap, bnd_cols + i * bnd_cap);
        }
      }
    });
  }
  for (auto& x : th) x.join();
  for (int d = 0; d < ndev; ++d)
    if (!err[d].empty()) return fail("fl_price_batch_multi: " + err[d]);
  return 0;
}

int fl_apply_linear_steps(const double* x, int64_t L, int taps, double c0, double c1, double c2, int64_t h,
                          double* y, void* stream) {
  if (taps != 2 && taps != 3) return fail("fl_apply_linear_steps: taps must be 2 or 3");
  if (h < 1 || h > (1 << 30)) return fail("fl_apply_linear_steps: h out of range");
  if (!(c0 >= 0.0 && c1 >= 0.0 && c2 >= 0.0)) return fail("fl_apply_linear_steps: negative coefficient");
  const int span = taps - 1;
  const int64_t Lout = L - h * span;
  if (Lout < 1) return fail("fl_apply_linear_steps: row too narrow");
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  FL_CUDA(ensure_device_init(dev, st));
  double *dx = nullptr, *dy = nullptr;
  FL_CUDA(cudaMalloc(&dx, sizeof(double) * L));
  FL_CUDA(cudaMalloc(&dy, sizeof(double) * Lout));
  cudaError_t e = cudaMemcpyAsync(dx, x, sizeof(double) * L, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = fl::launch_linear_steps(dx, L, dy, Lout, (int)h, c0, c1, taps == 3 ? c2 : 0.0, span, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(y, dy, sizeof(double) * Lout, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(dx);
  cudaFree(dy);
  if (e != cudaSuccess) return fail(std::string("fl_apply_linear_steps: ") + cudaGetErrorString(e));
  return 0;
}

}  // extern "C"
