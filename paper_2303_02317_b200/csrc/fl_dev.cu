// fl_dev.cu -- device-pointer entry points: the caller (torch)
// owns every input and output buffer in device memory, the call is ordered on
// the caller's stream and never synchronizes it.
//
// fl_price_batch plans on the host (bit-identical derivation with glibc, then
// one H2D copy of the parameter records).  Here the inputs never leave the
// device, so the plan runs there too, from the same host_params.h code:
//   1. dev_plan_kernel   -- per option: validation, lattice / grid constants,
//                           the reference's dispatch (fast / baseline /
//                           European / closed price / error), a work-list id
//                           and a cost key; errors and closed prices are
//                           written straight to the caller's outputs;
//   2. cub radix sort    -- (list id, decreasing cost) keys, so every work
//                           list is contiguous and costliest-first (the
//                           longest chains start first);
//   3. dev_lists_kernel  -- [start, end) of every list, on the device;
//   4. the pricing kernels, launched with upper-bound grids, each reading its
//      list bounds from device memory (BatchOut::dlist);
//   5. dev_finalize_kernel -- the boundary-record fix-ups fl_price_batch does
//      on the host (records of calls priced as European; call records reversed
//      into ascending time).
// Workspaces are library-owned, cached per (thread, device, stream) and sized
// from max_steps (fl_dev_workspace_bytes), so no count is ever read back.
#include <cub/device/device_radix_sort.cuh>

namespace fl {

enum : int { DL_AMER = 0, DL_PUT_BASE, DL_CALL_BASE, DL_EURO_FAST, DL_EURO_BASE, DL_NONE, DL_COUNT };

struct DevPlan {
  PutParams* put;
  CallParams* call;
  EuroParams* euro;
  int8_t* mode;
  int8_t* kind;
  unsigned long long* key;
  int32_t* item;
};

__device__ __forceinline__ double dev_cost(int kind, int64_t n) {  // shard.py / fl_abi.cu cost model
  const double l = log2((double)(n > 2 ? n : 2));
  return kind == FL_KIND_PUT ? 24.8 * (double)n * l * l : kind == FL_KIND_CALL ? 10.0 * (double)n * l * l
                                                                               : 8.0 * (double)n;
}

__global__ void dev_plan_kernel(int64_t n, const int8_t* __restrict__ kind, int kind_all, const double* __restrict__ S,
                                const double* __restrict__ K, const double* __restrict__ R,
                                const double* __restrict__ Y, const double* __restrict__ V,
                                const double* __restrict__ E, const int64_t* __restrict__ T, double lam,
                                int64_t call_cutoff, int64_t put_cutoff, int method, int64_t max_steps, DevPlan pl,
                                BatchOut out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = kind ? kind[i] : kind_all;
    const SpecIn s{S[i], K[i], R[i], Y[i], V[i], E[i], T[i]};
    int32_t st = 0;
    int mode = MODE_ERROR, list = DL_NONE;
    switch (k) {  // the dispatch of plan_host (fl_abi.cu)
      case FL_KIND_EURO:
        st = prep_euro(s, pl.euro[i]);
        if (!st) {
          mode = method == FL_METHOD_FAST ? MODE_FAST : MODE_BASELINE;
          list = method == FL_METHOD_FAST ? DL_EURO_FAST : DL_EURO_BASE;
        }
        break;
      case FL_KIND_CALL:
        if (method == FL_METHOD_FAST) {
          st = prep_call(s, call_cutoff, pl.call[i], pl.euro[i]);
          if (!st) {
            mode = pl.call[i].mode;
            list = mode == MODE_FAST ? DL_AMER : mode == MODE_BASELINE ? DL_CALL_BASE
                                                : mode == MODE_EURO    ? DL_EURO_FAST
                                                                       : DL_NONE;
          }
        } else {
          Binom bn;
          st = derive_binomial(s, bn);
          if (!st) {
            CallParams& c = pl.call[i];
            c.S = s.S; c.K = s.K; c.wd = bn.wd; c.wu = bn.wu; c.lu = bn.lu; c.n = s.T;
            c.top_b = -1; c.junc_j = -1; c.cutoff = (int32_t)call_cutoff; c.mode = MODE_BASELINE; c.price = 0;
            mode = MODE_BASELINE;
            list = DL_CALL_BASE;
          }
        }
        break;
      case FL_KIND_PUT: {
        PutParams& p = pl.put[i];
        st = prep_put(s, lam, put_cutoff, p);
        if (method == FL_METHOD_BASELINE && (!st || st == (FL_E_VALIDATION | FL_F_CUTOFF))) {
          st = 0;
          p.mode = MODE_BASELINE;
        }
        if (!st) {
          mode = p.mode;
          list = mode == MODE_FAST ? DL_AMER : mode == MODE_BASELINE ? DL_PUT_BASE : DL_NONE;
        }
        break;
      }
      default:
        st = FL_E_VALIDATION;
    }
    // workspaces were sized for max_steps (the European fast path needs none)
    if (!st && list != DL_NONE && list != DL_EURO_FAST && s.T > max_steps) st = FL_E_CAPACITY | FL_F_STEPS;
    if (st) {
      mode = MODE_ERROR;
      list = DL_NONE;
    }
    pl.mode[i] = (int8_t)mode;
    pl.kind[i] = (int8_t)k;
    const double cost = st ? 0.0 : dev_cost(k, s.T);
    const unsigned long long lim = (1ull << 56) - 1;
    const unsigned long long c = cost >= (double)lim ? lim : (unsigned long long)cost;
    pl.key[i] = ((unsigned long long)list << 56) | (lim - c);
    pl.item[i] = (list == DL_AMER && k == FL_KIND_CALL) ? (int32_t)(-i - 1) : (int32_t)i;
    if (list == DL_NONE) {  // the outputs fetch() writes on the host path
      out.status[i] = st;
      if (st) {
        out.price[i] = __longlong_as_double(0x7ff8000000000000ll);
        if (out.bcount) out.bcount[i] = 0;
      } else {  // put, k* <= -T: closed price, one record (bsm.py:615-620)
        const PutParams& p = pl.put[i];
        out.price[i] = p.price;
        if (out.bt && out.cap > 0) {
          out.bt[i * out.cap] = 0;
          out.bc[i * out.cap] = (p.ks + p.n < 0) ? p.ks + p.n : 0;
        }
        if (out.bcount) out.bcount[i] = 1;
      }
    }
  }
}

__global__ void dev_lists_kernel(int64_t n, const unsigned long long* __restrict__ key, int32_t* __restrict__ info) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(key[i] >> 56);
    if (i == 0 || (int)(key[i - 1] >> 56) != l) info[2 * l] = (int32_t)i;
    if (i == n - 1 || (int)(key[i + 1] >> 56) != l) info[2 * l + 1] = (int32_t)(i + 1);
  }
}

__global__ void dev_finalize_kernel(int64_t n, DevPlan pl, BatchOut out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (pl.kind[i] != FL_KIND_CALL) continue;
    const int m = pl.mode[i];
    const CallParams& p = pl.call[i];
    if (m == MODE_EURO) {  // american.py:451-468: the terminal row's record only
      if (out.bt && out.cap > 0) {
        out.bt[i * out.cap] = p.n;
        out.bc[i * out.cap] = (p.top_b >= p.n) ? INT64_MIN : p.top_b + 1;
      }
      if (out.bcount) out.bcount[i] = 1;
    } else if (m == MODE_FAST && out.bt && out.cap > 0 && out.status[i] == 0) {
      // device records run T, T-1, ..., 0: ascending order
      const int64_t c = out.bcount ? (out.bcount[i] < out.cap ? out.bcount[i] : out.cap) : 0;
      int64_t* bt = out.bt + i * out.cap;
      int64_t* bc = out.bc + i * out.cap;
      for (int64_t a = 0, b = c - 1; a < b; ++a, --b) {
        const int64_t t0 = bt[a], c0 = bc[a];
        bt[a] = bt[b]; bc[a] = bc[b];
        bt[b] = t0; bc[b] = c0;
      }
    }
  }
}

}  // namespace fl

namespace {

// library-owned device workspace of the device-pointer entry
struct DevWS {
  int dev = -1;
  cudaStream_t stream = nullptr;
  int64_t cap_n = -1, cap_steps = -1;
  int method = -1;
  int64_t call_cutoff = -1, put_cutoff = -1;
  DevBuf put, call, euro, mode, kind, key, key2, item, item2, info, counter, cub, ws_am, ws_base;
  int64_t ws_am_stride = 0, ws_base_stride = 0;
  size_t cub_bytes = 0;
  int grid_am = 0, grid_base = 0, grid_euro = 0;
  int64_t base_steps = 0;
  void release() {
    for (DevBuf* b : {&put, &call, &euro, &mode, &kind, &key, &key2, &item, &item2, &info, &counter, &cub, &ws_am,
                      &ws_base})
      b->release();
    cap_n = cap_steps = -1;
  }
};

struct DevWSCache {
  std::vector<DevWS*> v;
  ~DevWSCache() { release_all(); }
  void release_all() {
    for (DevWS* w : v) {
      w->release();
      delete w;
    }
    v.clear();
  }
  DevWS* get(int dev, cudaStream_t s) {
    for (DevWS* w : v)
      if (w->dev == dev && w->stream == s) return w;
    DevWS* w = new DevWS();
    w->dev = dev;
    w->stream = s;
    v.push_back(w);
    return w;
  }
};
thread_local DevWSCache t_dev_ws;

struct DevSizes {
  int64_t am_stride, base_steps, base_stride;
  int grid_am, grid_base, grid_euro;
  size_t cub_bytes;
  int64_t total;
};

// Every device byte the entry needs for (n, max_steps): parameter records,
// sort buffers, chain arenas (put k* can reach 8 T before DomainError) and, for
// baseline rows wider than the register sweep, the global march rows.
int dev_sizes(int64_t n, int64_t max_steps, int method, int64_t call_cutoff, int64_t put_cutoff, int nsm,
              DevSizes& z) {
  const int nc = fl::put_chains_per_cta();
  const int nn = (int)std::min<int64_t>(n, INT32_MAX);
  z.grid_am = grid_for(nn, nc, nsm);
  z.am_stride = std::max(fl::put_ws_doubles(max_steps, 8 * max_steps), fl::call_ws_doubles(max_steps));
  z.base_steps = method == FL_METHOD_FAST ? std::min<int64_t>(max_steps, std::max<int64_t>(2 * put_cutoff, call_cutoff))
                                          : max_steps;
  z.grid_base = (int)std::min<int64_t>(n, 4 * (int64_t)nsm);
  z.grid_euro = (int)std::min<int64_t>(n, 16 * (int64_t)nsm);
  z.base_stride = (2 * z.base_steps + 1 > fl::sweep_max_cells() || fl::sweep_disabled())
                      ? 3 * (2 * z.base_steps + 2) + 16
                      : 0;
  size_t tmp = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs<unsigned long long, int32_t>(
      nullptr, tmp, (const unsigned long long*)nullptr, (unsigned long long*)nullptr, (const int32_t*)nullptr,
      (int32_t*)nullptr, (int)std::max<int64_t>(n, 1), 0, 64, (cudaStream_t)0);
  if (e != cudaSuccess) return fail(std::string("cub sort size query: ") + cudaGetErrorString(e));
  z.cub_bytes = tmp;
  z.total = n * (int64_t)(sizeof(fl::PutParams) + sizeof(fl::CallParams) + sizeof(fl::EuroParams) + 2 +
                          2 * (8 + 4)) +
            (int64_t)tmp + 2 * fl::DL_COUNT * 4 + 64 +
            (int64_t)sizeof(double) * z.am_stride * z.grid_am * nc +
            (int64_t)sizeof(double) * z.base_stride * z.grid_base;
  return 0;
}

}  // namespace

extern "C" {

int fl_dev_workspace_bytes(int64_t n, int64_t max_steps, int method, int64_t call_cutoff, int64_t put_cutoff,
                           int64_t* bytes) {
  if (!bytes || n < 0 || max_steps < 1) return fail("fl_dev_workspace_bytes: bad argument");
  int dev = 0, nsm = 0;
  FL_CUDA(cudaGetDevice(&dev));
  FL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  DevSizes z;
  if (const int rc = dev_sizes(n, max_steps, method, call_cutoff, put_cutoff, nsm, z)) return rc;
  *bytes = z.total;
  return 0;
}

int fl_price_batch_dev(int64_t n, const int8_t* kind, int kind_all, const double* S, const double* K, const double* R,
                       const double* Y, const double* V, const double* E, const int64_t* T, double lam,
                       int64_t call_cutoff, int64_t put_cutoff, int method, int64_t max_steps, double* price,
                       int32_t* status, int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap,
                       void* stream_v) {
  if (n < 0 || n > INT32_MAX) return fail("fl_price_batch_dev: n out of range");
  if (n == 0) return 0;
  if (max_steps < 1) return fail("fl_price_batch_dev: max_steps must be >= 1");
  if (method != FL_METHOD_FAST && method != FL_METHOD_BASELINE) return fail("fl_price_batch_dev: bad method");
  if (!kind && (kind_all < FL_KIND_EURO || kind_all > FL_KIND_PUT)) return fail("fl_price_batch_dev: bad kind_all");
  if (!S || !K || !R || !Y || !V || !E || !T || !price || !status) return fail("fl_price_batch_dev: null buffer");
  cudaStream_t stream = (cudaStream_t)stream_v;
  int dev = 0, nsm = 0;
  FL_CUDA(cudaGetDevice(&dev));
  FL_CUDA(ensure_device_init(dev, stream));
  FL_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  DevWS* w = t_dev_ws.get(dev, stream);
  if (w->cap_n < n || w->cap_steps < max_steps || w->method != method || w->call_cutoff != call_cutoff ||
      w->put_cutoff != put_cutoff) {
    DevSizes z;
    if (const int rc = dev_sizes(n, max_steps, method, call_cutoff, put_cutoff, nsm, z)) return rc;
    const int nc = fl::put_chains_per_cta();
    FL_CUDA(w->put.ensure(sizeof(fl::PutParams) * n));
    FL_CUDA(w->call.ensure(sizeof(fl::CallParams) * n));
    FL_CUDA(w->euro.ensure(sizeof(fl::EuroParams) * n));
    FL_CUDA(w->mode.ensure(n));
    FL_CUDA(w->kind.ensure(n));
    FL_CUDA(w->key.ensure(8 * n));
    FL_CUDA(w->key2.ensure(8 * n));
    FL_CUDA(w->item.ensure(4 * n));
    FL_CUDA(w->item2.ensure(4 * n));
    FL_CUDA(w->info.ensure(2 * fl::DL_COUNT * sizeof(int32_t)));
    FL_CUDA(w->counter.ensure(64));
    FL_CUDA(w->cub.ensure(z.cub_bytes));
    FL_CUDA(w->ws_am.ensure(sizeof(double) * z.am_stride * z.grid_am * nc));
    if (z.base_stride > 0) FL_CUDA(w->ws_base.ensure(sizeof(double) * z.base_stride * z.grid_base));
    w->ws_am_stride = z.am_stride;
    w->ws_base_stride = z.base_stride;
    w->grid_am = z.grid_am;
    w->grid_base = z.grid_base;
    w->grid_euro = z.grid_euro;
    w->base_steps = z.base_steps;
    w->cub_bytes = z.cub_bytes;
    w->cap_n = n;
    w->cap_steps = max_steps;
    w->method = method;
    w->call_cutoff = call_cutoff;
    w->put_cutoff = put_cutoff;
  }
  fl::BatchOut out;
  out.price = price;
  out.status = status;
  const bool want_b = bnd_cap > 0 && bnd_times && bnd_cols;
  out.bt = want_b ? bnd_times : nullptr;
  out.bc = want_b ? bnd_cols : nullptr;
  out.bcount = bnd_count;
  out.cap = want_b ? bnd_cap : 0;
  out.flops = nullptr;
  out.prof = nullptr;
  out.acct = 0;
  const fl::DevPlan pl{w->put.as<fl::PutParams>(), w->call.as<fl::CallParams>(), w->euro.as<fl::EuroParams>(),
                       w->mode.as<int8_t>(), w->kind.as<int8_t>(), w->key.as<unsigned long long>(),
                       w->item.as<int32_t>()};
  int32_t* info = w->info.as<int32_t>();
  FL_CUDA(cudaMemsetAsync(info, 0, 2 * fl::DL_COUNT * sizeof(int32_t), stream));
  const int pgrid = (int)std::min<int64_t>((n + 255) / 256, 8 * (int64_t)nsm);
  fl::dev_plan_kernel<<<pgrid, 256, 0, stream>>>(n, kind, kind_all, S, K, R, Y, V, E, T, lam, call_cutoff,
                                                  put_cutoff, method, max_steps, pl, out);
  FL_CUDA(cudaGetLastError());
  size_t tmp = w->cub_bytes;
  FL_CUDA(cub::DeviceRadixSort::SortPairs(w->cub.p, tmp, w->key.as<unsigned long long>(),
                                          w->key2.as<unsigned long long>(), w->item.as<int32_t>(),
                                          w->item2.as<int32_t>(), (int)n, 0, 64, stream));
  fl::dev_lists_kernel<<<pgrid, 256, 0, stream>>>(n, w->key2.as<unsigned long long>(), info);
  FL_CUDA(cudaGetLastError());
  const int32_t* order = w->item2.as<int32_t>();
  const int nn = (int)n;
  auto with_list = [&](int l) {
    fl::BatchOut o = out;
    o.dlist = info + 2 * l;
    return o;
  };
  FL_CUDA(fl::launch_american_fast(w->put.as<fl::PutParams>(), w->call.as<fl::CallParams>(), order, nn,
                                   w->counter.as<int32_t>(), w->ws_am.as<double>(), w->ws_am_stride, w->grid_am,
                                   with_list(fl::DL_AMER), stream));
  FL_CUDA(fl::launch_put_baseline(w->put.as<fl::PutParams>(), order, nn, w->base_steps, w->grid_base,
                                  w->ws_base.as<double>(), w->ws_base_stride, with_list(fl::DL_PUT_BASE), stream));
  FL_CUDA(fl::launch_call_baseline(w->call.as<fl::CallParams>(), order, nn, w->base_steps, w->grid_base,
                                   w->ws_base.as<double>(), w->ws_base_stride, with_list(fl::DL_CALL_BASE), stream));
  FL_CUDA(fl::launch_euro_fast(w->euro.as<fl::EuroParams>(), order, nn, w->grid_euro, with_list(fl::DL_EURO_FAST),
                               stream));
  FL_CUDA(fl::launch_euro_baseline(w->euro.as<fl::EuroParams>(), order, nn, w->base_steps, w->grid_base,
                                   w->ws_base.as<double>(), w->ws_base_stride, with_list(fl::DL_EURO_BASE), stream));
  fl::dev_finalize_kernel<<<pgrid, 256, 0, stream>>>(n, pl, out);
  FL_CUDA(cudaGetLastError());
  return 0;
}

int fl_price_put_bsm(int64_t n, const double* S, const double* K, const double* R, const double* Y, const double* V,
                     const double* E, const int64_t* T, double lam, int64_t base_cutoff, int64_t max_steps,
                     double* price, int32_t* status, int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count,
                     int32_t bnd_cap, void* stream) {
  return fl_price_batch_dev(n, nullptr, FL_KIND_PUT, S, K, R, Y, V, E, T, lam, 256, base_cutoff, FL_METHOD_FAST,
                            max_steps, price, status, bnd_times, bnd_cols, bnd_count, bnd_cap, stream);
}

int fl_price_american_call(int64_t n, const double* S, const double* K, const double* R, const double* Y,
                           const double* V, const double* E, const int64_t* T, int64_t base_cutoff, int64_t max_steps,
                           double* price, int32_t* status, int64_t* bnd_times, int64_t* bnd_cols,
                           int32_t* bnd_count, int32_t bnd_cap, void* stream) {
  return fl_price_batch_dev(n, nullptr, FL_KIND_CALL, S, K, R, Y, V, E, T, 0.4, base_cutoff, 128, FL_METHOD_FAST,
                            max_steps, price, status, bnd_times, bnd_cols, bnd_count, bnd_cap, stream);
}

int fl_price_european(int64_t n, const double* S, const double* K, const double* R, const double* Y, const double* V,
                      const double* E, const int64_t* T, double* price, int32_t* status, void* stream) {
  return fl_price_batch_dev(n, nullptr, FL_KIND_EURO, S, K, R, Y, V, E, T, 0.4, 256, 128, FL_METHOD_FAST, 1, price,
                            status, nullptr, nullptr, nullptr, 0, stream);
}

int fl_sync(void* stream) {
  FL_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

void fl_release_dev_cache(void) { t_dev_ws.release_all(); }

}  // extern "C"
