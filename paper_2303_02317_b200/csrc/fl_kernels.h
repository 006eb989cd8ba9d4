// fl_kernels.h -- device-kernel launchers shared by the C-ABI layer.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "host_params.h"

namespace fl {

// Per-option outputs (device pointers).  Boundary records are optional
// (bt == nullptr); at most `cap` records per option are stored, bcount holds
// the true count.
struct BatchOut {
  double* price;
  int32_t* status;
  int64_t* bt;
  int64_t* bc;
  int32_t* bcount;
  int32_t cap;
  unsigned long long* flops;  // [0] executed fp64 flops, [1] reference-algorithmic flops (accumulated), may be null
  unsigned long long* prof;   // optional profile counters (PROF_* in fl_sched.cuh), may be null
  // 1: the chains count executed / reference-algorithmic flops into flops[0..1];
  // 0: production runs skip the per-node accounting (an untimed accounting run
  // of the same batch supplies the counts, fl_abi.cu)
  int acct = 1;
  // optional fast-put row snapshots (record_rows): option o appends its handoff
  // segments at snap + o * snap_cap, snap_len[o] = total length (may exceed cap)
  double* snap = nullptr;
  int64_t snap_cap = 0;
  int64_t* snap_len = nullptr;
  // device-planned launches (fl_price_batch_dev): when set, the work list is
  // order[dlist[0] .. dlist[1]) (decided on the device, so the host launches
  // with an upper bound and never reads the count back)
  const int32_t* dlist = nullptr;
};

// Apply a device-side work list (BatchOut::dlist) at kernel entry.
template <class Ptr>
__device__ __forceinline__ void apply_dlist(const BatchOut& out, Ptr& order, int& nwork) {
  if (out.dlist) {
    order += out.dlist[0];
    nwork = out.dlist[1] - out.dlist[0];
  }
}

void init_twiddles(cudaStream_t stream);
cudaError_t probe_fp64(double* tflops, cudaStream_t stream);
cudaError_t probe_transcendentals(double* exp_per_s, double* log_per_s, cudaStream_t stream);

int64_t put_ws_doubles(int64_t n_max, int64_t ks_pos_max);
int put_fast_smem_bytes();
int put_chains_per_cta();
cudaError_t launch_put_fast(const PutParams* opts, const int32_t* order, int nwork, int32_t* counter, double* ws,
                            int64_t ws_stride, int grid, BatchOut out, cudaStream_t stream);
cudaError_t launch_put_baseline(const PutParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                                double* ws, int64_t ws_stride, BatchOut out, cudaStream_t stream);
int64_t put_trap_ws_doubles(int64_t f, int64_t W, int64_t h);
cudaError_t launch_put_trapezoid(const PutParams& P, int64_t f, int64_t W, int64_t h, const double* seg,
                                 double* out, int64_t* meta, int32_t* counter, double* ws, int64_t ws_stride,
                                 unsigned long long* flops, cudaStream_t stream);

cudaError_t launch_euro_fast(const EuroParams* opts, const int32_t* order, int nwork, int grid, BatchOut out,
                             cudaStream_t stream);
cudaError_t launch_euro_baseline(const EuroParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                                 double* ws, int64_t ws_stride, BatchOut out, cudaStream_t stream);

// register-resident O(T^2) sweeps (fl_sweep.cu); rows of at most sweep_max_cells()
int64_t sweep_max_cells();
bool sweep_disabled();
cudaError_t launch_put_sweep(const PutParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                             BatchOut out, cudaStream_t stream);
cudaError_t launch_put_sweep_cluster(const PutParams* opts, const int32_t* order, int nwork, int64_t n_max,
                                     BatchOut out, cudaStream_t stream);
cudaError_t launch_call_sweep(const CallParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                              BatchOut out, cudaStream_t stream);
cudaError_t launch_euro_sweep(const EuroParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                              BatchOut out, cudaStream_t stream);

int linear_steps_smem_bytes();
cudaError_t launch_linear_steps(const double* x, int64_t L, double* y, int64_t Lout, int h, double c0, double c1,
                                double c2, int span, cudaStream_t stream);

// American call (fl_call.cu)
int64_t call_ws_doubles(int64_t n_max);
int call_chains_per_cta();
int64_t call_trap_ws_doubles(int64_t width, int64_t h);
cudaError_t launch_call_trapezoid(const CallParams& P, int64_t i, int64_t j, int64_t first, int64_t h,
                                  const double* run, double* out, int64_t* meta, int32_t* counter, double* ws,
                                  int64_t ws_stride, unsigned long long* flops, cudaStream_t stream);
cudaError_t launch_call_fast(const CallParams* opts, const int32_t* order, int nwork, int32_t* counter, double* ws,
                             int64_t ws_stride, int grid, BatchOut out, cudaStream_t stream);
cudaError_t launch_call_baseline(const CallParams* opts, const int32_t* order, int nwork, int64_t n_max, int grid,
                                 double* ws, int64_t ws_stride, BatchOut out, cudaStream_t stream);

// mixed American put / call batches (fl_american.cu): work item e >= 0 is put
// option e, e < 0 call option -e-1
cudaError_t launch_american_fast(const PutParams* put, const CallParams* call, const int32_t* order, int nwork,
                                 int32_t* counter, double* ws, int64_t ws_stride, int grid, BatchOut out,
                                 cudaStream_t stream);

// grid / row snapshots for the structural APIs
cudaError_t launch_put_march_rows(const PutParams& P, const int64_t* times, int ntimes, double* snap,
                                  int64_t* last_green, double* price, double* ws, cudaStream_t stream);
cudaError_t launch_call_grid(const CallParams& P, double* rows, uint8_t* masks, int64_t* cols, double* price,
                             double* ws, cudaStream_t stream);

// European normal-limit approximations (fl_euro.cu); method 2 Gaussian, 3 closed form
cudaError_t launch_euro_approx(const EuroApprox* opts, int n_opts, int method, double* price, cudaStream_t stream);

// generic transform utilities (fl_fft.cu)
cudaError_t fft_pow2(double2* buf, double2* tmp, int64_t n, int sign, double2** result, cudaStream_t stream);
cudaError_t launch_cmul(double2* a, const double2* b, int64_t n, double scale, cudaStream_t stream);
cudaError_t launch_cscale(double2* a, int64_t n, double scale, cudaStream_t stream);
cudaError_t launch_cpow(double2* a, int64_t n, int64_t h, double scale, cudaStream_t stream);

}  // namespace fl
