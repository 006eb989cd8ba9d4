// fl_american.cu -- one persistent kernel for a batch mixing American puts and
// calls (the C4 / C5 batches): chains take work items of either kind from one
// cost-ordered queue, so the two kinds share every SM instead of running as two
// kernels back to back.  Work item e >= 0 is put option e, e < 0 call option -e-1.
#include <cstdint>

#include "fl_kernels.h"
#include "fl_sched.cuh"

namespace fl {

template <bool ACCT>  // see PutPricer: production and accounting kernel instances
struct AmericanPricer {
  const PutParams* put;
  const CallParams* call;
  const int32_t* order;
  BatchOut out;
  __device__ void chain(SchedShared& S, int c, int w, double* arena, double* scratch, double* flops) const {
    const int e = order[w];
    if (e >= 0) {
      double ref = 0.0;
      put_chain_option_retry<ACCT>(S, c, put[e], e, arena, scratch, out, flops, &ref);
      if (lane_id() == 0 && out.flops) atomicAdd(out.flops + 1, (unsigned long long)ref);
    } else {
      const int o = -e - 1;
      call_chain_option(S, c, call[o], o, arena, scratch, out, flops);
    }
  }
  __device__ double exec(SchedShared& S, const Task& t, double2* sbuf, int slots, int logN, const double2* tq,
                         const Grp& g) const {
    if (t.kind == TK_CALL_INIT || t.kind == TK_CALL_RESID) return call_exec_task(S, t, sbuf, slots, logN, tq, g);
    return put_exec_task(S, t, sbuf, slots, logN, tq, g);  // put kinds, else the generic jumps
  }
};

template <bool ACCT>
__global__ void __launch_bounds__(SCHED_THREADS, 1)
american_fast_kernel(const PutParams* __restrict__ put, const CallParams* __restrict__ call,
                     const int32_t* __restrict__ order, int nwork, int32_t* counter, double* __restrict__ ws,
                     int64_t ws_stride, BatchOut out) {
  apply_dlist(out, order, nwork);
  const AmericanPricer<ACCT> pr{put, call, order, out};
  sched_body(pr, nwork, counter, ws, ws_stride, out.flops, out.prof);
}

cudaError_t launch_american_fast(const PutParams* put, const CallParams* call, const int32_t* order, int nwork,
                                 int32_t* counter, double* ws, int64_t ws_stride, int grid, BatchOut out,
                                 cudaStream_t stream) {
  static std::atomic<unsigned long long> configured{0};
  const int smem = sched_smem_bytes();
  {
    cudaError_t e = once_per_device(configured, [&] {
      cudaError_t r = cudaFuncSetAttribute(american_fast_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(american_fast_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      return r;
    });
    if (e != cudaSuccess) return e;
  }
  if (nwork <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  if (out.acct)
    american_fast_kernel<true><<<grid, SCHED_THREADS, smem, stream>>>(put, call, order, nwork, counter, ws, ws_stride,
                                                                      out);
  else
    american_fast_kernel<false><<<grid, SCHED_THREADS, smem, stream>>>(put, call, order, nwork, counter, ws,
                                                                       ws_stride, out);
  return cudaGetLastError();
}

}  // namespace fl
