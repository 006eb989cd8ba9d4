/* fftlattice_b200.h -- C ABI of the B200-native fftlattice pricing library.
 *
 * Drop-in boundary for the reference package `fftlattice` (pure Python; its
 * pricing entry points are plain functions, no plugin registry).  Each entry
 * point below replaces the reference function named beside it; the reference
 * binding a maintainer would add is the ctypes stub in INTEGRATION.md.
 *
 * Conventions
 *  - Plain C types only: host pointers to struct-of-arrays option inputs,
 *    host pointers for outputs, an optional cudaStream_t passed as void*.
 *  - Returns 0 on success, nonzero on a launch / configuration error
 *    (message via fl_last_error()).  Per-option pricing failures are NOT call
 *    errors: they are reported in status[i] (see paper_2303_02317_b200/csrc/
 *    fl_status.h: (class << 8) | detail, classes mirroring model.py:44-97).
 *  - Boundary records are optional (pass NULL); at most bnd_cap records per
 *    option are stored row-major at [i * bnd_cap], bnd_count[i] holds the true
 *    count.  Columns use the reference sentinel NO_GREEN = INT64_MIN.
 *  - The host-buffer entry points synchronize the given stream before
 *    returning, except fl_batch_run, which only enqueues.  The device-pointer
 *    entry points (fl_price_batch_dev, fl_price_put_bsm,
 *    fl_price_american_call, fl_price_european) never synchronize: they only
 *    enqueue on the caller's stream (fl_sync waits for it).
 *  - Reentrant across devices; one library context per device.
 */
#ifndef FFTLATTICE_B200_H
#define FFTLATTICE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FL_KIND_EURO 0 /* binomial European call  */
#define FL_KIND_CALL 1 /* binomial American call  */
#define FL_KIND_PUT 2  /* BSM American put        */

#define FL_METHOD_FAST 0     /* fast_european / fast_american_call / fast_put_bsm        */
#define FL_METHOD_BASELINE 1 /* baseline_european / baseline_american_call / baseline_put_fd */
#define FL_METHOD_GAUSS 2    /* gaussian_approx_european (fl_euro_approx only)                */
#define FL_METHOD_CLOSED 3   /* closed_form_european (fl_euro_approx only)                    */

/* Library version (major*10000 + minor*100 + patch). */
int fl_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char* fl_last_error(void);

/* Price a batch of options of mixed kinds.
 *   kind[i] in {FL_KIND_*}; S,K,R,Y,V,E as in fftlattice.OptionSpec
 *   (spot, strike, rate, dividend_yield, volatility, days_to_expiry; Y is
 *   validated but unused for puts, as in the reference); T = steps.
 *   lam: BSM grid ratio (bsm.py:66 default 0.4); call_cutoff / put_cutoff:
 *   the reference base_cutoff arguments (defaults 256 / 128).
 * Replaces, per option:
 *   FL_KIND_EURO + FAST      binomial.py:161  fast_european
 *   FL_KIND_EURO + BASELINE  binomial.py:80   baseline_european
 *   FL_KIND_CALL + FAST      american.py:428  fast_american_call
 *   FL_KIND_CALL + BASELINE  binomial.py:94   baseline_american_call
 *   FL_KIND_PUT  + FAST      bsm.py:585       fast_put_bsm
 *   FL_KIND_PUT  + BASELINE  bsm.py:273       baseline_put_fd
 * and cli.py:753-794 (_batch_row_price) for a whole portfolio at once. */
int fl_price_batch(int64_t n, const int8_t* kind, const double* S, const double* K, const double* R,
                   const double* Y, const double* V, const double* E, const int64_t* T, double lam,
                   int64_t call_cutoff, int64_t put_cutoff, int method, double* price, int32_t* status,
                   int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap, void* stream);

/* fl_price_batch with caller-supplied lattice constants for binomial options
 * (the reference pricers' `params=` argument: binomial.py:80/161,
 * american.py:428): bparams is n x 4 doubles {weight_down, weight_up, log_up,
 * step_years}; a row whose weight_down is NaN (or bparams == NULL) derives them
 * from the spec as fl_price_batch does.  Puts ignore it. */
int fl_price_batch_ex(int64_t n, const int8_t* kind, const double* S, const double* K, const double* R,
                      const double* Y, const double* V, const double* E, const int64_t* T, const double* bparams,
                      double lam, int64_t call_cutoff, int64_t put_cutoff, int method, double* price,
                      int32_t* status, int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap,
                      void* stream);

/* Release the calling thread's cached batch buffers (fl_price_batch keeps one
 * grow-only batch per (thread, device); they are also freed at thread exit). */
void fl_release_cache(void);

/* Cost-balanced shard plan: longest-processing-time greedy over
 * the per-option cost model (put 24.8 T log2^2 T, American call 10 T log2^2 T,
 * European 8 T); owner[i] in [0, nshard).  Host-only. */
int fl_shard_plan(int64_t n, const int8_t* kind, const int64_t* T, int nshard, int32_t* owner);

/* fl_price_batch across several GPUs of this process in one call: options are
 * LPT-sharded over devices[0..ndev), each shard priced by its own host thread
 * on its own stream and device, results scattered back into the host outputs.
 * Per-option results are bit-identical to fl_price_batch on one device.
 * Replaces the reference's sequential portfolio loop (cli.py:820-841). */
int fl_price_batch_multi(int ndev, const int* devices, int64_t n, const int8_t* kind, const double* S,
                         const double* K, const double* R, const double* Y, const double* V, const double* E,
                         const int64_t* T, double lam, int64_t call_cutoff, int64_t put_cutoff, int method,
                         double* price, int32_t* status, int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count,
                         int32_t bnd_cap);

/* Device-pointer entry: every array argument is a DEVICE
 * pointer owned by the caller (e.g. torch data_ptr()), the work is enqueued on
 * `stream` and the call returns without synchronizing.  Same semantics,
 * statuses and boundary records as fl_price_batch; kind == NULL prices every
 * option as kind_all.  The plan (validation, lattice constants, dispatch,
 * costliest-first work lists) runs on the device from the same derivation code
 * with the CUDA libm, so constants may differ from the host path's in the
 * last bit (prices agree within the parity tolerance).  Workspaces are sized
 * for T <= max_steps; an option with T > max_steps (other than a European,
 * which needs none) gets status FL_E_CAPACITY | 7.  Replaces, per kind, the
 * call sites binomial.py:161, american.py:428 and bsm.py:585. */
int fl_price_batch_dev(int64_t n, const int8_t* kind, int kind_all, const double* S, const double* K, const double* R,
                       const double* Y, const double* V, const double* E, const int64_t* T, double lam,
                       int64_t call_cutoff, int64_t put_cutoff, int method, int64_t max_steps, double* price,
                       int32_t* status, int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap,
                       void* stream);
/* bsm.py:585 fast_put_bsm over a device batch (fl_price_batch_dev, kind PUT). */
int fl_price_put_bsm(int64_t n, const double* S, const double* K, const double* R, const double* Y, const double* V,
                     const double* E, const int64_t* T, double lam, int64_t base_cutoff, int64_t max_steps,
                     double* price, int32_t* status, int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count,
                     int32_t bnd_cap, void* stream);
/* american.py:428 fast_american_call over a device batch (kind CALL). */
int fl_price_american_call(int64_t n, const double* S, const double* K, const double* R, const double* Y,
                           const double* V, const double* E, const int64_t* T, int64_t base_cutoff, int64_t max_steps,
                           double* price, int32_t* status, int64_t* bnd_times, int64_t* bnd_cols,
                           int32_t* bnd_count, int32_t bnd_cap, void* stream);
/* binomial.py:161 fast_european over a device batch (kind EURO; no workspace). */
int fl_price_european(int64_t n, const double* S, const double* K, const double* R, const double* Y, const double* V,
                      const double* E, const int64_t* T, double* price, int32_t* status, void* stream);
/* Device bytes fl_price_batch_dev allocates for (n, max_steps) on the current
 * device (library-owned, cached per thread, device and stream). */
int fl_dev_workspace_bytes(int64_t n, int64_t max_steps, int method, int64_t call_cutoff, int64_t put_cutoff,
                           int64_t* bytes);
/* Wait for every call enqueued on `stream` (the only synchronizing call of the
 * device-pointer API). */
int fl_sync(void* stream);
/* Free the calling thread's device-pointer workspaces. */
void fl_release_dev_cache(void);

/* Host-only (no CUDA call): the per-option constants and dispatch the batch
 * entry points derive, for inspection and CPU-side parity tests.
 *   mode[i]: -1 error, 0 device D&C, 1 O(T^2) baseline, 2 closed price,
 *            3 European (American call the reference prices as European)
 *   EURO: dparams = {wd, wu, gauged wu e^{2 lu}, lu}     (binomial.py:161-194)
 *   CALL: dparams = {wd, wu, lu, closed price}, iparams = {terminal boundary,
 *         row T-1 boundary}                             (american.py:260-470)
 *   PUT:  dparams = {cd, cm, cu, ds}, iparams = {k*, sliding-strip flag}
 *                                                       (bsm.py:150-229, 585-625)
 * dparams: n x 4 doubles, iparams: n x 2 int64. */
int fl_inspect(int64_t n, const int8_t* kind, const double* S, const double* K, const double* R, const double* Y,
               const double* V, const double* E, const int64_t* T, double lam, int64_t call_cutoff,
               int64_t put_cutoff, int32_t* status, int32_t* mode, double* dparams, int64_t* iparams);

/* Device-resident batches (for repeated pricing and benchmarking): prepare
 * does the host-side parameter derivation and the H2D copy once; run only
 * enqueues the kernels on `stream` (inputs and outputs stay in HBM); fetch
 * copies results back and synchronizes. */
typedef struct fl_batch fl_batch;
int fl_batch_prepare(fl_batch** out, int64_t n, const int8_t* kind, const double* S, const double* K,
                     const double* R, const double* Y, const double* V, const double* E, const int64_t* T,
                     double lam, int64_t call_cutoff, int64_t put_cutoff, int method, int32_t bnd_cap,
                     void* stream);
int fl_batch_run(fl_batch* b, void* stream);
int fl_batch_fetch(fl_batch* b, double* price, int32_t* status, int64_t* bnd_times, int64_t* bnd_cols,
                   int32_t* bnd_count, void* stream);
/* Device memory the batch holds (bytes): parameter records, outputs and the
 * per-chain workspaces (the arenas of the recursion rows, payoff tables and
 * kernel tables); -1 on a null batch.  The workspace-size query of SURVEY
 * 8(b): size a batch against the 180 GB of one B200 before pricing. */
int64_t fl_batch_device_bytes(const fl_batch* b);
/* Number of kernel launches one fl_batch_run enqueues. */
int fl_batch_launches(const fl_batch* b);
/* After a run: fp64 flops the fast kernels executed in it (FFT convention
 * 5 C log2 C per complex transform + 5 per explicit cell), and the bytes the
 * last prepare / fetch moved H2D / D2H. */
int fl_batch_stats(fl_batch* b, double* fp64_flops, int64_t* h2d_bytes, int64_t* d2h_bytes, void* stream);
/* After a run: the REFERENCE-ALGORITHMIC fp64 flops of the batch -- the work
 * the reference decomposition at its base_cutoff performs (5 flops per
 * projected cell of each reference strip; 5 N log2 N + 6 (N/2+1) per
 * reference FFT jump of size N = next_pow2(L + M - 1)), counted by the fast
 * kernels as they walk the same recursion.  The roofline numerator.  Production
 * runs skip the per-node counting (it costs ~5 % on the chains' critical
 * path): the first stats / ref-flops query of a prepared batch makes one extra,
 * untimed accounting run of the same kernel on the same inputs (results are
 * deterministic, so the counts are exact for every run of the batch). */
int fl_batch_ref_flops(fl_batch* b, double* ref_flops, void* stream);
void fl_batch_free(fl_batch* b);
/* Scheduler profile counters of the last run (requires FL_PROFILE set in the
 * environment at run time; zeros otherwise): 56 uint64 slots, see PROF_* in
 * csrc/fl_sched.cuh. */
int fl_batch_profile(fl_batch* b, uint64_t* counters56, void* stream);
/* Per-work-item timeline of the last fast run (FL_PROFILE set): 3 uint64 per
 * work item in scheduling (decreasing-cost) order: start ns, end ns, SM << 1 | chain. */
int fl_batch_timeline(fl_batch* b, uint64_t* out3n, void* stream);

/* Batched valid-mode composed-stencil correlation (fft.py:263 apply_linear_steps,
 * american.py:180 / bsm.py:384 _valid_corr), on host buffers:
 *   y[k] = sum_{r=0}^{h*(taps-1)} W_h[r] x[k+r],  k = 0 .. L - h*(taps-1) - 1,
 * W_h = coefficients of (c0 + c1 z [+ c2 z^2])^h (fft.py:203 kernel_power).
 * taps in {2,3}; coefficients must be nonnegative (lattice / FD weights). */
int fl_apply_linear_steps(const double* x, int64_t L, int taps, double c0, double c1, double c2, int64_t h,
                          double* y, void* stream);

/* One boundary-tracking stage of the put from a given row state
 * (bsm.py:504 solve_bsm_trapezoid / _advance_stage bsm.py:557-582).
 * Grid: weights cd, cm, cu and spacing ds of a BsmDiscretization; base_cutoff
 * as in the reference (work accounting only).  Input: boundary f and the
 * continuation values of columns f+1 .. f+W (host, W >= 2h).  Output: new
 * boundary *kp, values of columns kp+1 .. f+W-h into out_seg (capacity W+h),
 * *status = 0 or a GeometryError code. */
int fl_put_trapezoid(double cd, double cm, double cu, double ds, int64_t base_cutoff, int64_t f,
                     const double* seg, int64_t W, int64_t h, double* out_seg, int64_t* kp, int32_t* status,
                     void* stream);

/* One trapezoid of the American call (american.py:298 solve_trapezoid):
 * lattice S, K, wd, wu, lu (BinomialParams weight_down / weight_up / log_up),
 * row i, boundary j, red run of columns first .. j (host), height h.
 * Output: boundary *jp of row i-h and the red values of columns first .. jp
 * into out_run (capacity j-first+1), *status = 0 or a GeometryError code. */
int fl_call_trapezoid(double S, double K, double wd, double wu, double lu, int64_t base_cutoff, int64_t i,
                      int64_t j, int64_t first, const double* run, int64_t h, double* out_run, int64_t* jp,
                      int32_t* status, void* stream);

/* binomial.py:94 baseline_american_call(keep_grid=True): the projected
 * induction with every row retained (binomial.py:133-158): rows packed, row i
 * (i+1 values) at offset i(i+1)/2; masks the same layout (1 = exercise);
 * cols[i] = first exercise column of row i or INT64_MIN.  steps <= 32768. */
int fl_call_grid(double S, double K, double wd, double wu, double lu, int64_t n, double* rows, uint8_t* masks,
                 int64_t* cols, double* price, void* stream);

/* bsm.py:273 baseline_put_fd(record_rows=times): the O(T^2) march of one put
 * (grid weights cd, cm, cu, spacing ds, anchor k*, strike K, n steps) with the
 * valid window of each requested row (increasing times in [1, n]) packed into
 * snap: row t contributes 2n+1-2t values for columns k*-n+t .. k*+n-t.
 * last_green[0..n]: the boundary record (window offsets already converted to
 * columns, INT64_MIN once the window loses the boundary). */
int fl_put_march_rows(double cd, double cm, double cu, double ds, double K, int64_t ks, int64_t n,
                      const int64_t* times, int ntimes, double* snap, int64_t snap_cap, int64_t* last_green,
                      double* price, void* stream);

/* bsm.py:585 fast_put_bsm(record_rows=True): one put (Y = 0) priced by the
 * fast path with the continuation segment of every stage-handoff row appended
 * to snap (capacity snap_cap doubles; *snap_len = total length needed): the
 * row recorded at (times[k], cols[k]), k >= 1, holds columns cols[k]+1 ..
 * k* + T - times[k].  Price, status and boundary record as fl_price_batch. */
int fl_put_fast_rows(double S, double K, double R, double V, double E, int64_t T, double lam, int64_t base_cutoff,
                     double* snap, int64_t snap_cap, int64_t* snap_len, double* price, int32_t* status,
                     int64_t* bnd_times, int64_t* bnd_cols, int32_t* bnd_count, int32_t bnd_cap, void* stream);

/* binomial.py:218 gaussian_approx_european (method FL_METHOD_GAUSS) and
 * binomial.py:243 closed_form_european (FL_METHOD_CLOSED) for a batch of
 * European calls; per-option status as fl_price_batch (DomainError for a
 * degenerate window / non-positive strike). */
int fl_euro_approx(int64_t n, const double* S, const double* K, const double* R, const double* Y, const double* V,
                   const double* E, const int64_t* T, int method, double* price, int32_t* status, void* stream);

/* fft.py:84 fft_forward / fft.py:114 fft_inverse: unnormalised power-of-two
 * DFT (inverse with the 1/N factor) of n complex values, interleaved
 * (re, im) doubles, host buffers. */
int fl_fft(const double* in, int64_t n, int inverse, double* out, void* stream);

/* fft.py:203-260 kernel_power for a generic kernel (any number of taps, any
 * finite real weights): the zero-padded spectrum raised to the h-th power
 * and inverted on the device (a one-tap kernel: its weight to the h-th
 * power).  out receives h (L - 1) + 1 weights.  The pricers' own two- and
 * three-tap nonnegative kernels take fl_apply_linear_steps' analytic path. */
int fl_kernel_power(const double* w, int64_t L, int64_t h, double* out, void* stream);

/* fft.py:130 convolve: full linear convolution of two complex sequences
 * (interleaved re, im; real inputs with zero imaginary parts), zero-padded to
 * the next power of two >= nx + ny - 1; out receives nx + ny - 1 complex values. */
int fl_convolve(const double* x, int64_t nx, const double* y, int64_t ny, double* out, void* stream);

/* Measured FP64 (DFMA) throughput of the current device in TFLOP/s: the
 * roofline denominator bench.py reports against. */
int fl_probe_fp64(double* tflops, void* stream);

/* Measured fp64 exp and log throughput of the current device (evaluations per
 * second): the European path's roofline counts each at its DFMA-equivalent
 * cost. */
int fl_probe_transcendentals(double* exp_per_s, double* log_per_s, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FFTLATTICE_B200_H */
