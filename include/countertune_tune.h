/*
 * countertune_tune.h -- C ABI of the live measurement path: an NVRTC variant
 * compiler + launcher for the tunable benchmark kernels and a CUPTI
 * range-profiler collector for the paper's counter set (Table 1).
 *
 * It replaces the reference's measurement plug point: the MeasurementSource
 * duck type (search.py:188-217) and the out-of-process runner protocol
 * (search.py:220-275, "runtime_us,threads,NAME=val,...").  The Python
 * CudaMeasurementSource (paper_2102_05297_b200/tuner.py) binds these
 * through ctypes and returns Measurement(runtime_us, global_threads,
 * counters) exactly as the reference's sources do.
 *
 * Conventions as countertune_b200.h: plain C types, borrowed host pointers,
 * CT_OK / negative CT_ERR_* status with ct_tune_last_error().
 */
#ifndef COUNTERTUNE_TUNE_H
#define COUNTERTUNE_TUNE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CT_TUNE_ABI_VERSION 1

#define CT_TUNE_OK              0
#define CT_TUNE_ERR_CUDA       -1   /* driver / runtime failure            */
#define CT_TUNE_ERR_VALUE      -2   /* bad argument                        */
#define CT_TUNE_ERR_COMPILE    -3   /* NVRTC rejected the variant          */
#define CT_TUNE_ERR_LAUNCH     -4   /* launch failed (invalid configuration) */
#define CT_TUNE_ERR_PROFILER   -5   /* CUPTI failure / metric unavailable  */

typedef struct ct_tuner ct_tuner;

int         ct_tune_abi_version(void);
const char* ct_tune_last_error(void);

/* one tuner per GPU: primary context, own stream, variant cache */
int ct_tuner_create(int device, ct_tuner** out);
int ct_tuner_destroy(ct_tuner* t);
/* "sm_100a" etc.; SM count; clock; copies into the caller's buffers */
int ct_tuner_device_info(ct_tuner* t, char* arch, int32_t arch_cap, int32_t* sm_count,
                         int32_t* max_threads_per_sm);

/* Compile `source` with NVRTC for this device (-arch=sm_XXa) plus the
 * caller's options (typically -D<PARAM>=<value> per tuning parameter) and
 * load `kernel_name`.  *variant receives a handle for launches.  On
 * CT_TUNE_ERR_COMPILE the NVRTC log is in ct_tune_last_error() and (if
 * given) in log[0..log_cap). */
int ct_tuner_compile(ct_tuner* t, const char* source, const char* kernel_name,
                     const char* const* options, int32_t n_options, int32_t* variant,
                     char* log, int64_t log_cap);
/* Compile n_variants variants of one source concurrently on `threads` host
 * threads (0 = all cores).  Variant i's options are options_flat[
 * sum(n_options[:i]) .. +n_options[i]).  variants[i] receives the handle (or
 * -1), status[i] CT_TUNE_OK or the variant's error (a configuration NVRTC
 * rejects is CT_TUNE_ERR_COMPILE, like an invalid configuration in the
 * reference's runner protocol, search.py:241-253).  Returns CT_TUNE_OK when
 * the batch itself ran; ct_tune_last_error() holds the first variant error. */
int ct_tuner_compile_batch(ct_tuner* t, const char* source, const char* kernel_name,
                           const char* const* options_flat, const int32_t* n_options,
                           int32_t n_variants, int32_t threads, int32_t* variants,
                           int32_t* status);
/* registers / static smem / max threads per block of a loaded variant */
int ct_tuner_variant_info(ct_tuner* t, int32_t variant, int32_t* regs, int32_t* static_smem,
                          int32_t* max_threads);
int ct_tuner_unload(ct_tuner* t, int32_t variant);

/* device memory owned by the tuner (freed by ct_tuner_destroy) */
int ct_tuner_alloc(ct_tuner* t, int64_t bytes, uint64_t* dev_ptr);
int ct_tuner_free(ct_tuner* t, uint64_t dev_ptr);
int ct_tuner_h2d(ct_tuner* t, uint64_t dev_ptr, const void* host, int64_t bytes);
int ct_tuner_d2h(ct_tuner* t, void* host, uint64_t dev_ptr, int64_t bytes);
int ct_tuner_memset(ct_tuner* t, uint64_t dev_ptr, int32_t value, int64_t bytes);

/* Kernel launch geometry + arguments: args is a packed blob, arg_offsets[i]
 * the byte offset of argument i (cuLaunchKernel kernelParams). */
typedef struct {
    uint32_t grid[3];
    uint32_t block[3];
    uint32_t dynamic_smem;
    const void* args;
    const int32_t* arg_offsets;
    int32_t n_args;
} ct_launch;

/* `warmup` untimed launches, then `reps` launches each timed with CUDA
 * events on the tuner's stream; flush_l2 != 0 writes a buffer larger than
 * L2 between timed launches (outside the timed region).  times_us[reps]. */
int ct_tuner_time(ct_tuner* t, int32_t variant, const ct_launch* l, int32_t warmup,
                  int32_t reps, int32_t flush_l2, double* times_us);

/* CUPTI range profiler: collect `n_metrics` metrics (Volta+ names, e.g.
 * "dram__sectors_read.sum") over one launch of the variant, replaying the
 * kernel once per pass (user replay; the benchmark kernels are idempotent).
 * values[n_metrics]; *passes receives the number of replay passes used. */
int ct_tuner_profile(ct_tuner* t, int32_t variant, const ct_launch* l,
                     const char* const* metrics, int32_t n_metrics, double* values,
                     int32_t* passes);

/* The same collection for k launches at once (an exhaustive sweep): one
 * range per launch, every pass launches all k, so the profiler's
 * per-collection cost (configuration, the SASS-instrumentation passes) is
 * paid once per k configurations.  values[k * n_metrics], row i = launch i. */
int ct_tuner_profile_batch(ct_tuner* t, int32_t k, const int32_t* variants,
                           const ct_launch* launches, const char* const* metrics,
                           int32_t n_metrics, double* values, int32_t* passes);

/* Number of replay passes the metric set needs on this device (host-side
 * configuration only, no launch). */
int ct_tuner_profile_passes(ct_tuner* t, const char* const* metrics, int32_t n_metrics,
                            int32_t* passes);

/* Accumulated wall time of ct_tuner_profile by phase, microseconds:
 * [0] counter-data init + SetConfig, [1] replay passes (range + launch),
 * [2] stream sync, [3] DecodeData, [4] metric evaluation, [5] number of
 * calls, [6] replay passes, [7] host-configuration builds.  reset != 0
 * clears the counters after reading. */
/* A 2-D fp32 TMA tensor map (CUtensorMap, 128 bytes into out128) of the
 * dim1 x dim0 row-major array at dev_ptr (dim0 contiguous, rows
 * row_stride_bytes apart), box box1 x box0, no swizzle, no interleave --
 * passed by value to kernels that load with cp.async.bulk.tensor. */
int ct_tuner_tensor_map_2d(ct_tuner* t, uint64_t dev_ptr, uint64_t dim0, uint64_t dim1,
                           uint64_t row_stride_bytes, uint32_t box0, uint32_t box1,
                           void* out128);

int ct_tuner_profile_timing(ct_tuner* t, double* out8, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* COUNTERTUNE_TUNE_H */
