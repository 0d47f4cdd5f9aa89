/*
 * countertune_b200.h -- C ABI of the B200 searcher hot path.
 *
 * The reference (`countertune`, pure Python + numpy) has no native code and
 * therefore no FFI of its own.  Each entry point below replaces one function
 * of the reference's Python API on the searcher's data-parallel hot path; the
 * replaced interface is cited as <file>:<line> relative to
 * /root/reference/pkg/src/countertune/.  The Python mirror in
 * paper_2102_05297_b200/ binds these through ctypes.
 *
 * Conventions
 *   - plain C types only; host pointers are borrowed for the duration of the
 *     call and never retained;
 *   - every function returns CT_OK (0) or a negative CT_ERR_* status and
 *     leaves a message in ct_last_error() (thread-local); no C++ exception
 *     ever crosses the boundary;
 *   - one ct_ctx per GPU; calls on one context are serialised by the caller;
 *     different contexts may be driven from different host threads;
 *   - all floating point is IEEE binary64, evaluated in the reference's
 *     operation order (no FMA contraction on the parity path).
 */
#ifndef COUNTERTUNE_B200_H
#define COUNTERTUNE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CT_ABI_VERSION 1

/* status codes; the Python shim maps them onto the reference's exception
 * classes (errors.py:4-43) */
#define CT_OK                 0
#define CT_ERR_CUDA          -1  /* CUDA runtime failure                  -> CounterTuneError      */
#define CT_ERR_VALUE         -2  /* bad argument (search.py:353-356,177)  -> ValueError            */
#define CT_ERR_EXHAUSTED     -3  /* empty pool (search.py:155,183)        -> SpaceExhaustedError   */
#define CT_ERR_NO_RECORD     -4  /* replay miss (search.py:209)           -> CounterTuneError      */
#define CT_ERR_MISMATCH      -5  /* table/space mismatch (search.py:69)   -> CounterTuneError      */
#define CT_ERR_STATE         -6  /* call-order error (no table uploaded)  -> CounterTuneError      */
#define CT_ERR_NONFINITE     -7  /* NaN weight reached selection          -> CounterTuneError      */
#define CT_ERR_UNSUPPORTED   -8  /* feature outside the device path       -> CounterTuneError      */

/* SearchTrace.status (search.py:33-35) */
#define CT_STATUS_BUDGET      0
#define CT_STATUS_STOPPED     1
#define CT_STATUS_EXHAUSTED   2
#define CT_STATUS_ERROR       3  /* see ct_rep_error codes below */

/* number of counters analyze() reads, REQUIRED_COUNTERS order
 * (bottlenecks.py:21-30) */
#define CT_N_REQUIRED 23
/* number of keys react() emits, insertion order (bottlenecks.py:216-229) */
#define CT_N_DELTA 18
/* most keys a single score_configurations call may carry */
#define CT_MAX_SCORE_KEYS 32

typedef struct ct_ctx ct_ctx;

/* ---- context ---------------------------------------------------------- */
int         ct_abi_version(void);
const char* ct_last_error(void);
int         ct_device_count(int* count);
int         ct_create(int device, ct_ctx** out);
int         ct_destroy(ct_ctx* ctx);
/* launch on an external cudaStream_t (e.g. torch's current stream); NULL
 * restores the context's own stream */
int         ct_set_stream(ct_ctx* ctx, void* cuda_stream);
int         ct_synchronize(ct_ctx* ctx);

/* ---- resident inputs -------------------------------------------------- */

/* PredictionTable.matrix (search.py:38-63): n_configs x n_counters float64,
 * row-major as the reference stores it.  Stored on the device column-major
 * (one contiguous float64 column per counter). */
int ct_table_upload(ct_ctx* ctx, const double* matrix_rowmajor,
                    int64_t n_configs, int32_t n_counters);

/* Parameter assignments (space.py:67-104), n_configs x n_params row-major;
 * only needed for score_top_k (search.py:133-140). */
int ct_space_upload(ct_ctx* ctx, const double* assignments_rowmajor,
                    int64_t n_configs, int32_t n_params);

/* DatasetReplaySource (search.py:197-217) over Dataset.records
 * (space.py:130-174): per configuration runtime_us, global_threads and the
 * 23 REQUIRED_COUNTERS (row-major n x 23).  has_record[i] == 0 marks a
 * configuration without a measurement (measuring it is an error).
 * stop_mask (nullable) is the well-performing set (space.py:177-186). */
int ct_replay_upload(ct_ctx* ctx, int64_t n_configs, const double* runtime_us,
                     const int64_t* global_threads, const double* counters_rowmajor,
                     const uint8_t* has_record, const uint8_t* stop_mask);

/* ---- single-call hot-path functions ------------------------------------ */

/* score_configurations (search.py:89-141).  delta_columns[k] is the table
 * column of the k-th delta key in react() insertion order (-1: the table has
 * no such counter), delta_values[k] its value.  explored: n bytes.
 * score_top_k < 0 means None.  raw_out: n float64.  scoreable_out (n bytes,
 * nullable) receives the top-K mask; *has_scoreable tells whether top-K was
 * applied (ScoreVector.scoreable is None otherwise). */
int ct_score(ct_ctx* ctx, int64_t profile_index, const int32_t* delta_columns,
             const double* delta_values, int32_t n_delta, const uint8_t* explored,
             int32_t literal_sign, int64_t score_top_k, double* raw_out,
             uint8_t* scoreable_out, int32_t* has_scoreable);

/* normalize_scores (search.py:144-172): pool = scoreable & ~explored.
 * Weights use a correctly rounded x**8 (the reference's numpy pow is within
 * 1 ulp of it); norm_out: n float64.  Returns CT_ERR_EXHAUSTED on an empty
 * pool. */
int ct_normalize(ct_ctx* ctx, const double* raw, const uint8_t* pool, int64_t n,
                 double gamma, double* norm_out);

/* weighted_select (search.py:175-185) with the uniform u = rng.random()
 * already drawn by the caller.  The inverse-CDF index is found on an exact
 * fixed-point prefix of the weights and certified against the rounding of
 * the reference's sequential float cumsum; an uncertified draw is re-decided
 * on the device with the sequential float64 cumsum.  *certified_out = 1 when
 * the exact and sequential decisions provably agree. */
int ct_select(ct_ctx* ctx, const double* norm, int64_t n, double u,
              int64_t* chosen_out, int32_t* certified_out);

/* analyze() + react() (bottlenecks.py:115-230) on the device for one
 * measured counter map (REQUIRED_COUNTERS order).  out37 receives the 18
 * bottleneck components (COMPONENT_NAMES order), the 18 deltas (react()
 * insertion order) and the degenerate_instructions flag as 0.0 / 1.0. */
int ct_analyze_react(ct_ctx* ctx, const double* counters23, int32_t generation, int64_t cores,
                     int64_t global_threads, double inst_reaction, double issue_delta_sign,
                     double* out37);

/* Diagnostics: the device's inline IEEE division (ct_hd.cuh dvd_fast)
 * against __ddiv_rn on n generated operand pairs of 4 kinds (raw bit
 * patterns, small integers, two Eq. 16 shapes); *mismatches counts pairs
 * whose quotients differ in any bit (NaN == NaN).  first_bad (nullable,
 * 16 doubles) receives a, b, fast, reference of the first mismatch per kind. */
int ct_check_division(ct_ctx* ctx, int64_t n, uint64_t seed, int64_t* mismatches,
                      double* first_bad);

/* ---- batched replay searches (harness.py:139-163) ---------------------- */

typedef struct {
    int32_t outer_iterations;      /* i  (search.py:338)                    */
    int32_t inner_steps;           /* n  (search.py:338)                    */
    double  inst_reaction;         /* bottlenecks.py:62-65                  */
    double  issue_delta_sign;      /* bottlenecks.py:60                     */
    double  gamma;                 /* search.py:30                          */
    int32_t literal_sign;          /* search.py:126                         */
    int64_t score_top_k;           /* < 0: None (search.py:133)             */
    int32_t use_stop;              /* stop_indices is not None              */
    int32_t generation;            /* 0 pre_volta, 1 volta_plus (counters.py:30-31) */
    int64_t cores;                 /* ArchProfile.cores (counters.py:151)   */
    int32_t delta_columns[CT_N_DELTA]; /* table column per react() key, -1 absent */
} ct_search_params;

/* numpy SeedSequence of repetition r (harness.py:135-136):
 *   SeedSequence(entropy, spawn_key = spawn_prefix [+ (rep_offset + r,)]) */
typedef struct {
    const uint32_t* entropy;       /* entropy as little-endian uint32 words */
    int32_t         n_entropy;
    const uint32_t* spawn_prefix;  /* spawn key words                       */
    int32_t         n_prefix;
    int32_t         child_per_rep; /* 1: append (rep_offset + r) to the key */
    int64_t         rep_offset;
} ct_seed_spec;

typedef struct {
    int64_t configs_scored;        /* sum of pool sizes at scoring time     */
    int64_t draws;                 /* weighted draws made                   */
    int64_t uncertified;           /* draws re-decided by sequential cumsum */
    int64_t outer_iterations;      /* outer iterations executed             */
    int64_t algorithmic_bytes;     /* sum over scorings of pool * (8 * C_used + 16) */
} ct_batch_stats;

/* run_profile_search (search.py:338-399) for n_reps repetitions on the
 * resident table + replay data.  Launches asynchronously; results stay on
 * the device until ct_profile_results(). */
int ct_profile_search_launch(ct_ctx* ctx, const ct_search_params* params,
                             const ct_seed_spec* seeds, int32_t n_reps);

/* run_random_search (search.py:317-335); max_steps < 0 means None. */
int ct_random_search_launch(ct_ctx* ctx, const ct_seed_spec* seeds, int32_t n_reps,
                            int64_t max_steps, int32_t use_stop);

/* Trajectories of the last launch.  step_index / step_profiled are
 * n_reps x max_steps (row-major, max_steps = ct_result_max_steps()),
 * n_steps / status / rep_error are n_reps each (rep_error: CT_ERR_* of a
 * repetition that stopped with CT_STATUS_ERROR, else 0).  Slots past a
 * repetition's steps are 0, except that an error repetition's failing
 * configuration index follows its steps.  Any pointer may be NULL.
 * Synchronises. */
int ct_result_max_steps(ct_ctx* ctx, int64_t* max_steps);
int ct_fetch_results(ct_ctx* ctx, int32_t* step_index, uint8_t* step_profiled,
                     int32_t* n_steps, int32_t* status, int32_t* rep_error,
                     ct_batch_stats* stats);

/* Device pointers of the last launch's result buffers (for zero-copy
 * consumers such as torch); valid until the next launch. */
int ct_result_device_ptrs(ct_ctx* ctx, void** step_index, void** step_profiled,
                          void** n_steps, void** status);

/* ---- batched model inference (search.py:54-63 over models.py:310-333) ---
 * A trained ModelSet flattened by paper_2102_05297_b200.models.
 * compile_model_program: trees as node arrays (feature -1 = leaf), per
 * column either a tree root or a key-sorted list of binary-subspace
 * regression models (key bits = binary parameters in declared order, first
 * parameter most significant), each a list of terms (kind 0 intercept,
 * 1 lin, 2 quad, 3 cross; p1/p2 parameter positions; coefficient). */
typedef struct {
    int32_t n_cols, n_nodes, n_models, n_terms, n_binary;
    const int32_t* node_feature;
    const int32_t* node_left;
    const int32_t* node_right;
    const double*  node_threshold;
    const double*  node_value;
    const int32_t* col_root;
    const int32_t* col_model_first;
    const int32_t* col_model_count;
    const uint64_t* model_key;
    const int32_t* model_term_first;
    const int32_t* model_term_count;
    const int32_t* term_kind;
    const int32_t* term_p1;
    const int32_t* term_p2;
    const double*  term_coef;
    const int32_t* binary_pos;
} ct_model_program;

/* PredictionTable.from_model_set for a whole space on the GPU: every
 * configuration's predicted counters, clamped at 0, 0 where the reference
 * omits a counter (no model for the subspace) -- bit-identical to the
 * reference.  The result also becomes the context's resident prediction
 * table (as ct_table_upload would make it); out_rowmajor (nullable,
 * n x n_cols) receives a host copy. */
int ct_model_predict(ct_ctx* ctx, const ct_model_program* prog, const double* assign_rowmajor,
                     int64_t n_configs, int32_t n_params, double* out_rowmajor);

/* ---- on-device aggregation of the last launch (harness.py:187-244) ------
 * The ConvergenceReport statistics computed where the trajectories live, with
 * the reference's float operations in its order (sequential sums over
 * repetitions), so that reports stay byte-identical while only O(R + steps)
 * numbers cross PCIe.  Repetitions split over several contexts are chained:
 * the *_init arrays (nullable = zeros) carry the partial sums of the
 * contexts holding the earlier repetitions.
 *
 * ct_aggregate_steps: per repetition best-so-far and completion times
 * (SearchTrace.best_so_far / completion_times_us, search.py:294-304, with
 * profiled steps charged `overhead`), then for every step column k < max_len
 * the sums over repetitions of the padded best-so-far value and its square.
 * total_times_out / first_times_out (nullable) receive times[-1] / times[0]
 * of each repetition. */
int ct_aggregate_steps(ct_ctx* ctx, double overhead, int32_t max_len,
                       const double* col_sum_init, const double* col_sq_init,
                       double* col_sum_out, double* col_sq_out,
                       double* total_times_out, double* first_times_out);

/* ct_aggregate_time: the time-curve sums over the first time_reps repetitions
 * of the last launch: for every grid point g, best-so-far sampled at
 * searchsorted(times, grid[g], 'right') - 1 (clipped), summed with its
 * square.  Requires ct_aggregate_steps on the same launch. */
int ct_aggregate_time(ct_ctx* ctx, int32_t time_reps, const double* grid, int32_t n_grid,
                      const double* sum_init, const double* sq_init,
                      double* sum_out, double* sq_out);

/* ct_report: the whole report of the last launch (one experiment on one
 * device) in one call and ONE stream synchronisation: the per-repetition
 * n_steps / status / rep_error and the batch stats (as ct_fetch_results),
 * max_len = the longest trajectory, the step-curve column sums (as
 * ct_aggregate_steps; col_sum / col_sq hold max_steps of the launch, the
 * first max_len are written), total_times (R), and the time curve over the
 * first time_reps repetitions with its grid computed on the device as
 * harness.py:207-213 does it (np.linspace of 100 points, or the single
 * point t_start); grid / tc_sum / tc_sq hold 100, the first n_grid are
 * written.  Replaces harness.simulate's aggregation (harness.py:187-244). */
int ct_report(ct_ctx* ctx, double overhead, int32_t time_reps, int32_t* n_steps,
              int32_t* status, int32_t* rep_error, ct_batch_stats* stats, int32_t* max_len,
              double* col_sum, double* col_sq, double* total_times, int32_t* n_grid,
              double* grid, double* tc_sum, double* tc_sq);

#ifdef __cplusplus
}
#endif
#endif /* COUNTERTUNE_B200_H */
