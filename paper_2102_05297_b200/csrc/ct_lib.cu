// ct_lib.cu -- C ABI (include/countertune_b200.h) over the sm_100a kernels.
//
// Owns the device copies of the searcher's inputs (prediction table, replay
// data, space assignments), the result buffers of batched searches and the
// single-call kernels behind score_configurations / normalize_scores /
// weighted_select.  No C++ exception crosses the ABI; errors are negative
// status codes with a thread-local message.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "countertune_b200.h"
#include "ct_search.cuh"
#include "ct_tiled.cuh"
#include "ct_models.cuh"

using namespace ct;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CT_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess)                                                     \
            return fail(CT_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
    cudaError_t ensure(size_t n) {
        if (n <= cap && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr; cap = 0;
        size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = std::max<size_t>(n, 1);
        return e;
    }
    void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

}  // namespace

// Page-locked host staging for an upload: the caller's (pageable) arrays are
// copied into it on the host, the H2D copy then runs asynchronously on the
// context's stream and the next upload through the same stage first waits
// for the previous copy's event.  No stream synchronisation per upload.
struct PinnedStage {
    void* p = nullptr;
    size_t bytes = 0;
    cudaEvent_t done = nullptr;
    cudaError_t acquire(size_t want) {
        if (!done) {
            cudaError_t e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        cudaError_t e = cudaEventSynchronize(done);      // previous copy finished
        if (e != cudaSuccess) return e;
        if (want > bytes) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            bytes = 0;
            e = cudaHostAlloc(&p, want, cudaHostAllocDefault);
            if (e != cudaSuccess) return e;
            bytes = want;
        }
        return cudaSuccess;
    }
    void release() {
        if (done) { cudaEventSynchronize(done); cudaEventDestroy(done); done = nullptr; }
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
};

struct ct_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    // prediction table (column-major)
    DevBuf<double> table;
    int64_t n = 0;
    int64_t ld = 0;          // padded column stride
    int32_t n_counters = 0;
    // column flags on the device (the search kernel reads them): [0] columns
    // inside raw_term_cert's domain, [1] columns without an exact zero
    DevBuf<unsigned long long> col_flags;
    DevBuf<double> table_rm;        // row-major upload staging
    DevBuf<double> col_part;        // per-chunk column statistics
    // space assignments (row-major n x P)
    DevBuf<double> assign;
    int32_t n_params = 0;
    int64_t assign_n = 0;
    // replay data
    DevBuf<double> runtime;
    DevBuf<int64_t> threads;
    DevBuf<double> counters;
    DevBuf<uint8_t> has_record;
    DevBuf<uint32_t> stop_bits;
    int64_t replay_n = 0;
    bool has_stop = false;
    // results of the last batched launch
    DevBuf<int32_t> step_index;
    DevBuf<uint8_t> step_profiled;
    DevBuf<int32_t> n_steps, status, rep_error;
    DevBuf<unsigned long long> stats;
    int64_t res_reps = 0, res_max_steps = 0;
    bool res_valid = false;
    // scratch
    DevBuf<double> scratch_w;
    DevBuf<unsigned char> scratch_head;
    DevBuf<unsigned char> scratch_tiled;   // tiled path: state, row totals, bits, partials
    DevBuf<int32_t> tiled_live;            // tiled path: live repetitions (+ host mirror below)
    int32_t* tiled_live_host = nullptr;
    DevBuf<int32_t> scratch_perm;
    // single-call buffers
    DevBuf<double> vec_a, vec_b;
    DevBuf<uint8_t> mask_a, mask_b;
    DevBuf<unsigned long long> key_a, key_b;
    DevBuf<int32_t> val_a, val_b;
    DevBuf<unsigned char> cub_tmp;
    DevBuf<double> part_d;
    PinnedStage stage_table, stage_replay, stage_report;
    DevBuf<int32_t> part_i;
    DevBuf<u128> tiles;
    DevBuf<long long> pick;
    // on-device aggregation
    DevBuf<double> agg_bsf, agg_times, agg_vec, agg_sampled;
    // model inference
    DevBuf<unsigned char> model_blob;
    DevBuf<double> model_out;
    bool agg_valid = false;
    double agg_overhead = 1.0;
};

// ===========================================================================
// single-call kernels
// ===========================================================================
namespace {

struct ScoreSingleArgs {
    const double* table; int64_t ld; int64_t n;
    int64_t profile;
    int32_t n_delta;
    int32_t cols[CT_MAX_SCORE_KEYS];
    double vals[CT_MAX_SCORE_KEYS];
    const uint8_t* explored;
    const uint8_t* scoreable;  // nullable
    int32_t literal_sign;
    double* raw;
};

__global__ void k_score_single(const ScoreSingleArgs a) {
    __shared__ ActiveTerm act[CT_MAX_SCORE_KEYS];
    __shared__ int n_act;
    if (threadIdx.x == 0) {
        int na = 0;
        for (int k = 0; k < a.n_delta; ++k) {
            if (a.vals[k] == 0.0 || a.cols[k] < 0) continue;
            double pv = a.table[(size_t)a.cols[k] * a.ld + a.profile];
            if (pv == 0.0) continue;
            act[na].col = a.cols[k]; act[na].nz = 0; act[na].d = a.vals[k]; act[na].p = pv; ++na;
        }
        n_act = na;
    }
    __syncthreads();
    const bool lit = a.literal_sign != 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.n;
         e += (int64_t)gridDim.x * blockDim.x) {
        double raw = 0.0;
        if (!a.explored[e] && (!a.scoreable || a.scoreable[e])) {
            for (int k = 0; k < n_act; ++k)
                raw = add(raw, raw_term(__ldg(a.table + (size_t)act[k].col * a.ld + e), act[k], lit));
        }
        a.raw[e] = raw;
    }
}

// Euclidean parameter distance to the profile (search.py:134-136) as an
// order-preserving key; explored -> +inf (np_row_sum: ct_hd.cuh).
__global__ void k_topk_keys(const double* assign, int32_t P, int64_t n, int64_t profile,
                            const uint8_t* explored, unsigned long long* keys, int32_t* vals) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        double sq[64];
        int k = P < 64 ? P : 64;
        for (int j = 0; j < k; ++j) {
            double d = sub(assign[(size_t)e * P + j], assign[(size_t)profile * P + j]);
            sq[j] = mul(d, d);
        }
        double dist = dsqrt(np_row_sum(sq, k));
        if (explored[e]) dist = INFINITY;
        keys[e] = (unsigned long long)dbits(dist);   // dist >= 0: bit order == value order
        vals[e] = (int32_t)e;
    }
}

__global__ void k_topk_mark(const int32_t* sorted_vals, int64_t k, uint8_t* scoreable, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x)
        scoreable[sorted_vals[i]] = 1;
}

// normalize_scores: pool extrema (per-block partials)
__global__ void k_minmax(const double* raw, const uint8_t* pool, int64_t n,
                         double* pmax, double* pmin, int32_t* pcount) {
    double mx = -INFINITY, mn = INFINITY;
    int cnt = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (pool[e]) { mx = nmax(mx, raw[e]); mn = nmin(mn, raw[e]); ++cnt; }
    }
    __shared__ double smx[32], smn[32];
    __shared__ int scn[32];
    mx = warp_max(mx); mn = warp_min(mn); cnt = warp_sum_i(cnt);
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { smx[warp] = mx; smn[warp] = mn; scn[warp] = cnt; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            mx = nmax(mx, smx[i]); mn = nmin(mn, smn[i]); cnt += scn[i];
        }
        pmax[blockIdx.x] = mx; pmin[blockIdx.x] = mn; pcount[blockIdx.x] = cnt;
    }
}

__global__ void k_weights(const double* raw, const uint8_t* pool, int64_t n, const double* pmax,
                          const double* pmin, int nparts, double gamma, double* norm) {
    __shared__ double smax, smin;
    if (threadIdx.x == 0) {
        double mx = pmax[0], mn = pmin[0];
        for (int i = 1; i < nparts; ++i) { mx = nmax(mx, pmax[i]); mn = nmin(mn, pmin[i]); }
        smax = mx; smin = mn;
    }
    __syncthreads();
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x)
        norm[e] = pool[e] ? weight(raw[e], smax, smin, gamma) : 0.0;
}

// weighted_select: exact tile totals, then one warp locates + certifies.
__global__ void k_tile_totals(const double* w, int64_t n, int rows, int ntiles, u128* tiles,
                              int32_t* bad) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int64_t tile_len = 32LL * rows;
    for (int t = gw; t < ntiles; t += nw) {
        u128 s = 0;
        int b = 0;
        for (int j = 0; j < rows; ++j) {
            int64_t e = (int64_t)t * tile_len + 32LL * j + lane;
            if (e < n) { u128 f; if (to_fx(w[e], &f)) s += f; else b = 1; }
        }
        s = warp_sum(s);
        b = __any_sync(FULL, b);
        if (lane == 0) { tiles[t] = s; if (b) atomicExch(bad, 1); }
    }
}

__global__ void k_select_single(const double* w, int64_t n, int rows, int ntiles,
                                const u128* tiles, const int32_t* bad, double u, long long* out) {
    const int lane = threadIdx.x;
    if (*bad) {
        if (lane == 0) { out[0] = sequential_select(w, n, u); out[1] = 0; out[2] = 1; }
        return;
    }
    u128 total = 0;
    for (int t = lane; t < ntiles; t += 32) total += tiles[t];
    total = warp_sum(total);
    if (total == 0) { if (lane == 0) { out[0] = -1; out[1] = 0; out[2] = 0; } return; }
    double total_d = fx_to_double(total);
    double r = mul(u, total_d);
    u128 r_fx = floor_fx(r);
    Located pk = warp_locate(tiles, ntiles, w, n, rows, r_fx, lane);
    bool ok = certify(pk, r_fx, total_d, n);
    if (lane == 0) {
        out[0] = ok ? pk.idx : sequential_select(w, n, u);
        out[1] = ok ? 1 : 0;
        out[2] = 0;
    }
}

__global__ void k_analyze_react(const double* c, int gen, int64_t cores, int64_t threads,
                                double inst_reaction, double issue_sign, double* out) {
    // one warp, lane k = component k: the search kernel's own code path
    // (analyze_component_warp), so the expert-system parity tests pin it
    if (blockIdx.x != 0) return;
    const int lane = threadIdx.x & 31;
    const bool deg = degenerate_of(c);
    const double b = analyze_component_warp(c, lane < N_COMP ? lane : N_COMP - 1, gen, cores,
                                            threads, deg);
    if (lane < N_COMP) {
        out[lane] = b;
        out[N_COMP + lane] = react_component(b, lane, inst_reaction, issue_sign);
    }
    if (lane == 0) out[2 * N_COMP] = deg ? 1.0 : 0.0;
}

// Self-check of dvd_fast against __ddiv_rn on generated operand pairs:
// raw random bit patterns (all classes incl. zero/denormal/inf/nan), small
// integers (exact quotients), and Eq. 16-shaped operands d*(c-p) / (c+p).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__global__ void k_check_division(int64_t n, uint64_t seed, unsigned long long* bad,
                                 double* first) {
    unsigned long long local = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t h1 = mix64(seed ^ (uint64_t)i * 0x9e3779b97f4a7c15ull);
        uint64_t h2 = mix64(h1 + 0x632be59bd9b4e019ull);
        double a, b;
        switch ((int)(h1 & 3)) {
        case 0: a = bitsd(h1); b = bitsd(h2); break;
        case 1: a = (double)(int64_t)(h1 % 20001) - 10000.0; b = (double)(int64_t)(h2 % 2001) - 1000.0; break;
        case 2: {
            double c = (double)(h1 >> 11) * 0x1.0p-53 * 1e6, p = (double)(h2 >> 11) * 0x1.0p-53 * 1e6;
            double d = (double)((h1 ^ h2) >> 11) * 0x1.0p-52 - 1.0;
            a = mul(d, sub(c, p)); b = add(c, p); break; }
        default: {
            double c = (double)(h1 % 100000), p = (double)(h2 % 100000) + 1.0;
            double d = (double)((h1 ^ h2) >> 11) * 0x1.0p-52 - 1.0;
            a = mul(d, sub(c, p)); b = add(c, p); break; }
        }
        double x = dvd_fast(a, b), y = __ddiv_rn(a, b), z = dvd_term(a, b);
        bool same = (dbits(x) == dbits(y)) || (x != x && y != y);
        // dvd_term: equal value (a zero's sign is unspecified)
        same = same && ((dbits(z) == dbits(y)) || (z != z && y != y) || (z == 0.0 && y == 0.0));
        if (!same) {
            int cat = (int)(h1 & 3);
            if (atomicAdd(&bad[1 + cat], 1ull) == 0ull) {
                first[4 * cat + 0] = a; first[4 * cat + 1] = b;
                first[4 * cat + 2] = x; first[4 * cat + 3] = y;
            }
            ++local;
        }
    }
    if (local) atomicAdd(bad, local);
}

// ---- aggregation (harness.py:187-244) ---------------------------------
// One warp per repetition: best-so-far and cumulative completion times.
// The lanes gather a chunk of 32 steps at once (coalesced index reads, the
// runtime lookups in parallel); the completion-time sum and the running
// minimum then fold through the chunk in step order by shuffles, so the sums
// keep the reference's left-to-right order (harness.py:189-205).
__global__ void __launch_bounds__(256)
k_agg_rows(const int32_t* __restrict__ step_index, const uint8_t* __restrict__ step_profiled,
           const int32_t* __restrict__ n_steps, int32_t reps, int64_t width,
           const double* __restrict__ runtime, double overhead, double* __restrict__ bsf,
           double* __restrict__ times, double* __restrict__ total, double* __restrict__ first) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < reps; r += warps) {
        const int n = n_steps[r];
        double best = INFINITY, t = 0.0, t_first = 0.0;
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            const size_t o = (size_t)r * width + k;
            double rt = 0.0, cost = 0.0;
            if (k < n) {
                rt = runtime[step_index[o]];
                cost = mul(rt, step_profiled[o] ? overhead : 1.0);
            }
            const int cnt = min(32, n - k0);
            double my_t = 0.0, my_b = 0.0;
            for (int j = 0; j < cnt; ++j) {
                const double cj = __shfl_sync(0xffffffffu, cost, j);
                const double rj = __shfl_sync(0xffffffffu, rt, j);
                const bool head = (k0 + j == 0);
                t = head ? cj : add(t, cj);
                best = head ? rj : nmin(best, rj);
                if (head) t_first = t;
                if (lane == j) { my_t = t; my_b = best; }
            }
            if (k < n) {
                bsf[o] = my_b;
                times[o] = my_t;
            }
        }
        if (lane == 0) {
            total[r] = t;
            first[r] = t_first;
        }
    }
}

// Step-curve column sums over repetitions, in repetition order (numpy's
// axis-0 reduction adds row after row).  A block owns AGG_COLS columns: all
// its threads gather a chunk of AGG_CHUNK repetitions' (padded) values into
// shared memory in parallel, then one thread per column runs the sequential
// sum over the chunk; the L2 round trips overlap instead of forming the chain.
constexpr int AGG_COLS = 8, AGG_CHUNK = 256;
__global__ void __launch_bounds__(AGG_CHUNK)
k_agg_cols(const double* __restrict__ bsf, const int32_t* __restrict__ n_steps, int32_t reps,
           int64_t width, int32_t max_len, const double* __restrict__ sum0,
           const double* __restrict__ sq0, double* __restrict__ sum, double* __restrict__ sq,
           const int32_t* __restrict__ max_len_dev = nullptr) {
    __shared__ double tile[AGG_CHUNK][AGG_COLS + 1];
    if (max_len_dev) max_len = *max_len_dev;     // launched for the step capacity
    const int k0 = blockIdx.x * AGG_COLS;
    if (k0 >= max_len) return;
    const int tid = threadIdx.x;
    const int kc = k0 + tid;
    double s = 0.0, q = 0.0;
    if (tid < AGG_COLS && kc < max_len) {
        s = sum0 ? sum0[kc] : 0.0;
        q = sq0 ? sq0[kc] : 0.0;
    }
    for (int r0 = 0; r0 < reps; r0 += AGG_CHUNK) {
        const int cnt = min(AGG_CHUNK, reps - r0);
        if (tid < cnt) {
            const int r = r0 + tid;
            const int last = max(n_steps[r] - 1, 0);
            const double* row = bsf + (size_t)r * width;
#pragma unroll
            for (int c = 0; c < AGG_COLS; ++c) {
                const int k = k0 + c;
                tile[tid][c] = (k < max_len) ? row[k < last ? k : last] : 0.0;
            }
        }
        __syncthreads();
        if (tid < AGG_COLS) {
            for (int j = 0; j < cnt; ++j) {
                const double v = tile[j][tid];
                s = add(s, v);
                q = add(q, mul(v, v));
            }
        }
        __syncthreads();
    }
    if (tid < AGG_COLS && kc < max_len) {
        sum[kc] = s;
        sq[kc] = q;
    }
}

// The report's scalars computed on the device (harness.py:187-224): the
// longest trajectory, the time axis' ends over the first time_reps
// repetitions (max is exact in any order) and np.linspace's grid
// (numpy 2.x: y = arange(num) * step + start, step = (stop - start) / (num - 1),
// the last point = stop; a zero step goes through i / div * delta).
constexpr int AGG_GRID = 100;    // TIME_GRID_POINTS (harness.py:46)
struct AggMeta {
    int32_t max_len, n_grid;
    double t_start, t_end;
    double grid[AGG_GRID];
};

__global__ void __launch_bounds__(1024)
k_agg_meta(const int32_t* __restrict__ n_steps, const double* __restrict__ total,
           const double* __restrict__ first, int32_t reps, int32_t time_reps,
           AggMeta* __restrict__ meta) {
    int mx = 0;
    double ts = -INFINITY, te = -INFINITY;
    for (int r = threadIdx.x; r < reps; r += blockDim.x) {
        mx = max(mx, n_steps[r]);
        if (r < time_reps) { ts = fmax(ts, first[r]); te = fmax(te, total[r]); }
    }
    __shared__ int smx[32];
    __shared__ double sts[32], ste[32];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        ts = fmax(ts, __shfl_xor_sync(0xffffffffu, ts, d));
        te = fmax(te, __shfl_xor_sync(0xffffffffu, te, d));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { smx[w] = mx; sts[w] = ts; ste[w] = te; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
            mx = max(mx, smx[k]); ts = fmax(ts, sts[k]); te = fmax(te, ste[k]);
        }
        meta->max_len = mx;
        meta->t_start = ts;
        meta->t_end = te;
        if (te > ts) {
            meta->n_grid = AGG_GRID;
            const double delta = sub(te, ts), div = (double)(AGG_GRID - 1);
            const double step = delta / div;
            for (int i = 0; i < AGG_GRID; ++i) {
                const double y = (step == 0.0) ? mul((double)i / div, delta) : mul((double)i, step);
                meta->grid[i] = add(y, ts);
            }
            meta->grid[AGG_GRID - 1] = te;
        } else {
            meta->n_grid = 1;
            meta->grid[0] = ts;
        }
    }
}

// One thread per (grid point, repetition): sampled best-so-far.
__global__ void k_agg_sample(const double* bsf, const double* times, const int32_t* n_steps,
                             int32_t reps, int64_t width, const double* grid, int32_t n_grid,
                             double* sampled, const AggMeta* meta = nullptr) {
    if (meta) { grid = meta->grid; n_grid = meta->n_grid; }
    const int64_t total = (int64_t)reps * n_grid;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int g = (int)(i / reps), r = (int)(i % reps);
        const double x = grid[g];
        const double* t = times + (size_t)r * width;
        int lo = 0, hi = n_steps[r];          // first index with t[idx] > x
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (t[mid] > x) hi = mid; else lo = mid + 1;
        }
        int pos = lo - 1;
        pos = pos < 0 ? 0 : (pos > n_steps[r] - 1 ? n_steps[r] - 1 : pos);
        sampled[(size_t)g * reps + r] = bsf[(size_t)r * width + pos];
    }
}

__global__ void k_agg_time_sums(const double* __restrict__ sampled, int32_t reps, int32_t n_grid,
                                const double* __restrict__ sum0, const double* __restrict__ sq0,
                                double* __restrict__ sum, double* __restrict__ sq,
                                const AggMeta* __restrict__ meta = nullptr) {
    if (meta) n_grid = meta->n_grid;
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n_grid; g += gridDim.x * blockDim.x) {
        double s = sum0 ? sum0[g] : 0.0, q = sq0 ? sq0[g] : 0.0;
#pragma unroll 8
        for (int r = 0; r < reps; ++r) {
            const double v = sampled[(size_t)g * reps + r];
            s = add(s, v);
            q = add(q, mul(v, v));
        }
        sum[g] = s;
        sq[g] = q;
    }
}

// ---- prediction-table preparation on the device ----------------------
// Row-major n x c (the reference's PredictionTable.matrix) -> column-major
// with the stride padded to ld (zeros), through a shared-memory tile of 32
// rows: the reads are the rows' contiguous bytes, the writes 32 consecutive
// configurations of one column (256 B).
constexpr int TT_ROWS = 32, TT_MAXC = 64;
__global__ void __launch_bounds__(256)
k_table_transpose(const double* __restrict__ rm, int64_t n, int32_t c, double* __restrict__ cm,
                  int64_t ld) {
    __shared__ double tile[TT_ROWS * (TT_MAXC + 1)];
    const int per = TT_ROWS * c;
    for (int64_t t = blockIdx.x; t * TT_ROWS < ld; t += gridDim.x) {
        const int64_t r0 = t * TT_ROWS;
        for (int k = threadIdx.x; k < per; k += blockDim.x) {
            const int i = k / c, j = k - i * c;
            tile[i * (TT_MAXC + 1) + j] = (r0 + i < n) ? rm[(size_t)r0 * c + k] : 0.0;
        }
        __syncthreads();
        for (int k = threadIdx.x; k < per; k += blockDim.x) {
            const int j = k / TT_ROWS, i = k - j * TT_ROWS;
            cm[(size_t)j * ld + r0 + i] = tile[i * (TT_MAXC + 1) + j];
        }
        __syncthreads();
    }
}

// Column statistics of the column-major table for the search kernel's fast
// paths: block (g, j) reduces chunk g of column j to (min, max, smallest
// positive, non-finite seen, zero seen); k_col_flags folds the chunks and
// sets bit j of [certified, no-zero] (column_certified, ct_hd.cuh).  min /
// max are exact in any order.
struct ColPart { double vmin, vmax, vpos; int bad, zero; };

__global__ void __launch_bounds__(256)
k_col_stats(const double* __restrict__ cm, int64_t ld, int64_t n, int32_t chunks,
            ColPart* __restrict__ part) {
    const int j = blockIdx.y, g = blockIdx.x;
    const int64_t per = (n + chunks - 1) / chunks;
    const int64_t lo = g * per, hi = min(n, lo + per);
    double vmin = INFINITY, vmax = -INFINITY, vpos = INFINITY;
    int bad = 0, zero = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double v = cm[(size_t)j * ld + i];
        if (!(v == v) || isinf(v)) { bad = 1; continue; }
        vmin = fmin(vmin, v);
        vmax = fmax(vmax, v);
        if (v > 0.0) vpos = fmin(vpos, v);
        zero |= (v == 0.0);
    }
    __shared__ ColPart red[8];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, d));
        vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, d));
        vpos = fmin(vpos, __shfl_xor_sync(0xffffffffu, vpos, d));
        bad |= __shfl_xor_sync(0xffffffffu, bad, d);
        zero |= __shfl_xor_sync(0xffffffffu, zero, d);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = ColPart{vmin, vmax, vpos, bad, zero};
    __syncthreads();
    if (threadIdx.x == 0) {
        ColPart p = red[0];
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
            p.vmin = fmin(p.vmin, red[k].vmin); p.vmax = fmax(p.vmax, red[k].vmax);
            p.vpos = fmin(p.vpos, red[k].vpos); p.bad |= red[k].bad; p.zero |= red[k].zero;
        }
        part[(size_t)j * chunks + g] = p;
    }
}

__global__ void k_col_flags(const ColPart* __restrict__ part, int32_t chunks, int32_t c,
                            unsigned long long* __restrict__ flags) {
    __shared__ unsigned long long f[2];
    if (threadIdx.x == 0) { f[0] = 0ull; f[1] = 0ull; }
    __syncthreads();
    const int j = threadIdx.x;
    if (j < c && j < 64) {
        ColPart p = part[(size_t)j * chunks];
        for (int g = 1; g < chunks; ++g) {
            const ColPart q = part[(size_t)j * chunks + g];
            p.vmin = fmin(p.vmin, q.vmin); p.vmax = fmax(p.vmax, q.vmax);
            p.vpos = fmin(p.vpos, q.vpos); p.bad |= q.bad; p.zero |= q.zero;
        }
        const double vpos = (p.vpos == INFINITY) ? 0.0 : p.vpos;
        if (!p.bad && column_certified(p.vmin, vpos, p.vmax)) atomicOr(&f[0], 1ull << j);
        if (!p.zero) atomicOr(&f[1], 1ull << j);   // (a non-finite value is not a zero)
    }
    __syncthreads();
    if (threadIdx.x == 0) { flags[0] = f[0]; flags[1] = f[1]; }
}

int rows_for(int64_t n) {
    // ~sqrt(N)/32 rows balances the two scans of a draw; at least 2 rows so
    // that each lane sums two weights per tile before the warp reduction
    int rows = (int)std::lround(std::sqrt((double)n) / 32.0);
    return std::max(2, rows);
}

int grid_for(int64_t n, int threads, int sm_count) {
    int64_t g = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_count * 16));
}

int check_ctx(ct_ctx* ctx) {
    if (!ctx) return fail(CT_ERR_VALUE, "null context");
    CT_CUDA(cudaSetDevice(ctx->device));
    return CT_OK;
}

int pack_seeds(const ct_seed_spec* seeds, SeedInline* out) {
    if (!seeds) return fail(CT_ERR_VALUE, "null seed spec");
    if (seeds->n_entropy < 0 || seeds->n_prefix < 0 || (seeds->n_entropy && !seeds->entropy) ||
        (seeds->n_prefix && !seeds->spawn_prefix))
        return fail(CT_ERR_VALUE, "bad seed spec");
    if (seeds->n_entropy + seeds->n_prefix > SEED_INLINE_WORDS)
        return fail(CT_ERR_UNSUPPORTED, "seed entropy + spawn key exceed " +
                                            std::to_string(SEED_INLINE_WORDS) + " words");
    std::memset(out, 0, sizeof(*out));
    for (int i = 0; i < seeds->n_entropy; ++i) out->w[i] = seeds->entropy[i];
    for (int i = 0; i < seeds->n_prefix; ++i) out->w[seeds->n_entropy + i] = seeds->spawn_prefix[i];
    out->n_entropy = seeds->n_entropy;
    out->n_prefix = seeds->n_prefix;
    out->child_per_rep = seeds->child_per_rep;
    out->rep_offset = seeds->rep_offset;
    return CT_OK;
}

int ensure_results(ct_ctx* ctx, int64_t reps, int64_t max_steps) {
    CT_CUDA(ctx->step_index.ensure((size_t)reps * max_steps));
    CT_CUDA(ctx->step_profiled.ensure((size_t)reps * max_steps));
    CT_CUDA(ctx->n_steps.ensure(reps));
    CT_CUDA(ctx->status.ensure(reps));
    CT_CUDA(ctx->rep_error.ensure(reps));
    CT_CUDA(cudaMemsetAsync(ctx->stats.p, 0, 8 * sizeof(unsigned long long), ctx->stream));
    ctx->res_reps = reps;
    ctx->res_max_steps = max_steps;
    ctx->res_valid = true;
    ctx->agg_valid = false;
    return CT_OK;
}

template <int NT, bool SMEM, bool PRE, bool TOPK = false, bool HG = false>
int launch_profile_t(ct_ctx* ctx, SearchArgs& a, size_t smem, int n_reps) {
    auto kern = k_profile_search<NT, SMEM, PRE, TOPK, HG>;
    if (smem > 48 * 1024)
        CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem));
    if (occ < 1) return fail(CT_ERR_CUDA, "search kernel does not fit on an SM");
    int grid = std::min(n_reps, occ * ctx->sm_count);
    if (!SMEM) {
        CT_CUDA(ctx->scratch_w.ensure((size_t)grid * 64 * (size_t)a.nrows));
        a.scratch_w = ctx->scratch_w.p;
    }
    if (HG) {
        const size_t head = (16 * (size_t)a.nrows + 4 * (size_t)a.nwords + 15) & ~(size_t)15;
        CT_CUDA(ctx->scratch_head.ensure((size_t)grid * head));
        a.scratch_head = ctx->scratch_head.p;
    }
    kern<<<grid, NT, smem, ctx->stream>>>(a);
    CT_CUDA(cudaGetLastError());
    return CT_OK;
}

// warp-specialised kernel: two repetitions per CTA, PW parallel warps
template <int PW, bool SMEM>
int launch_profile_ws_t(ct_ctx* ctx, SearchArgs& a, size_t smem, int n_reps) {
    auto kern = k_profile_search_ws<PW, SMEM>;
    constexpr int NTT = 32 * (PW + 1);
    if (smem > 48 * 1024)
        CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NTT, smem));
    if (occ < 1) return fail(CT_ERR_CUDA, "search kernel does not fit on an SM");
    int grid = std::min((n_reps + 1) / 2, occ * ctx->sm_count);
    if (!SMEM) {
        CT_CUDA(ctx->scratch_w.ensure((size_t)2 * grid * 64 * (size_t)a.nrows));
        a.scratch_w = ctx->scratch_w.p;
    }
    kern<<<grid, NTT, smem, ctx->stream>>>(a);
    CT_CUDA(cudaGetLastError());
    return CT_OK;
}

// tiled path (ct_tiled.cuh): grid-wide phase kernels per outer iteration,
// the repetitions in batches that fit the scratch budget
__global__ void k_tiled_count_live(const TiledArgs t, int32_t* live) {
    int c = 0;
    for (int b = threadIdx.x; b < t.batch; b += blockDim.x) c += t.state[b].live;
    c = __reduce_add_sync(FULL, c);
    if ((threadIdx.x & 31) == 0) atomicAdd(live, c);
}

int launch_tiled(ct_ctx* ctx, SearchArgs& a, int n_reps) {
    const int64_t ntiles = (a.n + TILE_CONFIGS - 1) / TILE_CONFIGS;
    const int64_t w_stride = (int64_t)a.nrows * 32;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t per_rep = al(sizeof(TiledRep)) + al(8 * (size_t)a.nrows) + al(4 * (size_t)a.nwords) +
                           al(sizeof(double4) * (size_t)ntiles);
    const size_t per_rep_all = per_rep + 8 * (size_t)w_stride;
    size_t free_b = 0, total_b = 0;
    CT_CUDA(cudaMemGetInfo(&free_b, &total_b));
    size_t budget = std::min<size_t>(free_b / 2, (size_t)48 << 30);
    if (const char* env = std::getenv("CT_TILED_BUDGET_MB")) budget = (size_t)std::atoll(env) << 20;
    const int batch = (int)std::max<int64_t>(1, std::min<int64_t>(n_reps, (int64_t)(budget / per_rep_all)));
    CT_CUDA(ctx->scratch_w.ensure((size_t)batch * w_stride));
    CT_CUDA(ctx->scratch_tiled.ensure((size_t)batch * per_rep));
    CT_CUDA(ctx->tiled_live.ensure(1));
    if (!ctx->tiled_live_host) CT_CUDA(cudaMallocHost(&ctx->tiled_live_host, sizeof(int32_t)));
    unsigned char* base = ctx->scratch_tiled.p;
    TiledArgs t;
    t.state = reinterpret_cast<TiledRep*>(base);
    base += al(sizeof(TiledRep) * (size_t)batch);
    t.row_tot = reinterpret_cast<double*>(base);
    base += al(8 * (size_t)a.nrows * batch);
    t.expl = reinterpret_cast<uint32_t*>(base);
    base += al(4 * (size_t)a.nwords * batch);
    t.partial = reinterpret_cast<double4*>(base);
    t.w = ctx->scratch_w.p;
    t.w_stride = w_stride;
    t.ntiles = (int32_t)ntiles;
    for (int r0 = 0; r0 < n_reps; r0 += batch) {
        t.rep0 = r0;
        t.batch = std::min(batch, n_reps - r0);
        // defined bytes everywhere (the score kernel copies whole control blocks)
        CT_CUDA(cudaMemsetAsync(t.state, 0, sizeof(TiledRep) * (size_t)t.batch, ctx->stream));
        const int warps_grid = (t.batch + 3) / 4;
        const dim3 tiles((unsigned)t.batch, (unsigned)ntiles);
        k_tiled_begin<<<warps_grid, 128, 0, ctx->stream>>>(a, t);
        CT_CUDA(cudaGetLastError());
        for (int it = 0; it < a.outer; ++it) {
            k_tiled_score<<<tiles, TILED_NT, 0, ctx->stream>>>(a, t);
            k_tiled_reduce<<<warps_grid, 128, 0, ctx->stream>>>(a, t);
            k_tiled_weights<<<tiles, TILED_NT, 0, ctx->stream>>>(a, t);
            k_tiled_draw<<<warps_grid, 128, 0, ctx->stream>>>(a, t);
            CT_CUDA(cudaGetLastError());
            // stop launching once every repetition of the batch has ended
            // (searches run until a stop configuration / exhaustion)
            if ((it & 15) == 15 && it + 1 < a.outer) {
                CT_CUDA(cudaMemsetAsync(ctx->tiled_live.p, 0, sizeof(int32_t), ctx->stream));
                k_tiled_count_live<<<1, 256, 0, ctx->stream>>>(t, ctx->tiled_live.p);
                CT_CUDA(cudaMemcpyAsync(ctx->tiled_live_host, ctx->tiled_live.p, sizeof(int32_t),
                                        cudaMemcpyDeviceToHost, ctx->stream));
                CT_CUDA(cudaStreamSynchronize(ctx->stream));
                if (*ctx->tiled_live_host == 0) break;
            }
        }
    }
    return CT_OK;
}

// spaces in [TILED_MIN_N, TILED_MAX_N] take the tiled path by default
// (measured, profiles/r02/r02ah_large_space_sweep.jsonl): from ~10^5
// configurations the grid-wide phases beat one CTA per repetition
// (GEMM-full 205k R=444: 13.6 vs 18.9 ms; 1M: 79 vs 119 ms; 4M: 347 vs
// 497 ms); above 2^22 nothing was measured
constexpr int64_t TILED_MIN_N = 131072;
constexpr int64_t TILED_MAX_N = 1ll << 22;

template <int PW>
int launch_profile_ws(ct_ctx* ctx, SearchArgs& a, bool in_smem, size_t smem, int n_reps) {
    return in_smem ? launch_profile_ws_t<PW, true>(ctx, a, smem, n_reps)
                   : launch_profile_ws_t<PW, false>(ctx, a, smem, n_reps);
}

// PRE: in-row prefixes computed by all warps in the weight pass (default), or
// the drawn row scanned by the drawing warp (CT_SEARCH_PRE=0)
template <int NT>
int launch_profile(ct_ctx* ctx, SearchArgs& a, bool pre, bool in_smem, size_t smem, int n_reps) {
    if (a.topk >= 0) {   // top-K builds exist for 128-512 threads (the dispatcher ensures it)
        if constexpr (NT >= 128) {
            if (pre)
                return in_smem ? launch_profile_t<NT, true, true, true>(ctx, a, smem, n_reps)
                               : launch_profile_t<NT, false, true, true>(ctx, a, smem, n_reps);
            return in_smem ? launch_profile_t<NT, true, false, true>(ctx, a, smem, n_reps)
                           : launch_profile_t<NT, false, false, true>(ctx, a, smem, n_reps);
        } else {
            return fail(CT_ERR_UNSUPPORTED, "score_top_k needs >= 128 threads per repetition");
        }
    }
    if (pre)
        return in_smem ? launch_profile_t<NT, true, true>(ctx, a, smem, n_reps)
                       : launch_profile_t<NT, false, true>(ctx, a, smem, n_reps);
    return in_smem ? launch_profile_t<NT, true, false>(ctx, a, smem, n_reps)
                   : launch_profile_t<NT, false, false>(ctx, a, smem, n_reps);
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int ct_abi_version(void) { return CT_ABI_VERSION; }

const char* ct_last_error(void) { return g_err.c_str(); }

int ct_device_count(int* count) {
    if (!count) return fail(CT_ERR_VALUE, "null count");
    CT_CUDA(cudaGetDeviceCount(count));
    return CT_OK;
}

int ct_create(int device, ct_ctx** out) {
    if (!out) return fail(CT_ERR_VALUE, "null output");
    *out = nullptr;
    CT_CUDA(cudaSetDevice(device));
    ct_ctx* c = new ct_ctx();
    c->device = device;
    cudaError_t e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete c; return fail(CT_ERR_CUDA, cudaGetErrorString(e)); }
    c->stream = c->own;
    e = c->stats.ensure(8);
    if (e != cudaSuccess) { delete c; return fail(CT_ERR_CUDA, cudaGetErrorString(e)); }
    *out = c;
    return CT_OK;
}

int ct_destroy(ct_ctx* ctx) {
    if (!ctx) return CT_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->table.release(); ctx->assign.release(); ctx->runtime.release();
    ctx->threads.release(); ctx->counters.release(); ctx->has_record.release();
    ctx->stop_bits.release(); ctx->step_index.release(); ctx->step_profiled.release();
    ctx->n_steps.release(); ctx->status.release(); ctx->rep_error.release();
    ctx->stats.release(); ctx->scratch_w.release(); ctx->scratch_head.release();
    ctx->scratch_tiled.release(); ctx->tiled_live.release();
    if (ctx->tiled_live_host) { cudaFreeHost(ctx->tiled_live_host); ctx->tiled_live_host = nullptr; }
    ctx->col_flags.release(); ctx->table_rm.release(); ctx->col_part.release();
    ctx->scratch_perm.release(); ctx->vec_a.release();
    ctx->vec_b.release(); ctx->mask_a.release(); ctx->mask_b.release(); ctx->key_a.release();
    ctx->key_b.release(); ctx->val_a.release(); ctx->val_b.release(); ctx->cub_tmp.release();
    ctx->part_d.release(); ctx->part_i.release(); ctx->tiles.release(); ctx->pick.release();
    ctx->agg_bsf.release(); ctx->agg_times.release(); ctx->agg_vec.release();
    ctx->agg_sampled.release(); ctx->model_blob.release(); ctx->model_out.release();
    ctx->stage_table.release(); ctx->stage_replay.release(); ctx->stage_report.release();
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
    return CT_OK;
}

int ct_set_stream(ct_ctx* ctx, void* cuda_stream) {
    int rc = check_ctx(ctx); if (rc) return rc;
    CT_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->stream = cuda_stream ? (cudaStream_t)cuda_stream : ctx->own;
    return CT_OK;
}

int ct_synchronize(ct_ctx* ctx) {
    int rc = check_ctx(ctx); if (rc) return rc;
    CT_CUDA(cudaStreamSynchronize(ctx->stream));
    return CT_OK;
}

// the search kernel's column flags of the resident column-major table
static int table_flags(ct_ctx* ctx, int64_t n, int32_t c) {
    cudaStream_t s = ctx->stream;
    const int32_t chunks = (int32_t)std::max<int64_t>(1, std::min<int64_t>((n + 4095) / 4096, 64));
    CT_CUDA(ctx->col_part.ensure(sizeof(ColPart) / 8 * (size_t)chunks * c));
    CT_CUDA(ctx->col_flags.ensure(2));
    k_col_stats<<<dim3(chunks, c), 256, 0, s>>>(ctx->table.p, ctx->ld, n, chunks,
                                                reinterpret_cast<ColPart*>(ctx->col_part.p));
    CT_CUDA(cudaGetLastError());
    k_col_flags<<<1, 64, 0, s>>>(reinterpret_cast<const ColPart*>(ctx->col_part.p), chunks, c,
                                  ctx->col_flags.p);
    CT_CUDA(cudaGetLastError());
    return CT_OK;
}

int ct_table_upload(ct_ctx* ctx, const double* matrix, int64_t n, int32_t c) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!matrix || n < 1 || c < 1) return fail(CT_ERR_VALUE, "table needs n >= 1 and counters >= 1");
    if (n > INT32_MAX) return fail(CT_ERR_VALUE, "spaces above 2^31-1 configurations are not supported");
    if (c > TT_MAXC) return fail(CT_ERR_UNSUPPORTED, "tables of more than 64 counters are not supported");
    // the borrowed row-major matrix goes to the device as it is (one
    // contiguous copy through the pinned stage); the column-major layout with
    // its stride padded to a multiple of 2048 configurations (the search
    // kernel's unrolled loads never need a bounds test) and the column flags
    // are made there
    const int64_t ld = (n + 2047) / 2048 * 2048;
    const size_t bytes = sizeof(double) * (size_t)n * c;
    CT_CUDA(ctx->stage_table.acquire(bytes));
    std::memcpy(ctx->stage_table.p, matrix, bytes);
    CT_CUDA(ctx->table_rm.ensure((size_t)n * c));
    CT_CUDA(cudaMemcpyAsync(ctx->table_rm.p, ctx->stage_table.p, bytes, cudaMemcpyHostToDevice,
                            ctx->stream));
    CT_CUDA(cudaEventRecord(ctx->stage_table.done, ctx->stream));
    CT_CUDA(ctx->table.ensure((size_t)ld * c));
    k_table_transpose<<<(int)std::min<int64_t>(ld / TT_ROWS, (int64_t)ctx->sm_count * 8), 256, 0,
                        ctx->stream>>>(ctx->table_rm.p, n, c, ctx->table.p, ld);
    CT_CUDA(cudaGetLastError());
    ctx->n = n;
    ctx->ld = ld;
    ctx->n_counters = c;
    return table_flags(ctx, n, c);
}

int ct_model_predict(ct_ctx* ctx, const ct_model_program* pg, const double* assign, int64_t n,
                     int32_t p, double* out_rowmajor) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!pg || !assign || n < 1 || p < 1 || pg->n_cols < 1)
        return fail(CT_ERR_VALUE, "model inference needs a programme, n >= 1 and params >= 1");
    if (n > INT32_MAX) return fail(CT_ERR_VALUE, "spaces above 2^31-1 configurations are not supported");
    if (pg->n_binary < 0 || pg->n_binary > 63) return fail(CT_ERR_VALUE, "bad binary parameter count");
    for (int b = 0; b < pg->n_binary; ++b)
        if (pg->binary_pos[b] < 0 || pg->binary_pos[b] >= p) return fail(CT_ERR_VALUE, "binary position out of range");
    for (int i = 0; i < pg->n_nodes; ++i)
        if (pg->node_feature[i] >= p) return fail(CT_ERR_MISMATCH, "tree feature outside the parameter list");
    for (int i = 0; i < pg->n_terms; ++i)
        if (pg->term_p1[i] >= p || pg->term_p2[i] >= p) return fail(CT_ERR_MISMATCH, "regression term outside the parameter list");
    // one blob: [assignments | program arrays], 16-byte aligned pieces
    std::vector<std::pair<const void*, size_t>> parts = {
        {assign, sizeof(double) * (size_t)n * p},
        {pg->node_feature, 4 * (size_t)pg->n_nodes}, {pg->node_left, 4 * (size_t)pg->n_nodes},
        {pg->node_right, 4 * (size_t)pg->n_nodes}, {pg->node_threshold, 8 * (size_t)pg->n_nodes},
        {pg->node_value, 8 * (size_t)pg->n_nodes}, {pg->col_root, 4 * (size_t)pg->n_cols},
        {pg->col_model_first, 4 * (size_t)pg->n_cols}, {pg->col_model_count, 4 * (size_t)pg->n_cols},
        {pg->model_key, 8 * (size_t)pg->n_models}, {pg->model_term_first, 4 * (size_t)pg->n_models},
        {pg->model_term_count, 4 * (size_t)pg->n_models}, {pg->term_kind, 4 * (size_t)pg->n_terms},
        {pg->term_p1, 4 * (size_t)pg->n_terms}, {pg->term_p2, 4 * (size_t)pg->n_terms},
        {pg->term_coef, 8 * (size_t)pg->n_terms}, {pg->binary_pos, 4 * (size_t)pg->n_binary}};
    std::vector<size_t> off(parts.size());
    size_t total = 0;
    for (size_t k = 0; k < parts.size(); ++k) { off[k] = total; total += (parts[k].second + 15) & ~(size_t)15; }
    std::vector<unsigned char> blob(std::max<size_t>(total, 16), 0);
    for (size_t k = 0; k < parts.size(); ++k)
        if (parts[k].second) std::memcpy(blob.data() + off[k], parts[k].first, parts[k].second);
    cudaStream_t s = ctx->stream;
    CT_CUDA(ctx->model_blob.ensure(blob.size()));
    CT_CUDA(cudaMemcpyAsync(ctx->model_blob.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, s));
    unsigned char* d = ctx->model_blob.p;
    ModelProgramDev m;
    m.n_cols = pg->n_cols; m.n_params = p; m.n_binary = pg->n_binary;
    m.node_feature = (const int32_t*)(d + off[1]); m.node_left = (const int32_t*)(d + off[2]);
    m.node_right = (const int32_t*)(d + off[3]); m.node_threshold = (const double*)(d + off[4]);
    m.node_value = (const double*)(d + off[5]); m.col_root = (const int32_t*)(d + off[6]);
    m.col_model_first = (const int32_t*)(d + off[7]); m.col_model_count = (const int32_t*)(d + off[8]);
    m.model_key = (const uint64_t*)(d + off[9]); m.model_term_first = (const int32_t*)(d + off[10]);
    m.model_term_count = (const int32_t*)(d + off[11]); m.term_kind = (const int32_t*)(d + off[12]);
    m.term_p1 = (const int32_t*)(d + off[13]); m.term_p2 = (const int32_t*)(d + off[14]);
    m.term_coef = (const double*)(d + off[15]); m.binary_pos = (const int32_t*)(d + off[16]);
    const int64_t ld = (n + 2047) / 2048 * 2048;
    CT_CUDA(ctx->table.ensure((size_t)ld * pg->n_cols));
    CT_CUDA(cudaMemsetAsync(ctx->table.p, 0, sizeof(double) * (size_t)ld * pg->n_cols, s));
    CT_CUDA(ctx->model_out.ensure((size_t)n * pg->n_cols));
    const int64_t work = n * pg->n_cols;
    k_model_predict<<<(int)std::min<int64_t>((work + 255) / 256, (int64_t)ctx->sm_count * 16), 256, 0, s>>>(
        m, (const double*)(d + off[0]), n, ctx->model_out.p, ctx->table.p, ld);
    CT_CUDA(cudaGetLastError());
    std::vector<double> host;
    double* dst = out_rowmajor;
    if (!dst) { host.resize((size_t)n * pg->n_cols); dst = host.data(); }
    CT_CUDA(cudaMemcpyAsync(dst, ctx->model_out.p, sizeof(double) * (size_t)n * pg->n_cols,
                            cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    ctx->n = n;
    ctx->ld = ld;
    ctx->n_counters = pg->n_cols;
    return table_flags(ctx, n, pg->n_cols);
}

int ct_space_upload(ct_ctx* ctx, const double* assign, int64_t n, int32_t p) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!assign || n < 1 || p < 1) return fail(CT_ERR_VALUE, "space needs n >= 1 and params >= 1");
    if (p > 64) return fail(CT_ERR_UNSUPPORTED, "top-K distance supports at most 64 parameters");
    CT_CUDA(ctx->assign.ensure((size_t)n * p));
    CT_CUDA(cudaMemcpyAsync(ctx->assign.p, assign, sizeof(double) * n * p,
                            cudaMemcpyHostToDevice, ctx->stream));
    CT_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->assign_n = n;
    ctx->n_params = p;
    return CT_OK;
}

int ct_replay_upload(ct_ctx* ctx, int64_t n, const double* runtime, const int64_t* threads,
                     const double* counters, const uint8_t* has_record, const uint8_t* stop_mask) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (n < 1 || !runtime || !threads || !counters || !has_record)
        return fail(CT_ERR_VALUE, "replay upload needs runtime, threads, counters and has_record");
    CT_CUDA(ctx->runtime.ensure(n));
    CT_CUDA(ctx->threads.ensure(n));
    CT_CUDA(ctx->counters.ensure((size_t)n * CT_N_REQUIRED));
    CT_CUDA(ctx->has_record.ensure(n));
    cudaStream_t s = ctx->stream;
    // one pinned stage: runtime | threads | counters | has_record | stop bits
    const size_t words = (size_t)((n + 31) / 32);
    const size_t b_rt = sizeof(double) * n, b_th = sizeof(int64_t) * n;
    const size_t b_cn = sizeof(double) * n * CT_N_REQUIRED;
    const size_t b_hr = ((size_t)n + 7) & ~(size_t)7;
    CT_CUDA(ctx->stage_replay.acquire(b_rt + b_th + b_cn + b_hr + 4 * words));
    unsigned char* st = static_cast<unsigned char*>(ctx->stage_replay.p);
    std::memcpy(st, runtime, b_rt);
    std::memcpy(st + b_rt, threads, b_th);
    std::memcpy(st + b_rt + b_th, counters, b_cn);
    std::memcpy(st + b_rt + b_th + b_cn, has_record, (size_t)n);
    CT_CUDA(cudaMemcpyAsync(ctx->runtime.p, st, b_rt, cudaMemcpyHostToDevice, s));
    CT_CUDA(cudaMemcpyAsync(ctx->threads.p, st + b_rt, b_th, cudaMemcpyHostToDevice, s));
    CT_CUDA(cudaMemcpyAsync(ctx->counters.p, st + b_rt + b_th, b_cn, cudaMemcpyHostToDevice, s));
    CT_CUDA(cudaMemcpyAsync(ctx->has_record.p, st + b_rt + b_th + b_cn, (size_t)n,
                            cudaMemcpyHostToDevice, s));
    ctx->has_stop = stop_mask != nullptr;
    if (stop_mask) {
        uint32_t* bits = reinterpret_cast<uint32_t*>(st + b_rt + b_th + b_cn + b_hr);
        std::memset(bits, 0, 4 * words);
        for (int64_t i = 0; i < n; ++i)
            if (stop_mask[i]) bits[i >> 5] |= 1u << (i & 31);
        CT_CUDA(ctx->stop_bits.ensure(words));
        CT_CUDA(cudaMemcpyAsync(ctx->stop_bits.p, bits, words * 4, cudaMemcpyHostToDevice, s));
    }
    CT_CUDA(cudaEventRecord(ctx->stage_replay.done, s));
    ctx->replay_n = n;
    return CT_OK;
}

int ct_score(ct_ctx* ctx, int64_t profile, const int32_t* cols, const double* vals, int32_t n_delta,
             const uint8_t* explored, int32_t literal_sign, int64_t top_k, double* raw_out,
             uint8_t* scoreable_out, int32_t* has_scoreable) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!ctx->table.p) return fail(CT_ERR_STATE, "no prediction table uploaded");
    if (n_delta < 0 || n_delta > CT_MAX_SCORE_KEYS || (n_delta && (!cols || !vals)))
        return fail(CT_ERR_VALUE, "delta must hold at most 32 scored keys");
    if (!explored || !raw_out) return fail(CT_ERR_VALUE, "null explored/raw buffer");
    const int64_t n = ctx->n;
    if (profile < 0 || profile >= n) return fail(CT_ERR_VALUE, "profile index out of range");
    for (int k = 0; k < n_delta; ++k)
        if (cols[k] >= ctx->n_counters) return fail(CT_ERR_VALUE, "delta column out of range");
    cudaStream_t s = ctx->stream;
    CT_CUDA(ctx->mask_a.ensure(n));
    CT_CUDA(ctx->vec_a.ensure(n));
    CT_CUDA(cudaMemcpyAsync(ctx->mask_a.p, explored, n, cudaMemcpyHostToDevice, s));
    int64_t pool = 0;
    for (int64_t i = 0; i < n; ++i) pool += explored[i] ? 0 : 1;
    bool topk = top_k >= 0 && top_k < pool;
    if (has_scoreable) *has_scoreable = topk ? 1 : 0;
    if (topk) {
        if (!ctx->assign.p || ctx->assign_n != n)
            return fail(CT_ERR_STATE, "score_top_k needs the space assignments (ct_space_upload)");
        CT_CUDA(ctx->key_a.ensure(n)); CT_CUDA(ctx->key_b.ensure(n));
        CT_CUDA(ctx->val_a.ensure(n)); CT_CUDA(ctx->val_b.ensure(n));
        CT_CUDA(ctx->mask_b.ensure(n));
        k_topk_keys<<<grid_for(n, 256, ctx->sm_count), 256, 0, s>>>(ctx->assign.p, ctx->n_params, n, profile,
                                                      ctx->mask_a.p, ctx->key_a.p, ctx->val_a.p);
        size_t tmp = 0;
        CT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, ctx->key_a.p, ctx->key_b.p,
                                                ctx->val_a.p, ctx->val_b.p, (int)n, 0, 64, s));
        CT_CUDA(ctx->cub_tmp.ensure(tmp));
        CT_CUDA(cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.p, tmp, ctx->key_a.p, ctx->key_b.p,
                                                ctx->val_a.p, ctx->val_b.p, (int)n, 0, 64, s));
        CT_CUDA(cudaMemsetAsync(ctx->mask_b.p, 0, n, s));
        if (top_k > 0)
            k_topk_mark<<<grid_for(top_k, 256, ctx->sm_count), 256, 0, s>>>(ctx->val_b.p, top_k, ctx->mask_b.p, n);
    }
    ScoreSingleArgs a;
    std::memset(&a, 0, sizeof(a));
    a.table = ctx->table.p; a.ld = ctx->ld; a.n = n; a.profile = profile; a.n_delta = n_delta;
    for (int k = 0; k < n_delta; ++k) { a.cols[k] = cols[k]; a.vals[k] = vals[k]; }
    a.explored = ctx->mask_a.p; a.scoreable = topk ? ctx->mask_b.p : nullptr;
    a.literal_sign = literal_sign; a.raw = ctx->vec_a.p;
    k_score_single<<<grid_for(n, 256, ctx->sm_count), 256, 0, s>>>(a);
    CT_CUDA(cudaGetLastError());
    CT_CUDA(cudaMemcpyAsync(raw_out, ctx->vec_a.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    if (topk && scoreable_out)
        CT_CUDA(cudaMemcpyAsync(scoreable_out, ctx->mask_b.p, n, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    return CT_OK;
}

int ct_normalize(ct_ctx* ctx, const double* raw, const uint8_t* pool, int64_t n, double gamma,
                 double* norm_out) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!raw || !pool || !norm_out || n < 0) return fail(CT_ERR_VALUE, "null buffers");
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) cnt += pool[i] ? 1 : 0;
    if (cnt == 0) return fail(CT_ERR_EXHAUSTED, "no unexplored configurations to normalize");
    cudaStream_t s = ctx->stream;
    CT_CUDA(ctx->vec_a.ensure(n)); CT_CUDA(ctx->vec_b.ensure(n)); CT_CUDA(ctx->mask_a.ensure(n));
    int g = std::min(grid_for(n, 256, ctx->sm_count), 512);
    CT_CUDA(ctx->part_d.ensure(2 * (size_t)g)); CT_CUDA(ctx->part_i.ensure(g));
    CT_CUDA(cudaMemcpyAsync(ctx->vec_a.p, raw, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    CT_CUDA(cudaMemcpyAsync(ctx->mask_a.p, pool, n, cudaMemcpyHostToDevice, s));
    k_minmax<<<g, 256, 0, s>>>(ctx->vec_a.p, ctx->mask_a.p, n, ctx->part_d.p, ctx->part_d.p + g,
                               ctx->part_i.p);
    k_weights<<<grid_for(n, 256, ctx->sm_count), 256, 0, s>>>(ctx->vec_a.p, ctx->mask_a.p, n, ctx->part_d.p,
                                               ctx->part_d.p + g, g, gamma, ctx->vec_b.p);
    CT_CUDA(cudaGetLastError());
    CT_CUDA(cudaMemcpyAsync(norm_out, ctx->vec_b.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    return CT_OK;
}

int ct_select(ct_ctx* ctx, const double* norm, int64_t n, double u, int64_t* chosen,
              int32_t* certified) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!norm || !chosen || n < 1) return fail(CT_ERR_EXHAUSTED, "every configuration is explored");
    cudaStream_t s = ctx->stream;
    int rows = rows_for(n);
    int ntiles = (int)((n + 32LL * rows - 1) / (32LL * rows));
    CT_CUDA(ctx->vec_a.ensure(n)); CT_CUDA(ctx->tiles.ensure(ntiles));
    CT_CUDA(ctx->part_i.ensure(1)); CT_CUDA(ctx->pick.ensure(3));
    CT_CUDA(cudaMemcpyAsync(ctx->vec_a.p, norm, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    CT_CUDA(cudaMemsetAsync(ctx->part_i.p, 0, sizeof(int32_t), s));
    int blocks = std::max(1, std::min((ntiles + 7) / 8, 1024));
    k_tile_totals<<<blocks, 256, 0, s>>>(ctx->vec_a.p, n, rows, ntiles, ctx->tiles.p, ctx->part_i.p);
    k_select_single<<<1, 32, 0, s>>>(ctx->vec_a.p, n, rows, ntiles, ctx->tiles.p, ctx->part_i.p, u,
                                     ctx->pick.p);
    CT_CUDA(cudaGetLastError());
    long long out[3];
    CT_CUDA(cudaMemcpyAsync(out, ctx->pick.p, sizeof(out), cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    if (out[0] < 0) return fail(CT_ERR_EXHAUSTED, "every configuration is explored");
    *chosen = out[0];
    if (certified) *certified = (int32_t)out[1];
    return CT_OK;
}

int ct_analyze_react(ct_ctx* ctx, const double* counters23, int32_t generation, int64_t cores,
                     int64_t global_threads, double inst_reaction, double issue_sign,
                     double* out37) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!counters23 || !out37) return fail(CT_ERR_VALUE, "null buffers");
    if (!(inst_reaction > 0.0 && inst_reaction < 1.0))
        return fail(CT_ERR_VALUE, "inst_reaction must lie in (0, 1), got " + std::to_string(inst_reaction));
    cudaStream_t s = ctx->stream;
    CT_CUDA(ctx->vec_a.ensure(CT_N_REQUIRED + 2 * CT_N_DELTA + 1));
    double* dc = ctx->vec_a.p;
    double* dout = ctx->vec_a.p + CT_N_REQUIRED;
    CT_CUDA(cudaMemcpyAsync(dc, counters23, sizeof(double) * CT_N_REQUIRED, cudaMemcpyHostToDevice, s));
    k_analyze_react<<<1, 32, 0, s>>>(dc, generation, cores, global_threads, inst_reaction,
                                     issue_sign, dout);
    CT_CUDA(cudaGetLastError());
    CT_CUDA(cudaMemcpyAsync(out37, dout, sizeof(double) * (2 * CT_N_DELTA + 1), cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    return CT_OK;
}

int ct_check_division(ct_ctx* ctx, int64_t n, uint64_t seed, int64_t* mismatches,
                      double* first_bad) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!mismatches || n < 0) return fail(CT_ERR_VALUE, "bad arguments");
    cudaStream_t s = ctx->stream;
    CT_CUDA(ctx->pick.ensure(5));
    CT_CUDA(ctx->part_d.ensure(16));
    CT_CUDA(cudaMemsetAsync(ctx->pick.p, 0, 5 * sizeof(long long), s));
    CT_CUDA(cudaMemsetAsync(ctx->part_d.p, 0, 16 * sizeof(double), s));
    k_check_division<<<ctx->sm_count * 8, 256, 0, s>>>(n, seed, (unsigned long long*)ctx->pick.p,
                                                        ctx->part_d.p);
    CT_CUDA(cudaGetLastError());
    long long out[5] = {0, 0, 0, 0, 0};
    CT_CUDA(cudaMemcpyAsync(out, ctx->pick.p, sizeof(out), cudaMemcpyDeviceToHost, s));
    if (first_bad)
        CT_CUDA(cudaMemcpyAsync(first_bad, ctx->part_d.p, 16 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    *mismatches = out[0];
    return CT_OK;
}

// ------------------------------------------------------------ batched searches

int ct_profile_search_launch(ct_ctx* ctx, const ct_search_params* prm, const ct_seed_spec* seeds,
                             int32_t n_reps) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!prm) return fail(CT_ERR_VALUE, "null params");
    if (!ctx->table.p) return fail(CT_ERR_STATE, "no prediction table uploaded");
    if (!ctx->runtime.p || ctx->replay_n != ctx->n)
        return fail(CT_ERR_MISMATCH, "prediction table was built for a different space");
    if (prm->outer_iterations < 1)
        return fail(CT_ERR_VALUE, "need at least one outer iteration, got i=" +
                                      std::to_string(prm->outer_iterations));
    if (prm->inner_steps < 0)
        return fail(CT_ERR_VALUE, "inner step count must be >= 0, got n=" +
                                      std::to_string(prm->inner_steps));
    if (!(prm->inst_reaction > 0.0 && prm->inst_reaction < 1.0))
        return fail(CT_ERR_VALUE, "inst_reaction must lie in (0, 1)");
    if (prm->score_top_k >= 0 && (!ctx->assign.p || ctx->assign_n != ctx->n))
        return fail(CT_ERR_STATE, "score_top_k needs the space assignments (ct_space_upload)");
    if (prm->use_stop && !ctx->has_stop) return fail(CT_ERR_STATE, "no stop mask uploaded");
    if (n_reps < 0) return fail(CT_ERR_VALUE, "n_reps must be >= 0");
    for (int k = 0; k < CT_N_DELTA; ++k)
        if (prm->delta_columns[k] >= ctx->n_counters) return fail(CT_ERR_VALUE, "delta column out of range");
    SeedInline seed_inline;
    rc = pack_seeds(seeds, &seed_inline); if (rc) return rc;
    const int64_t n = ctx->n;
    const int64_t max_steps = (int64_t)prm->outer_iterations * (prm->inner_steps + 1);
    rc = ensure_results(ctx, std::max(n_reps, 1), max_steps); if (rc) return rc;
    ctx->res_reps = n_reps;
    if (n_reps == 0) return CT_OK;

    SearchArgs a;
    std::memset(&a, 0, sizeof(a));
    a.table = ctx->table.p; a.ld = ctx->ld; a.n = n;
    a.runtime = ctx->runtime.p; a.threads = ctx->threads.p; a.counters = ctx->counters.p;
    a.has_record = ctx->has_record.p; a.stop_bits = prm->use_stop ? ctx->stop_bits.p : nullptr;
    a.outer = prm->outer_iterations; a.inner = prm->inner_steps;
    a.inst_reaction = prm->inst_reaction; a.issue_sign = prm->issue_delta_sign; a.gamma = prm->gamma;
    a.literal_sign = prm->literal_sign; a.generation = prm->generation; a.cores = prm->cores;
    for (int k = 0; k < CT_N_DELTA; ++k) a.delta_col[k] = prm->delta_columns[k];
    a.col_flags = ctx->col_flags.p;
    a.seed = seed_inline; a.n_reps = n_reps;
    a.nrows = (int32_t)((n + 31) / 32);
    a.nwords = (n + 31) / 32;
    if (const char* env = std::getenv("CT_SEARCH_FORCE_SEQUENTIAL")) a.force_sequential = std::atoi(env);
    a.cert_slack = 1.0;
    if (const char* env = std::getenv("CT_SEARCH_CERT_SLACK")) a.cert_slack = std::max(1.0, std::atof(env));
    a.topk = prm->score_top_k >= 0 ? prm->score_top_k : -1;
    a.assign = a.topk >= 0 ? ctx->assign.p : nullptr;
    a.n_params = a.topk >= 0 ? ctx->n_params : 0;
    a.step_index = ctx->step_index.p; a.step_profiled = ctx->step_profiled.p;
    a.max_steps = max_steps; a.n_steps = ctx->n_steps.p; a.status = ctx->status.p;
    a.rep_error = ctx->rep_error.p; a.stats = ctx->stats.p;

    // threads per repetition: the serial phases (expert system, draws) run on
    // one warp, so small spaces use small CTAs (many repetitions per SM, no
    // idle warps at the CTA barrier); CT_SEARCH_NT overrides (benchmarking)
    int nt = n <= 8192 ? 128 : (n <= 65536 ? 256 : 512);
    if (const char* env = std::getenv("CT_SEARCH_NT")) nt = std::atoi(env);
    if (a.topk >= 0 && nt < 128) nt = 128;
    // row totals + explored bits always in shared memory; the weights too
    // when that still lets all repetitions be resident at once (one wave),
    // otherwise a per-CTA slice of global scratch (L2-resident)
    const size_t budget = 200 * 1024;
    // (+ the top-K exclusion bits and radix-select scratch when top-K is on)
    const size_t head_b = ((16 * (size_t)a.nrows + 4 * (size_t)a.nwords + 15) & ~(size_t)15)
                          + (a.topk >= 0 ? topk_bytes(a.nwords) : 0);
    // in-row prefixes stored by the weight pass (PRE) only pay off when the
    // rows are few (the drawing warp then rescans nothing); otherwise the
    // weight pass keeps just the row totals and the draw scans the drawn row
    bool pre = a.nrows < 32;
    if (const char* env = std::getenv("CT_SEARCH_PRE")) pre = std::atoi(env) != 0;
    const size_t pref_b = (pre ? 16 : 8) * 32 * (size_t)a.nrows;   // weights [+ in-row prefixes]
    // large spaces: grid-wide phase kernels (ct_tiled.cuh); CT_SEARCH_TILED
    // forces (1) or disables (0) the path
    int tiled = (n >= TILED_MIN_N && n <= TILED_MAX_N && a.topk < 0) ? 1 : 0;
    if (const char* env = std::getenv("CT_SEARCH_TILED")) tiled = std::atoi(env) != 0 && a.topk < 0;
    if (tiled) return launch_tiled(ctx, a, n_reps);
    if (head_b > budget) {
        // the row index (row totals + explored bits) outgrows shared memory:
        // all per-repetition state in a per-CTA slice of global scratch
        if (a.topk >= 0)
            return fail(CT_ERR_UNSUPPORTED, "score_top_k on spaces above ~300k configurations");
        return launch_profile_t<512, false, false, false, true>(ctx, a, 0, n_reps);
    }
    const int64_t want_per_sm = std::min<int64_t>(std::min<int64_t>(
        (n_reps + ctx->sm_count - 1) / ctx->sm_count, 32), 2048 / nt);
    const size_t per_cta_cap = std::min<size_t>(
        budget, (size_t)(228 * 1024 / std::max<int64_t>(want_per_sm, 1)) - 3 * 1024);
    bool in_smem = head_b + pref_b <= per_cta_cap;
    if (const char* env = std::getenv("CT_SEARCH_SMEM")) in_smem = std::atoi(env) != 0 && head_b + pref_b <= budget;
    const size_t smem = head_b + (in_smem ? pref_b : 0);
    // warp-specialised two-repetition kernel (CT_SEARCH_WS = parallel warps)
    int ws = 0;
    if (const char* env = std::getenv("CT_SEARCH_WS")) ws = std::atoi(env);
    if (ws > 0 && 2 * head_b <= budget && a.topk < 0) {   // the WS kernel has no top-K phase
        // two slots per CTA: weights in shared memory when both fit
        const int64_t ctas_per_sm = std::max<int64_t>(1, (want_per_sm + 1) / 2);
        const size_t cap2 = std::min<size_t>(
            2 * budget, (size_t)(228 * 1024 / ctas_per_sm) - 3 * 1024);
        const size_t pref_ws = 16 * 32 * (size_t)a.nrows;   // this kernel always stores prefixes
        bool ws_smem = 2 * (head_b + pref_ws) <= cap2;
        if (const char* env = std::getenv("CT_SEARCH_SMEM")) ws_smem = std::atoi(env) != 0 && 2 * (head_b + pref_ws) <= 2 * budget;
        const size_t smem2 = 2 * (head_b + (ws_smem ? pref_ws : 0));
        switch (ws) {
        case 2: return launch_profile_ws<2>(ctx, a, ws_smem, smem2, n_reps);
        case 3: return launch_profile_ws<3>(ctx, a, ws_smem, smem2, n_reps);
        case 4: return launch_profile_ws<4>(ctx, a, ws_smem, smem2, n_reps);
        case 6: return launch_profile_ws<6>(ctx, a, ws_smem, smem2, n_reps);
        default: return launch_profile_ws<8>(ctx, a, ws_smem, smem2, n_reps);
        }
    }
    switch (nt) {
    case 32: return launch_profile<32>(ctx, a, pre, in_smem, smem, n_reps);
    case 64: return launch_profile<64>(ctx, a, pre, in_smem, smem, n_reps);
    case 128: return launch_profile<128>(ctx, a, pre, in_smem, smem, n_reps);
    case 256: return launch_profile<256>(ctx, a, pre, in_smem, smem, n_reps);
    default: return launch_profile<512>(ctx, a, pre, in_smem, smem, n_reps);
    }
}

int ct_random_search_launch(ct_ctx* ctx, const ct_seed_spec* seeds, int32_t n_reps,
                            int64_t max_steps_req, int32_t use_stop) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!ctx->runtime.p) return fail(CT_ERR_STATE, "no replay data uploaded");
    if (use_stop && !ctx->has_stop) return fail(CT_ERR_STATE, "no stop mask uploaded");
    if (n_reps < 0) return fail(CT_ERR_VALUE, "n_reps must be >= 0");
    SeedInline seed_inline;
    rc = pack_seeds(seeds, &seed_inline); if (rc) return rc;
    const int64_t n = ctx->replay_n;
    int64_t max_steps = n;
    if (max_steps_req >= 0 && max_steps_req < n) max_steps = max_steps_req;
    rc = ensure_results(ctx, std::max(n_reps, 1), std::max<int64_t>(max_steps, 1)); if (rc) return rc;
    ctx->res_reps = n_reps;
    if (n_reps == 0) return CT_OK;
    const int threads = 64;
    int slots = std::min<int64_t>(n_reps, std::max<int64_t>(ctx->sm_count * 2 * threads,
                                                            threads));
    int blocks = (slots + threads - 1) / threads;
    slots = blocks * threads;
    CT_CUDA(ctx->scratch_perm.ensure((size_t)slots * n));
    RandomArgs a;
    std::memset(&a, 0, sizeof(a));
    a.n = n; a.has_record = ctx->has_record.p; a.stop_bits = use_stop ? ctx->stop_bits.p : nullptr;
    a.max_steps_req = max_steps_req;
    a.seed = seed_inline; a.n_reps = n_reps;
    a.perm_scratch = ctx->scratch_perm.p; a.n_slots = slots;
    a.step_index = ctx->step_index.p; a.step_profiled = ctx->step_profiled.p;
    a.max_steps = ctx->res_max_steps; a.n_steps = ctx->n_steps.p; a.status = ctx->status.p;
    a.rep_error = ctx->rep_error.p;
    k_random_search<<<blocks, threads, 0, ctx->stream>>>(a);
    CT_CUDA(cudaGetLastError());
    return CT_OK;
}

int ct_result_max_steps(ct_ctx* ctx, int64_t* max_steps) {
    if (!ctx || !max_steps) return fail(CT_ERR_VALUE, "null argument");
    if (!ctx->res_valid) return fail(CT_ERR_STATE, "no batched search launched");
    *max_steps = ctx->res_max_steps;
    return CT_OK;
}

// Zero the trajectory slots a launch did not write (past a repetition's
// steps; an error repetition keeps the slot after them, its failing index),
// so that a fetch copies defined bytes only.
__global__ void k_clear_tails(int32_t* __restrict__ step_index, uint8_t* __restrict__ step_profiled,
                              const int32_t* __restrict__ n_steps, const int32_t* __restrict__ status,
                              int32_t reps, int64_t width) {
    const int64_t total = (int64_t)reps * width;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / width);
        const int64_t k = i % width;
        const int64_t keep = n_steps[r] + (status[r] == CT_STATUS_ERROR ? 1 : 0);
        if (k >= keep) {
            step_index[i] = 0;
            step_profiled[i] = 0;
        }
    }
}

int ct_fetch_results(ct_ctx* ctx, int32_t* step_index, uint8_t* step_profiled, int32_t* n_steps,
                     int32_t* status, int32_t* rep_error, ct_batch_stats* stats) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!ctx->res_valid) return fail(CT_ERR_STATE, "no batched search launched");
    cudaStream_t s = ctx->stream;
    size_t r = (size_t)ctx->res_reps, m = (size_t)ctx->res_max_steps;
    if (r) {
        if ((step_index || step_profiled) && m) {
            const int64_t total = (int64_t)(r * m);
            k_clear_tails<<<(int)std::min<int64_t>((total + 255) / 256, 4 * (int64_t)ctx->sm_count), 256, 0, s>>>(
                ctx->step_index.p, ctx->step_profiled.p, ctx->n_steps.p, ctx->status.p,
                (int32_t)r, (int64_t)m);
            CT_CUDA(cudaGetLastError());
        }
        if (step_index)
            CT_CUDA(cudaMemcpyAsync(step_index, ctx->step_index.p, 4 * r * m, cudaMemcpyDeviceToHost, s));
        if (step_profiled)
            CT_CUDA(cudaMemcpyAsync(step_profiled, ctx->step_profiled.p, r * m, cudaMemcpyDeviceToHost, s));
        if (n_steps) CT_CUDA(cudaMemcpyAsync(n_steps, ctx->n_steps.p, 4 * r, cudaMemcpyDeviceToHost, s));
        if (status) CT_CUDA(cudaMemcpyAsync(status, ctx->status.p, 4 * r, cudaMemcpyDeviceToHost, s));
        if (rep_error) CT_CUDA(cudaMemcpyAsync(rep_error, ctx->rep_error.p, 4 * r, cudaMemcpyDeviceToHost, s));
    }
    unsigned long long st[5] = {0, 0, 0, 0, 0};
    CT_CUDA(cudaMemcpyAsync(st, ctx->stats.p, sizeof(st), cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    if (stats) {
        stats->configs_scored = (int64_t)st[0];
        stats->draws = (int64_t)st[1];
        stats->uncertified = (int64_t)st[2];
        stats->outer_iterations = (int64_t)st[3];
        stats->algorithmic_bytes = (int64_t)st[4];
    }
    return CT_OK;
}

int ct_aggregate_steps(ct_ctx* ctx, double overhead, int32_t max_len, const double* sum0,
                       const double* sq0, double* sum_out, double* sq_out, double* total_out,
                       double* first_out) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!ctx->res_valid) return fail(CT_ERR_STATE, "no batched search launched");
    if (!ctx->runtime.p) return fail(CT_ERR_STATE, "no replay data uploaded");
    if (max_len < 0 || (max_len > 0 && (!sum_out || !sq_out)))
        return fail(CT_ERR_VALUE, "bad aggregation buffers");
    const int64_t R = ctx->res_reps, W = ctx->res_max_steps;
    if (max_len > W) return fail(CT_ERR_VALUE, "max_len exceeds the launch's step capacity");
    cudaStream_t s = ctx->stream;
    CT_CUDA(ctx->agg_bsf.ensure((size_t)std::max<int64_t>(R, 1) * W));
    CT_CUDA(ctx->agg_times.ensure((size_t)std::max<int64_t>(R, 1) * W));
    const size_t nv = 2 * (size_t)R + 4 * (size_t)max_len;
    CT_CUDA(ctx->agg_vec.ensure(nv));
    double* d_total = ctx->agg_vec.p;
    double* d_first = d_total + R;
    double* d_sum0 = d_first + R;
    double* d_sq0 = d_sum0 + max_len;
    double* d_sum = d_sq0 + max_len;
    double* d_sq = d_sum + max_len;
    if (R > 0) {
        k_agg_rows<<<(int)std::min<int64_t>((R + 7) / 8, 8 * (int64_t)ctx->sm_count), 256, 0, s>>>(
            ctx->step_index.p, ctx->step_profiled.p, ctx->n_steps.p, (int32_t)R, W, ctx->runtime.p,
            overhead, ctx->agg_bsf.p, ctx->agg_times.p, d_total, d_first);
        CT_CUDA(cudaGetLastError());
    }
    if (max_len > 0) {
        if (sum0) CT_CUDA(cudaMemcpyAsync(d_sum0, sum0, 8 * (size_t)max_len, cudaMemcpyHostToDevice, s));
        if (sq0) CT_CUDA(cudaMemcpyAsync(d_sq0, sq0, 8 * (size_t)max_len, cudaMemcpyHostToDevice, s));
        k_agg_cols<<<(max_len + AGG_COLS - 1) / AGG_COLS, AGG_CHUNK, 0, s>>>(ctx->agg_bsf.p, ctx->n_steps.p, (int32_t)R, W,
                                                      max_len, sum0 ? d_sum0 : nullptr,
                                                      sq0 ? d_sq0 : nullptr, d_sum, d_sq);
        CT_CUDA(cudaGetLastError());
        CT_CUDA(cudaMemcpyAsync(sum_out, d_sum, 8 * (size_t)max_len, cudaMemcpyDeviceToHost, s));
        CT_CUDA(cudaMemcpyAsync(sq_out, d_sq, 8 * (size_t)max_len, cudaMemcpyDeviceToHost, s));
    }
    if (R > 0 && total_out)
        CT_CUDA(cudaMemcpyAsync(total_out, d_total, 8 * (size_t)R, cudaMemcpyDeviceToHost, s));
    if (R > 0 && first_out)
        CT_CUDA(cudaMemcpyAsync(first_out, d_first, 8 * (size_t)R, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    ctx->agg_valid = true;
    return CT_OK;
}

int ct_aggregate_time(ct_ctx* ctx, int32_t time_reps, const double* grid, int32_t n_grid,
                      const double* sum0, const double* sq0, double* sum_out, double* sq_out) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!ctx->agg_valid) return fail(CT_ERR_STATE, "ct_aggregate_steps must run first");
    if (n_grid < 1 || !grid || !sum_out || !sq_out) return fail(CT_ERR_VALUE, "bad grid buffers");
    const int64_t W = ctx->res_max_steps;
    const int32_t R = (int32_t)std::min<int64_t>(std::max(time_reps, 0), ctx->res_reps);
    cudaStream_t s = ctx->stream;
    CT_CUDA(ctx->agg_sampled.ensure((size_t)std::max(R, 1) * n_grid + 5 * (size_t)n_grid));
    double* d_grid = ctx->agg_sampled.p + (size_t)std::max(R, 1) * n_grid;
    double* d_sum0 = d_grid + n_grid;
    double* d_sq0 = d_sum0 + n_grid;
    double* d_sum = d_sq0 + n_grid;
    double* d_sq = d_sum + n_grid;
    CT_CUDA(cudaMemcpyAsync(d_grid, grid, 8 * (size_t)n_grid, cudaMemcpyHostToDevice, s));
    if (sum0) CT_CUDA(cudaMemcpyAsync(d_sum0, sum0, 8 * (size_t)n_grid, cudaMemcpyHostToDevice, s));
    if (sq0) CT_CUDA(cudaMemcpyAsync(d_sq0, sq0, 8 * (size_t)n_grid, cudaMemcpyHostToDevice, s));
    if (R > 0) {
        const int64_t pairs = (int64_t)R * n_grid;
        k_agg_sample<<<(int)std::min<int64_t>((pairs + 255) / 256, 16 * (int64_t)ctx->sm_count), 256, 0, s>>>(
            ctx->agg_bsf.p, ctx->agg_times.p, ctx->n_steps.p, R, W, d_grid, n_grid,
            ctx->agg_sampled.p);
        CT_CUDA(cudaGetLastError());
    }
    k_agg_time_sums<<<(n_grid + 63) / 64, 64, 0, s>>>(ctx->agg_sampled.p, R, n_grid,
                                                      sum0 ? d_sum0 : nullptr,
                                                      sq0 ? d_sq0 : nullptr, d_sum, d_sq);
    CT_CUDA(cudaGetLastError());
    CT_CUDA(cudaMemcpyAsync(sum_out, d_sum, 8 * (size_t)n_grid, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaMemcpyAsync(sq_out, d_sq, 8 * (size_t)n_grid, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaStreamSynchronize(s));
    return CT_OK;
}

int ct_report(ct_ctx* ctx, double overhead, int32_t time_reps, int32_t* n_steps,
              int32_t* status, int32_t* rep_error, ct_batch_stats* stats, int32_t* max_len,
              double* col_sum, double* col_sq, double* total_times, int32_t* n_grid,
              double* grid, double* tc_sum, double* tc_sq) {
    int rc = check_ctx(ctx); if (rc) return rc;
    if (!ctx->res_valid) return fail(CT_ERR_STATE, "no batched search launched");
    if (!ctx->runtime.p) return fail(CT_ERR_STATE, "no replay data uploaded");
    if (!n_steps || !status || !rep_error || !stats || !max_len || !col_sum || !col_sq ||
        !total_times || !n_grid || !grid || !tc_sum || !tc_sq)
        return fail(CT_ERR_VALUE, "null report buffer");
    const int64_t R = ctx->res_reps, W = ctx->res_max_steps;
    if (R < 1) return fail(CT_ERR_VALUE, "the report needs at least one repetition");
    const int32_t TR = (int32_t)std::min<int64_t>(std::max(time_reps, 1), R);
    cudaStream_t s = ctx->stream;
    CT_CUDA(ctx->agg_bsf.ensure((size_t)R * W));
    CT_CUDA(ctx->agg_times.ensure((size_t)R * W));
    // agg_vec: total[R] | first[R] | sum[W] | sq[W] | tc_sum[G] | tc_sq[G] | meta
    const size_t meta_d = (sizeof(AggMeta) + 7) / 8;
    CT_CUDA(ctx->agg_vec.ensure(2 * (size_t)R + 2 * (size_t)W + 2 * AGG_GRID + meta_d));
    double* d_total = ctx->agg_vec.p;
    double* d_first = d_total + R;
    double* d_sum = d_first + R;
    double* d_sq = d_sum + W;
    double* d_tcs = d_sq + W;
    double* d_tcq = d_tcs + AGG_GRID;
    AggMeta* d_meta = reinterpret_cast<AggMeta*>(d_tcq + AGG_GRID);
    CT_CUDA(ctx->agg_sampled.ensure((size_t)TR * AGG_GRID));
    // the column sums past the longest trajectory and the time-grid sums past
    // the grid's length are copied but never written (one contiguous block)
    CT_CUDA(cudaMemsetAsync(d_sum, 0, 8 * (2 * (size_t)W + 2 * (size_t)AGG_GRID), s));
    k_agg_rows<<<(int)std::min<int64_t>((R + 7) / 8, 8 * (int64_t)ctx->sm_count), 256, 0, s>>>(
        ctx->step_index.p, ctx->step_profiled.p, ctx->n_steps.p, (int32_t)R, W, ctx->runtime.p,
        overhead, ctx->agg_bsf.p, ctx->agg_times.p, d_total, d_first);
    CT_CUDA(cudaGetLastError());
    k_agg_meta<<<1, 1024, 0, s>>>(ctx->n_steps.p, d_total, d_first, (int32_t)R, TR, d_meta);
    CT_CUDA(cudaGetLastError());
    k_agg_cols<<<(int)((W + AGG_COLS - 1) / AGG_COLS), AGG_CHUNK, 0, s>>>(
        ctx->agg_bsf.p, ctx->n_steps.p, (int32_t)R, W, (int32_t)W, nullptr, nullptr, d_sum, d_sq,
        &d_meta->max_len);
    CT_CUDA(cudaGetLastError());
    const int64_t pairs = (int64_t)TR * AGG_GRID;
    k_agg_sample<<<(int)std::min<int64_t>((pairs + 255) / 256, 16 * (int64_t)ctx->sm_count), 256, 0, s>>>(
        ctx->agg_bsf.p, ctx->agg_times.p, ctx->n_steps.p, TR, W, nullptr, AGG_GRID,
        ctx->agg_sampled.p, d_meta);
    CT_CUDA(cudaGetLastError());
    k_agg_time_sums<<<(AGG_GRID + 63) / 64, 64, 0, s>>>(ctx->agg_sampled.p, TR, AGG_GRID, nullptr,
                                                        nullptr, d_tcs, d_tcq, d_meta);
    CT_CUDA(cudaGetLastError());
    // one page-locked landing area, several async copies, ONE synchronisation
    const size_t b_i = 3 * 4 * (size_t)R, b_st = 5 * 8, b_v = 8 * (2 * (size_t)W + R + 2 * AGG_GRID);
    const size_t b_all = ((b_i + 7) & ~(size_t)7) + b_st + b_v + sizeof(AggMeta);
    CT_CUDA(ctx->stage_report.acquire(b_all));
    unsigned char* h = static_cast<unsigned char*>(ctx->stage_report.p);
    int32_t* h_i = reinterpret_cast<int32_t*>(h);
    unsigned long long* h_st = reinterpret_cast<unsigned long long*>(h + ((b_i + 7) & ~(size_t)7));
    double* h_v = reinterpret_cast<double*>(h_st + 5);
    AggMeta* h_meta = reinterpret_cast<AggMeta*>(h_v + 2 * W + R + 2 * AGG_GRID);
    CT_CUDA(cudaMemcpyAsync(h_i, ctx->n_steps.p, 4 * R, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaMemcpyAsync(h_i + R, ctx->status.p, 4 * R, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaMemcpyAsync(h_i + 2 * R, ctx->rep_error.p, 4 * R, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaMemcpyAsync(h_st, ctx->stats.p, b_st, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaMemcpyAsync(h_v, d_sum, 8 * 2 * (size_t)W, cudaMemcpyDeviceToHost, s));  // sum | sq
    CT_CUDA(cudaMemcpyAsync(h_v + 2 * W, d_total, 8 * (size_t)R, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaMemcpyAsync(h_v + 2 * W + R, d_tcs, 8 * 2 * AGG_GRID, cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaMemcpyAsync(h_meta, d_meta, sizeof(AggMeta), cudaMemcpyDeviceToHost, s));
    CT_CUDA(cudaEventRecord(ctx->stage_report.done, s));
    CT_CUDA(cudaEventSynchronize(ctx->stage_report.done));
    std::memcpy(n_steps, h_i, 4 * R);
    std::memcpy(status, h_i + R, 4 * R);
    std::memcpy(rep_error, h_i + 2 * R, 4 * R);
    stats->configs_scored = (int64_t)h_st[0];
    stats->draws = (int64_t)h_st[1];
    stats->uncertified = (int64_t)h_st[2];
    stats->outer_iterations = (int64_t)h_st[3];
    stats->algorithmic_bytes = (int64_t)h_st[4];
    const int32_t ml = h_meta->max_len, ng = h_meta->n_grid;
    *max_len = ml;
    *n_grid = ng;
    std::memcpy(col_sum, h_v, 8 * (size_t)ml);
    std::memcpy(col_sq, h_v + W, 8 * (size_t)ml);
    std::memcpy(total_times, h_v + 2 * W, 8 * (size_t)R);
    std::memcpy(tc_sum, h_v + 2 * W + R, 8 * (size_t)ng);
    std::memcpy(tc_sq, h_v + 2 * W + R + AGG_GRID, 8 * (size_t)ng);
    std::memcpy(grid, h_meta->grid, 8 * (size_t)ng);
    ctx->agg_valid = true;
    return CT_OK;
}

int ct_result_device_ptrs(ct_ctx* ctx, void** step_index, void** step_profiled, void** n_steps,
                          void** status) {
    if (!ctx) return fail(CT_ERR_VALUE, "null context");
    if (!ctx->res_valid) return fail(CT_ERR_STATE, "no batched search launched");
    if (step_index) *step_index = ctx->step_index.p;
    if (step_profiled) *step_profiled = ctx->step_profiled.p;
    if (n_steps) *n_steps = ctx->n_steps.p;
    if (status) *status = ctx->status.p;
    return CT_OK;
}

}  // extern "C"
