// ct_tiled.cuh -- the batched replay search for large spaces, as grid-wide
// phase kernels instead of one persistent CTA per repetition.
//
// k_profile_search gives each repetition one CTA.  From a few hundred
// thousand configurations up its per-repetition state (weights, row index,
// explored bits) no longer fits shared memory, one CTA of 512 threads then
// streams the whole space through one SM, and the SMs run at a quarter of
// their warp slots (profiles/r02e_stress.md: 0.17 of HBM at 1M configs).
// Here every outer iteration of every repetition in the batch is four
// launches on the context's stream:
//
//   k_tiled_score    grid (repetition, tile of 4096 configurations): Eq. 16
//                    raw scores of the tile into the repetition's weight
//                    slice, the tile's max / min / smallest magnitude / NaN
//                    flag into a partials array                     [parallel]
//   k_tiled_reduce   one warp per repetition: the pool extrema from the
//                    tile partials                                     [tiny]
//   k_tiled_weights  grid (repetition, tile): Eq. 17 weights over the raw
//                    scores in place, 32-configuration row totals    [parallel]
//   k_tiled_draw     one warp per repetition: the n certified draws, the
//                    replay bookkeeping and the next profile step +
//                    expert system (draw_step / profile_step, the same
//                    device functions k_profile_search runs)          [serial]
//
// The repetition index runs fastest in the grid, so the CTAs resident at any
// moment work on the same few table tiles: the table streams from HBM about
// once per outer iteration and the repetitions share it through the L2.
// Every repetition executes the phases of k_profile_search in the same order
// on the same operands (raw scores, weights, row totals -- any summation
// order of the row totals is covered by the draw certificate), so the
// trajectories are identical.
#pragma once
#include "ct_search.cuh"

namespace ct {

constexpr int TILE_CONFIGS = 4096;          // configurations per tile (128 rows)
constexpr int TILED_NT = 256;               // threads per tile CTA

// per-repetition state in global memory
struct __align__(16) TiledRep {
    RepState rs;
    Ctl<1> ctl;
    int32_t it;      // outer iterations completed
    int32_t live;    // 1 while the repetition runs
};

struct TiledArgs {
    TiledRep* state;          // [batch]
    double* w;                // [batch][w_stride]   raw scores, then weights
    double* row_tot;          // [batch][nrows]
    uint32_t* expl;           // [batch][nwords]
    double4* partial;         // [batch][ntiles]      (max, min, amin, nan flag)
    int64_t w_stride;
    int32_t ntiles;
    int32_t rep0, batch;      // global index of the batch's first repetition, batch size
};

__device__ __forceinline__ int32_t* tiled_out_idx(const SearchArgs& a, int rep) {
    return a.step_index + (size_t)rep * a.max_steps;
}
__device__ __forceinline__ uint8_t* tiled_out_prof(const SearchArgs& a, int rep) {
    return a.step_profiled + (size_t)rep * a.max_steps;
}

// one warp per repetition: Generator seeding, first profile step
__global__ void __launch_bounds__(128) k_tiled_begin(const SearchArgs a, const TiledArgs t) {
    __shared__ uint32_t seed_sh[SEED_INLINE_WORDS];
    load_seed_words(a.seed, seed_sh);
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (b >= t.batch) return;
    const int rep = t.rep0 + b;
    TiledRep& st = t.state[b];
    uint32_t* expl = t.expl + (size_t)b * a.nwords;
    rep_begin(a, seed_sh, rep, st.rs, st.ctl, expl, lane);
    if (lane == 0) { st.it = 0; st.live = 1; }
    const int pcol = (lane < N_COMP) ? a.delta_col[lane] : -1;
    if (a.outer > 0)
        profile_step(a, st.rs, st.ctl, expl, tiled_out_idx(a, rep), tiled_out_prof(a, rep), lane, pcol);
    __syncwarp();
    if (a.outer <= 0 || st.ctl.done) {
        if (lane == 0) { rep_end(a, rep, st.rs); st.live = 0; }
    }
}

// Eq. 16 over one tile of one repetition
__global__ void __launch_bounds__(TILED_NT) k_tiled_score(const SearchArgs a, const TiledArgs t) {
    constexpr int NW = TILED_NT / 32;
    const int b = blockIdx.x, tile = blockIdx.y;
    const TiledRep& st = t.state[b];
    if (!st.live) return;
    __shared__ Ctl<1> ctl;                       // the repetition's active terms
    __shared__ double r_max[NW], r_min[NW], r_amin[NW];
    __shared__ int r_nan[NW];
    {
        const int* src = reinterpret_cast<const int*>(&st.ctl);
        int* dst = reinterpret_cast<int*>(&ctl);
        for (int i = threadIdx.x; i < (int)(sizeof(Ctl<1>) / 4); i += TILED_NT) dst[i] = src[i];
    }
    __syncthreads();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t* expl = t.expl + (size_t)b * a.nwords;
    double* w = t.w + (size_t)b * t.w_stride;
    const int64_t lo = (int64_t)tile * TILE_CONFIGS;
    const int64_t hi = min(a.n, lo + TILE_CONFIGS);
    double lmax = -INFINITY, lmin = INFINITY, lamin = INFINITY;
    bool nan = false;
    if (ctl.cert_terms) score_pass<TILED_NT, true>(a, ctl, expl, w, tid, lmax, lmin, lamin, nan, lo, hi);
    else score_pass<TILED_NT, false>(a, ctl, expl, w, tid, lmax, lmin, lamin, nan, lo, hi);
    lmax = warp_max(lmax);
    lmin = warp_min(lmin);
    const bool wnan = __any_sync(FULL, nan);
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) lamin = fmin(lamin, __shfl_xor_sync(FULL, lamin, m));
    if (lane == 0) { r_max[warp] = lmax; r_min[warp] = lmin; r_amin[warp] = lamin; r_nan[warp] = wnan; }
    __syncthreads();
    if (tid == 0) {
        double mx = r_max[0], mn = r_min[0], am = r_amin[0];
        int nn = r_nan[0];
#pragma unroll
        for (int i = 1; i < NW; ++i) {
            mx = fmax(mx, r_max[i]); mn = fmin(mn, r_min[i]); am = fmin(am, r_amin[i]);
            nn |= r_nan[i];
        }
        t.partial[(size_t)b * t.ntiles + tile] = make_double4(mx, mn, am, nn ? 1.0 : 0.0);
    }
}

// one warp per repetition: pool extrema (NaN anywhere -> max = min = NaN, as
// numpy's max()/min(); the smallest magnitude ignores NaN) into ctl.red_*[0]
__global__ void __launch_bounds__(128) k_tiled_reduce(const SearchArgs a, const TiledArgs t) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (b >= t.batch) return;
    TiledRep& st = t.state[b];
    if (!st.live) return;
    double mx = -INFINITY, mn = INFINITY, am = INFINITY;
    bool nan = false;
    const double4* p = t.partial + (size_t)b * t.ntiles;
    for (int i = lane; i < t.ntiles; i += 32) {
        const double4 v = p[i];
        mx = fmax(mx, v.x); mn = fmin(mn, v.y); am = fmin(am, v.z); nan |= v.w != 0.0;
    }
    mx = warp_max(mx);
    mn = warp_min(mn);
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) am = fmin(am, __shfl_xor_sync(FULL, am, m));
    if (__any_sync(FULL, nan)) { mx = NAN; mn = NAN; }
    if (lane == 0) {
        st.ctl.red_max[0] = mx; st.ctl.red_min[0] = mn; st.ctl.red_amin[0] = am;
        st.ctl.red_bad[0] = 0;
    }
}

// Eq. 17 over one tile of one repetition: weights in place, row totals
__global__ void __launch_bounds__(TILED_NT) k_tiled_weights(const SearchArgs a, const TiledArgs t) {
    constexpr int NW = TILED_NT / 32;
    const int b = blockIdx.x, tile = blockIdx.y;
    TiledRep& st = t.state[b];
    if (!st.live) return;
    const int warp = threadIdx.x >> 5;
    const double smax = st.ctl.red_max[0], smin = st.ctl.red_min[0], amin = st.ctl.red_amin[0];
    // certified Eq. 17 domain (weight_phase)
    const double lo_c = 3.872591914849318e-121, hi_c = 2.5822498780869086e+120;
    const bool cert = (amin >= lo_c || amin == INFINITY) && smax <= hi_c && smin >= -hi_c;
    const uint32_t* expl = t.expl + (size_t)b * a.nwords;
    double* w = t.w + (size_t)b * t.w_stride;
    double* row_tot = t.row_tot + (size_t)b * a.nrows;
    const int r0 = tile * (TILE_CONFIGS / 32);
    const int r1 = min(a.nrows, r0 + TILE_CONFIGS / 32);
    // the tile's 32 KB of raw scores are pulled into L2 at once (one 128-byte
    // line per thread): the row groups below then wait an L2 round trip,
    // not a DRAM one, and the kernel streams instead of stalling per group
    static_assert(TILE_CONFIGS == TILED_NT * 16, "one line of 16 doubles per thread");
    {
        const int64_t e = (int64_t)tile * TILE_CONFIGS + 16 * threadIdx.x;
        if (e < a.n) asm volatile("prefetch.global.L2 [%0];" ::"l"(w + e));
    }
    int bad = 0;
    if (cert) weight_pass<true, false>(a, warp, NW, smax, smin, expl, w, w, row_tot, bad, r0, r1);
    else weight_pass<false, false>(a, warp, NW, smax, smin, expl, w, w, row_tot, bad, r0, r1);
    if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(&st.ctl.red_bad[0], 1);
}

// one warp per repetition: the n draws, bookkeeping, next profile step
__global__ void __launch_bounds__(128) k_tiled_draw(const SearchArgs a, const TiledArgs t) {
    __shared__ u128 jA[33], jC[33];
    if (threadIdx.x == 0) Pcg64::jump_tables(jA, jC, 32);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (b >= t.batch) return;
    TiledRep& st = t.state[b];
    if (!st.live) return;
    const int rep = t.rep0 + b;
    uint32_t* expl = t.expl + (size_t)b * a.nwords;
    double* w = t.w + (size_t)b * t.w_stride;
    double* row_tot = t.row_tot + (size_t)b * a.nrows;
    int32_t* out_idx = tiled_out_idx(a, rep);
    uint8_t* out_prof = tiled_out_prof(a, rep);
    draw_step<false, 1, true>(a, st.rs, st.ctl, expl, w, w, row_tot, jA, jC, out_idx, out_prof, lane);
    const int it = st.it + 1;
    const int pcol = (lane < N_COMP) ? a.delta_col[lane] : -1;
    if (!st.ctl.done && it < a.outer) profile_step(a, st.rs, st.ctl, expl, out_idx, out_prof, lane, pcol);
    __syncwarp();
    if (lane == 0) st.it = it;
    if (st.ctl.done || it >= a.outer) {
        if (lane == 0) { rep_end(a, rep, st.rs); st.live = 0; }
    }
}

}  // namespace ct
