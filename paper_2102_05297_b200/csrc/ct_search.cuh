// ct_search.cuh -- the batched replay search kernel (Alg. 1 over R repetitions).
//
// One CTA runs one repetition of run_profile_search (search.py:338-399) end to
// end and then takes the next repetition (persistent grid sized to the
// resident-CTA capacity).  Per outer iteration, inside the CTA:
//
//   warp 0     record the profiled step, replay its counters, analyze() +
//              react() (Eqs. 6-15) on 18 lanes, ballot-compact the active
//              terms                                                   [serial]
//   all warps  Eq. 16 raw score of every unexplored configuration,
//              coalesced column reads of the column-major table, pool
//              max / min / smallest magnitude                          [parallel]
//   all warps  Eq. 17 weights (stored over the raw scores); each 32-
//              configuration row's exact 2^-66 fixed-point total from
//              three 32-bit limb reductions (REDUX)                    [parallel]
//   warp 0     n certified inverse-CDF draws: a ballot over per-lane row
//              chunks finds the row, one limb scan of that row and a
//              ballot the configuration; zeroing a drawn weight patches
//              its row total and the lane prefixes (exact), then replay
//              lookups, stop test, argmin with later ties              [serial]
//
// The serial phases run on one warp while the others wait, so they are kept
// to a few hundred instructions per draw.  The weights live in shared memory
// when all repetitions still fit on the GPU at once, otherwise in a per-CTA
// slice of global scratch (L2-resident).  The numpy Generator stream of the
// repetition is regenerated on the device (ct_rng.cuh).
#pragma once
#include "ct_select.cuh"
#include "ct_expert.cuh"
#include "ct_rng.cuh"
#include "countertune_b200.h"

namespace ct {

constexpr int MAX_ACTIVE = 18;

// seed words travel inside the kernel arguments: a launch needs no copy and
// no host synchronisation
constexpr int SEED_INLINE_WORDS = 64;

struct SeedInline {
    uint32_t w[SEED_INLINE_WORDS];   // entropy words, then spawn-prefix words
    int32_t n_entropy, n_prefix;
    int32_t child_per_rep;
    int64_t rep_offset;
};

// Shared-memory copy of the launch's seed words (all threads take part).
__device__ __forceinline__ void load_seed_words(const SeedInline& s, uint32_t* sh) {
    for (int i = threadIdx.x; i < s.n_entropy + s.n_prefix; i += blockDim.x) sh[i] = s.w[i];
    __syncthreads();
}

__device__ __forceinline__ SeedWords seed_words_of(const SeedInline& s, const uint32_t* sh,
                                                   int64_t rep) {
    return SeedWords{sh, s.n_entropy, sh + s.n_entropy, s.n_prefix, s.child_per_rep != 0,
                     (uint32_t)(s.rep_offset + rep)};
}

struct SearchArgs {
    // prediction table, column-major: column j of config i at table[j * ld + i]
    const double* table;
    int64_t ld;
    int64_t n;
    // replay data (DatasetReplaySource)
    const double* runtime;
    const int64_t* threads;
    const double* counters;      // n x 23, REQUIRED_COUNTERS order
    const uint8_t* has_record;
    const uint32_t* stop_bits;   // nullable
    // search parameters
    int32_t outer, inner;
    double inst_reaction, issue_sign, gamma;
    int32_t literal_sign, generation;
    int64_t cores;
    int32_t delta_col[18];
    // device words written by the table upload: [0] bit j = table column j
    // admits raw_term_cert, [1] bit j = column j holds no exact zero
    const unsigned long long* col_flags;
    SeedInline seed;
    int32_t n_reps;
    // rows of 32 configurations
    int32_t nrows;
    int64_t nwords;
    int32_t force_sequential;    // test hook: decide every draw sequentially
    double cert_slack;           // test hook: certificate half-width multiplier (1 = proven bound)
    // score_top_k (search.py:133-140): < 0 is None; assign is the space's
    // n x n_params assignment matrix (row-major), read for the distances
    int64_t topk;
    const double* assign;
    int32_t n_params;
    // storage: weights (8 B each, nrows * 32) in shared memory or a per-CTA
    // slice of scratch_w
    double* scratch_w;
    unsigned char* scratch_head;   // HG kernels: per-CTA row totals + explored bits
    // outputs
    int32_t* step_index;
    uint8_t* step_profiled;
    int64_t max_steps;
    int32_t* n_steps;
    int32_t* status;
    int32_t* rep_error;
    unsigned long long* stats;   // configs_scored, draws, uncertified, outer, bytes
};

__device__ __forceinline__ bool bit_get(const uint32_t* b, int64_t i) {
    return (b[i >> 5] >> (i & 31)) & 1u;
}

struct __align__(16) RepState {
    Pcg64 rng;
    int64_t c_prof, ns, n_expl;
    int st, err;
    unsigned long long scored, draws, uncert, outers, abytes;
};

#ifdef CT_PHASE_CLOCKS
// sub-phase clocks of draw_step (lane 0 of the drawing warp): setup, locate,
// certify+zero, lookups, bookkeeping
__device__ unsigned long long g_subclk[8];
#define CT_SUB(k) do { if (lane == 0) { long long n_ = clock64(); atomicAdd(&g_subclk[k], (unsigned long long)(n_ - sub_t)); sub_t = n_; } } while (0)
#define CT_SUB_START() long long sub_t = clock64()
#else
#define CT_SUB(k) do { } while (0)
#define CT_SUB_START() do { } while (0)
#endif

template <int NW>
struct __align__(16) Ctl {
    double red_max[NW];
    double red_min[NW];
    double red_amin[NW];
    int red_bad[NW];
    ActiveTerm act[MAX_ACTIVE];
    double cnt[N_REQ];
    int n_act;
    int done;
    int cert_terms;
    int cmd;          // k_profile_search_ws: what the parallel warps do next
};

// Eq. 16 over the whole space for one repetition's active terms: raw score of
// configuration e into w[e], pool max / min / smallest nonzero magnitude
// returned per thread (max / min ignore NaN here; `nan` records one, and the
// caller turns the extrema into NaN as numpy's max()/min() would).  PT
// threads share the space (ptid = 0..PT-1).  Full groups of 4 configurations
// per thread run unguarded (columns are padded to a multiple of 2048, so the
// four loads use one base pointer and immediate offsets); the last partial
// group goes one configuration at a time, so no work is spent on the padding.
__device__ __forceinline__ void score_epilogue(double acc, int64_t e, const uint32_t* expl,
                                               double* w, double& lmax, double& lmin,
                                               double& lamin, bool& nan) {
    // branch-free: an explored configuration contributes the neutral element
    // and leaves a NaN, which Eq. 17 maps to weight 0 exactly as it maps an
    // explored one (the weight pass then needs no explored test)
    const bool in = !bit_get(expl, e);
    w[e] = in ? acc : __longlong_as_double(0x7ff8000000000000ll);
    const double vmax = in ? acc : -INFINITY, vmin = in ? acc : INFINITY;
    lmax = (vmax > lmax) ? vmax : lmax;
    lmin = (vmin < lmin) ? vmin : lmin;
    const double m = fabs(acc);
    lamin = (in && m != 0.0 && m < lamin) ? m : lamin;
    nan |= in && (acc != acc);
}

// one Eq. 16 term added to four configurations' raw scores
template <bool CERT>
__device__ __forceinline__ void term4(const ActiveTerm& t, const double* c, double* acc) {
    const double d = t.d, pv = t.p;
    if (CERT && t.nz) {      // block-uniform: no zero in the column
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = add(acc[u], raw_term_cert_nz(c[u], d, pv));
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
            acc[u] = add(acc[u], CERT ? raw_term_cert(c[u], d, pv) : raw_term_nb(c[u], d, pv));
    }
}

template <int PT, bool CERT, int NW>
__device__ __forceinline__ void score_pass(const SearchArgs& a, const Ctl<NW>& ctl,
                                           const uint32_t* expl, double* w, int ptid, double& lmax,
                                           double& lmin, double& lamin, bool& nan,
                                           int64_t lo, int64_t hi) {
    // configurations [lo, hi) (the whole space, or one tile of the tiled path)
    const int n_act = ctl.n_act;
    int64_t base = lo + ptid;
    for (; base + 3LL * PT < hi; base += 4LL * PT) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        // two terms per step: eight loads in flight, then the terms in
        // react() order for each configuration
        int k = 0;
        for (; k + 1 < n_act; k += 2) {
            const double* col0 = a.table + (size_t)ctl.act[k].col * a.ld + base;
            const double* col1 = a.table + (size_t)ctl.act[k + 1].col * a.ld + base;
            double c0[4], c1[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { c0[u] = __ldg(col0 + u * PT); c1[u] = __ldg(col1 + u * PT); }
            term4<CERT>(ctl.act[k], c0, acc);
            term4<CERT>(ctl.act[k + 1], c1, acc);
        }
        if (k < n_act) {
            const double* col = a.table + (size_t)ctl.act[k].col * a.ld + base;
            double c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) c[u] = __ldg(col + u * PT);
            term4<CERT>(ctl.act[k], c, acc);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            score_epilogue(acc[u], base + (int64_t)u * PT, expl, w, lmax, lmin, lamin, nan);
    }
    for (; base < hi; base += PT) {
        double acc = 0.0;
        for (int k = 0; k < n_act; ++k) {
            const double c = __ldg(a.table + (size_t)ctl.act[k].col * a.ld + base);
            acc = add(acc, CERT ? raw_term_cert(c, ctl.act[k].d, ctl.act[k].p)
                                : raw_term_nb(c, ctl.act[k].d, ctl.act[k].p));
        }
        score_epilogue(acc, base, expl, w, lmax, lmin, lamin, nan);
    }
}

// Eq. 17 weights over the raw scores (weight() in ct_hd.cuh with the pool's
// reciprocals hoisted, search.py:156-170), each row's total and -- with PRE -- each
// configuration's inclusive in-row prefix (float64): warp pw of the nw-warp
// group takes rows pw, pw+nw, ...; lane l owns configuration 32 t + l
// (padding and explored lanes write weight 0).  s_min == 0 makes every
// non-positive pool score 0 and its ratio 0, which dividing 0 by 1 gives
// too, so the per-element den == 0 test is folded into (smin_e, y_min).
// Every pool weight of finite scores is in [1e-4, 256]; bad flags NaN / Inf
// (the reference then draws from non-finite weights).
template <bool CERT>
__device__ __forceinline__ double weight_of(double s, double smax, double smin_e, double y_max,
                                            double y_min, double gamma) {
    const bool pos = s > 0.0;
    const double den = pos ? smax : smin_e;
    double r;
    double ratio = markstein(s, den, pos ? y_max : y_min, &r);
    if (!CERT) {
        if (__builtin_expect(!dvd_accept(s, den, r, ratio), 0)) ratio = dvd_term(s, den);
    }
    // 1 - ratio == 1 + (-ratio) exactly: one add, the sign by select
    const double w = pow8(add(1.0, pos ? ratio : -ratio));
    if (pos) return (w > SCORE_CEILING) ? SCORE_CEILING : w;            // np.minimum
    if (s > gamma) return (w < SCORE_FLOOR) ? SCORE_FLOOR : w;          // np.maximum
    return (s <= gamma) ? SCORE_FLOOR : 0.0;                            // NaN: no branch
}

template <bool CERT, bool PRE>
__device__ __forceinline__ void weight_pass(const SearchArgs& a, int pw, int nw, double smax,
                                            double smin, const uint32_t* expl, double* w,
                                            double* pre, double* row_tot, int& bad,
                                            int row_begin, int row_end) {
    // rows [row_begin, row_end) (all rows, or one tile's of the tiled path)
    const int lane = threadIdx.x & 31;
    const int64_t N = a.n;
    const double gamma = a.gamma;
    const double smin_e = (smin != 0.0) ? smin : 1.0;
    const double y_max = rcp_nv(smax), y_min = rcp_nv(smin_e);
    if constexpr (!PRE) {
        // row totals only, four rows of this warp at a time, reduced together:
        // two exchange levels halve the rows a lane holds (lane 8r ends up
        // with row r of the group), three butterfly levels finish the sums --
        // 6 shuffles per 4 rows instead of 20.  Any order is fine: the draw
        // certificate covers every summation order.
        for (int t0 = row_begin + pw; t0 < row_end; t0 += 4 * nw) {
            double v[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int t = t0 + i * nw;
                const int64_t e = 32LL * t + lane;
                double wt = 0.0;
                if (t < row_end) {
                    if (e < N && (CERT || !bit_get(expl, e)))
                        wt = weight_of<CERT>(w[e], smax, smin_e, y_max, y_min, gamma);
                    w[e] = wt;
                }
                bad |= !(wt <= SCORE_CEILING);
                v[i] = wt;
            }
            const bool up16 = lane & 16, up8 = lane & 8;
#pragma unroll
            for (int i = 0; i < 2; ++i) {      // rows {i, i+2}: lower lanes keep i
                const double send = up16 ? v[i] : v[i + 2];
                const double keep = up16 ? v[i + 2] : v[i];
                v[i] = add(keep, __shfl_xor_sync(FULL, send, 16));
            }
            {                                   // rows {0, 1} of what is left
                const double send = up8 ? v[0] : v[1];
                const double keep = up8 ? v[1] : v[0];
                v[0] = add(keep, __shfl_xor_sync(FULL, send, 8));
            }
#pragma unroll
            for (int d = 4; d > 0; d >>= 1) v[0] = add(v[0], __shfl_xor_sync(FULL, v[0], d));
            // lane 8r holds row r = 2 (lane >> 4 & 1) + (lane >> 3 & 1)
            const int r = ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);
            const int t = t0 + r * nw;
            if ((lane & 7) == 0 && t < row_end) row_tot[t] = v[0];
        }
    } else {
        for (int t = row_begin + pw; t < row_end; t += nw) {
            const int64_t e = 32LL * t + lane;
            double wt = 0.0;
            if (e < N && (CERT || !bit_get(expl, e))) wt = weight_of<CERT>(w[e], smax, smin_e, y_max, y_min, gamma);
            w[e] = wt;
            bad |= !(wt <= SCORE_CEILING);
            double incl = wt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double v = __shfl_up_sync(FULL, incl, d);
                if (lane >= d) incl = add(incl, v);
            }
            pre[e] = incl;
            if (lane == 31) row_tot[t] = incl;
        }
    }
}

// ---------------------------------------------------------------------------
// The phases of one outer iteration of one repetition.  A repetition's state
// is (RepState, Ctl, explored bits, weights, row totals); the phases below are
// shared by both kernels.

// Start a repetition: Generator seeded from the repetition's SeedSequence
// child, first profile drawn with integers(0, N) (search.py:359-364).  One
// full warp; the explored bits are cleared cooperatively.
template <int NW>
__device__ __forceinline__ void rep_begin(const SearchArgs& a, const uint32_t* seed_sh, int rep,
                                          RepState& rs, Ctl<NW>& ctl, uint32_t* expl, int lane) {
    for (int64_t i = lane; i < a.nwords; i += 32) expl[i] = 0u;
    if (lane == 0) {
        rs.c_prof = 0; rs.ns = 0; rs.n_expl = 0; rs.st = CT_STATUS_BUDGET; rs.err = 0;
        rs.scored = 0; rs.draws = 0; rs.uncert = 0; rs.outers = 0; rs.abytes = 0;
        rs.rng.seed(seed_pool(seed_words_of(a.seed, seed_sh, rep)));
        rs.c_prof = (int64_t)rs.rng.integers((uint64_t)a.n);
        ctl.done = 0;
    }
    __syncwarp();
}

__device__ __forceinline__ void rep_end(const SearchArgs& a, int rep, const RepState& rs) {
    a.n_steps[rep] = (int32_t)rs.ns;
    a.status[rep] = rs.st;
    a.rep_error[rep] = rs.err;
    atomicAdd(&a.stats[0], rs.scored);
    atomicAdd(&a.stats[1], rs.draws);
    atomicAdd(&a.stats[2], rs.uncert);
    atomicAdd(&a.stats[3], rs.outers);
    atomicAdd(&a.stats[4], rs.abytes);
}

// Profile step + expert system (one full warp).  One lane per counter
// fetches the profile's replayed counters and one lane per delta key its
// predicted value p; the 18 bottleneck components and their reactions are
// evaluated on 18 lanes (analyze_component_warp: the scalar analyze()'s
// operations) and the active terms compacted in react() order with a ballot.
template <int NW>
__device__ __forceinline__ void profile_step(const SearchArgs& a, RepState& rs, Ctl<NW>& ctl,
                                             uint32_t* expl, int32_t* out_idx, uint8_t* out_prof,
                                             int lane, int col) {
    // col: this lane's delta column (a.delta_col[lane], -1 past N_COMP),
    // loaded once per kernel so that every load here depends on c_prof only
    const int64_t N = a.n;
    const int64_t cp = rs.c_prof;
    if (lane < N_REQ) ctl.cnt[lane] = a.counters[(size_t)cp * N_REQ + lane];
    const double pv = (col >= 0) ? a.table[(size_t)col * a.ld + cp] : 0.0;
    const bool rec_ok = a.has_record[cp] != 0;
    const bool is_stop = a.stop_bits && bit_get(a.stop_bits, cp);
    const int64_t thr = a.threads[cp];
    const unsigned long long col_cert = a.col_flags[0], col_nz = a.col_flags[1];
    __syncwarp();
    double dk = 0.0;
    const double bk = analyze_component_warp(ctl.cnt, lane < N_COMP ? lane : N_COMP - 1,
                                             a.generation, a.cores, thr, degenerate_of(ctl.cnt));
    if (lane < N_COMP) dk = react_component(bk, lane, a.inst_reaction, a.issue_sign);
    const bool act = (lane < N_COMP) && dk != 0.0 && col >= 0 && pv != 0.0;
    const unsigned amask = __ballot_sync(FULL, act);
    if (act) {
        const int slot = __popc(amask & ((1u << lane) - 1u));
        ctl.act[slot].col = col;
        ctl.act[slot].nz = (col < 64 && ((col_nz >> col) & 1ull)) ? 1 : 0;
        ctl.act[slot].p = pv;
        // literal sign: (-d)(c - p) == d(p - c) exactly
        ctl.act[slot].d = a.literal_sign ? -dk : dk;
    }
    // certified division domain for every active term
    const double two_m200 = 6.223015277861142e-61;
    const bool cert_ok = !act || (col < 64 && ((col_cert >> col) & 1ull) && fabs(dk) >= two_m200);
    const bool cert_all = __all_sync(FULL, cert_ok);
    if (lane == 0) {
        const int na = __popc(amask);
        ctl.n_act = na;
        ctl.cert_terms = cert_all ? 1 : 0;
        if (!rec_ok) {
            rs.st = CT_STATUS_ERROR; rs.err = -4; ctl.done = 1;
            if (rs.ns < a.max_steps) out_idx[rs.ns] = (int32_t)cp;   // failing index
        } else {
            out_idx[rs.ns] = (int32_t)cp; out_prof[rs.ns] = 1; ++rs.ns;
            uint32_t m = 1u << (cp & 31);
            if (!(expl[cp >> 5] & m)) { expl[cp >> 5] |= m; ++rs.n_expl; }
            if (is_stop) { rs.st = CT_STATUS_STOPPED; ctl.done = 1; }
            else if (rs.n_expl >= N) { rs.st = CT_STATUS_EXHAUSTED; ctl.done = 1; }
            else {
                unsigned long long pool = (unsigned long long)(N - rs.n_expl);
                // top-K scores the K nearest unexplored configurations only
                if (a.topk >= 0 && (unsigned long long)a.topk < pool) pool = (unsigned long long)a.topk;
                rs.scored += pool; ++rs.outers;
                rs.abytes += pool * (8ull * (unsigned long long)na + 16ull);
            }
        }
    }
    __syncwarp();
}

// Eq. 16 for the group's share (PT threads, ptid = 0..PT-1), reduced per warp
// into ctl.red_*[ptid / 32].
template <int PT, int NW>
__device__ __forceinline__ void score_phase(const SearchArgs& a, Ctl<NW>& ctl, const uint32_t* expl,
                                            double* w, int ptid) {
    const int lane = ptid & 31, pw = ptid >> 5;
    double lmax = -INFINITY, lmin = INFINITY, lamin = INFINITY;
    bool nan = false;
    if (ctl.cert_terms) score_pass<PT, true>(a, ctl, expl, w, ptid, lmax, lmin, lamin, nan, 0, a.n);
    else score_pass<PT, false>(a, ctl, expl, w, ptid, lmax, lmin, lamin, nan, 0, a.n);
    lmax = warp_max(lmax);
    lmin = warp_min(lmin);
    if (__any_sync(FULL, nan)) { lmax = NAN; lmin = NAN; }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) lamin = fmin(lamin, __shfl_xor_sync(FULL, lamin, m));
    if (lane == 0) { ctl.red_max[pw] = lmax; ctl.red_min[pw] = lmin; ctl.red_amin[pw] = lamin; }
}

// Eq. 17 weights (+ in-row prefixes) for warp pw of the NW-warp group (after
// every warp's score_phase is visible), reduced into ctl.red_bad[pw].
template <bool PRE, int NW>
__device__ __forceinline__ void weight_phase(const SearchArgs& a, Ctl<NW>& ctl, const uint32_t* expl,
                                             double* w, double* pre, double* row_tot, int pw) {
    const int lane = threadIdx.x & 31;
    double smax = ctl.red_max[0], smin = ctl.red_min[0], amin = ctl.red_amin[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) {
        smax = nmax(smax, ctl.red_max[i]); smin = nmin(smin, ctl.red_min[i]);
        amin = fmin(amin, ctl.red_amin[i]);
    }
    // certified Eq. 17 domain: every nonzero |s| in [2^-400, 2^400]
    // (NaN extrema fail the comparisons)
    const double lo = 3.872591914849318e-121, hi = 2.5822498780869086e+120;
    const bool cert = (amin >= lo || amin == INFINITY) && smax <= hi && smin >= -hi;
    int bad = 0;
    if (cert) weight_pass<true, PRE>(a, pw, NW, smax, smin, expl, w, pre, row_tot, bad, 0, a.nrows);
    else weight_pass<false, PRE>(a, pw, NW, smax, smin, expl, w, pre, row_tot, bad, 0, a.nrows);
    bad = __any_sync(FULL, bad);
    if (lane == 0) ctl.red_bad[pw] = bad;
}

// n certified draws, replay lookups, stop test and the later-ties-win argmin
// (one full warp).  Sets ctl.done when the repetition ends here.
//
// Locating r: lane L owns a contiguous chunk of rows and keeps the inclusive
// prefix over the chunks (lane_pref); a ballot finds the chunk, lane L walks
// its rows, and the row's precomputed in-row prefixes give the configuration
// with one more ballot.  All sums are float64; the choice is CERTIFIED.  With
// u = 2^-53, W the exact sum of our weights, T our computed total:
//  * numpy's weights w' and ours w are each within 1 ulp of the exact x^8,
//    so |w_i - w'_i| < 4u w_i and |S'(j) - S(j)| < 4u W (exact prefixes);
//  * the reference's sequential cumsum c'(j) = recursive summation of
//    nonnegative terms: |c'(j) - S'(j)| <= gamma_(N-1) W';
//  * our prefix P(j) passes every weight through at most d additions -- 5
//    in the row-total tree, <= cpl in the lane-chunk sum, 5 in the lane
//    scan, <= max(cpl, 6) in the row walk (or 5 + 1 in the slab scan), 5 + 1
//    in the in-row scan: d <= 2 cpl + 22 -- plus <= 3 inner zeroing
//    subtractions (row total, chunk sum, lane prefix per draw): |P(j) -
//    S(j)| <= gamma_(d + 3 inner) W;
//  * hence E = |c'(j) - P(j)| <= (N + 2 cpl + 3 inner + 26) u W (1 + O(Nu)),
//    and r' = fl(U c'(N)), r = fl(U T) give |r' - r| <= E + 2u W;
//  * P(i-1) + B < r and r + B < P(i) with B >= 2E + 2uW + the comparisons'
//    own roundings imply c'(i-1) <= r' < c'(i): the reference picks i too.
// B = (2N + 4 cpl + 6 inner + 64) u T (1 + 2^-40) covers it (T >= W(1 -
// gamma_d), and the slack terms absorb the second-order parts).  Otherwise
// the draw is re-decided with the sequential float64 cumsum.
template <bool PRE, int NW, bool COOP = false>
__device__ __forceinline__ void draw_step(const SearchArgs& a, RepState& rs, Ctl<NW>& ctl,
                                          uint32_t* expl, double* w, double* pre, double* row_tot,
                                          const u128* jA, const u128* jC, int32_t* out_idx,
                                          uint8_t* out_prof, int lane) {
    const int64_t N = a.n;
    CT_SUB_START();
    // every pool configuration has a weight in [1e-4, 256] unless bad
    int positive = (int)(N - rs.n_expl), bad = 0;
    if (a.topk >= 0 && a.topk < positive) positive = (int)a.topk;   // the top-K pool
#pragma unroll
    for (int i = 0; i < NW; ++i) bad |= ctl.red_bad[i];
    const int cpl = (a.nrows + 31) >> 5;
    const int t0 = lane * cpl, t1 = min(t0 + cpl, a.nrows);
    double mine = 0.0;
    for (int t = t0; t < t1; ++t) mine = add(mine, row_tot[t]);
    double lane_pref = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double v = __shfl_up_sync(FULL, lane_pref, d);
        if (lane >= d) lane_pref = add(lane_pref, v);
    }
    double total = __shfl_sync(FULL, lane_pref, 31);
    // certificate half-width (derivation at the top of draw_step):
    // (2N + 4 cpl + 6 inner + 64) 2^-53 T, times the test hook's slack
    const double B = (double)(2 * N + 4 * (int64_t)cpl + 6 * (int64_t)a.inner + 64) *
                     1.1102230246251565e-16 * total * (1.0 + 0x1p-40) * a.cert_slack;
    int done = 0;
    if (bad) { if (lane == 0) { rs.st = CT_STATUS_ERROR; rs.err = -7; } done = 1; }
    double t_best = INFINITY;
    CT_SUB(0);
    // The iteration's uniforms come 32 at a time from the repetition's PCG64
    // by jump-ahead (lane j: the (j+1)-th next Generator.random()), the draws
    // of a chunk touch shared memory only, and their replay lookups are issued
    // together afterwards: one L2 round trip per chunk instead of one per
    // draw.  Draws past a stop / error are discarded (the repetition ends
    // there, as the reference's loop does).
    Pcg64 g;
    g.state = rs.rng.state;
    g.inc = rs.rng.inc;
    int k = 0;
    bool exhausted = false;
    while (k < a.inner && !done) {
        const int k0 = k;
        const int cnt = min(32, a.inner - k0);
        const double u_lane = (lane < cnt) ? g.double_after(jA[lane + 1], jC[lane + 1]) : 0.0;
        int64_t my_choice = -1;
        for (; k < k0 + cnt; ++k) {
            if (positive <= 0) { exhausted = true; break; }
            CT_SUB(1);
            const double u = __shfl_sync(FULL, u_lane, k - k0);
            const double r = mul(u, total);
            int64_t chosen = -1;
            bool ok = false;
            int row = -1, l2 = -1;
            const unsigned bal = __ballot_sync(FULL, lane_pref > r);
            if (bal) {
                const int L = __ffs(bal) - 1;
                double carry = __shfl_up_sync(FULL, lane_pref, 1);
                if (lane == 0) carry = 0.0;
                if constexpr (COOP) {
                    // long chunks (large spaces): the whole warp walks lane
                    // L's chunk 32 rows at a time -- a warp scan of the row
                    // totals and a ballot per slab instead of one dependent
                    // add per row (any summation order is certified)
                    carry = __shfl_sync(FULL, carry, L);
                    const int c0 = L * cpl, c1 = min(c0 + cpl, a.nrows);
                    for (int base = c0; base < c1; base += 32) {
                        const int t = base + lane;
                        double incl = (t < c1) ? row_tot[t] : 0.0;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const double v = __shfl_up_sync(FULL, incl, d);
                            if (lane >= d) incl = add(incl, v);
                        }
                        const double cand = add(carry, incl);
                        const unsigned fb = __ballot_sync(FULL, t < c1 && cand > r);
                        if (fb) {
                            const int l = __ffs(fb) - 1;
                            double prev = __shfl_up_sync(FULL, cand, 1);
                            if (lane == 0) prev = carry;
                            row = base + l;
                            carry = __shfl_sync(FULL, prev, l);
                            break;
                        }
                        carry = __shfl_sync(FULL, cand, 31);
                    }
                } else {
                    if (lane == L) {
                        for (int t = t0; t < t1; ++t) {
                            const double nxt = add(carry, row_tot[t]);
                            if (nxt > r) { row = t; break; }
                            carry = nxt;
                        }
                    }
                    row = __shfl_sync(FULL, row, L);
                    carry = __shfl_sync(FULL, carry, L);
                }
                if (row >= 0) {
                    double incl;
                    if (PRE) {
                        incl = pre[32LL * row + lane];
                    } else {   // in-row prefix of the row holding r, scanned now
                        incl = w[32LL * row + lane];
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const double t = __shfl_up_sync(FULL, incl, d);
                            if (lane >= d) incl = add(incl, t);
                        }
                    }
                    const double v = add(carry, incl);
                    l2 = __ffs(__ballot_sync(FULL, v > r)) - 1;
                    if (l2 >= 0) {
                        const double p_hi = __shfl_sync(FULL, v, l2);
                        double p_lo = __shfl_sync(FULL, v, l2 > 0 ? l2 - 1 : 0);
                        if (l2 == 0) p_lo = carry;
                        chosen = 32LL * row + l2;
                        ok = (add(p_lo, B) < r) && (add(r, B) < p_hi) && !a.force_sequential;
                    }
                }
            }
            CT_SUB(2);
            if (!ok) {
                chosen = sequential_select_warp(w, N, u, lane);
                if (lane == 0) ++rs.uncert;
                if (chosen >= 0 && chosen < N) { row = (int)(chosen >> 5); l2 = (int)(chosen & 31); }
            }
            if (lane == 0) ++rs.draws;
            if (lane == k - k0) my_choice = chosen;
            if (!(chosen >= 0 && chosen < N)) { ++k; break; }   // recorded as an error below
            // zero the drawn weight: its row's later in-row prefixes, the row
            // total, the chunk sums and the total drop by it
            const double wc = w[chosen];
            __syncwarp();
            // inclusive prefixes: the drawn configuration's own and the later ones
            if (PRE && lane >= l2) pre[32LL * row + lane] = sub(pre[32LL * row + lane], wc);
            if (lane == 0) { w[chosen] = 0.0; row_tot[row] = sub(row_tot[row], wc); }
            if (row >= t0 && row < t1) mine = sub(mine, wc);
            if (row < t1) lane_pref = sub(lane_pref, wc);
            total = __shfl_sync(FULL, lane_pref, 31);
            --positive;
            __syncwarp();
            CT_SUB(3);
        }
        const int made = k - k0;
        g.advance(jA[made], jC[made]);
        // replay lookups of the chunk's draws, one per lane
        const bool mine_in = lane < made && my_choice >= 0 && my_choice < N;
        const int64_t cs = mine_in ? my_choice : 0;
        const bool rec_ok = mine_in && a.has_record[cs];
        const double rt = a.runtime[cs];
        const bool is_stop = a.stop_bits && bit_get(a.stop_bits, cs);
        __syncwarp();
        CT_SUB(4);
        // the reference's bookkeeping (search.py:164-186), all draws of the
        // chunk at once: draw j is recorded iff no earlier draw was an error
        // or a stop; the first missing record ends the repetition unrecorded
        // (stored at out_idx[ns] as the reference's trajectory shows it), a
        // stop configuration is recorded and ends it too.  The profiled
        // candidate is the LAST draw attaining the running minimum runtime
        // (the reference's `<=`), which only matters while the repetition goes on.
        const unsigned in_chunk = made >= 32 ? FULL : ((1u << made) - 1u);
        const unsigned bad_m = __ballot_sync(FULL, lane < made && !rec_ok) & in_chunk;
        const unsigned stop_m = __ballot_sync(FULL, rec_ok && is_stop) & in_chunk & ~bad_m;
        const int first_bad = bad_m ? __ffs(bad_m) - 1 : 32;
        const int first_stop = stop_m ? __ffs(stop_m) - 1 : 32;
        const int nrec = min(made, min(first_bad, first_stop + 1));
        const int ns0 = rs.ns;
        bool fresh = false;
        if (lane < nrec) {
            out_idx[ns0 + lane] = (int32_t)my_choice;
            out_prof[ns0 + lane] = 0;
            const uint32_t m = 1u << (my_choice & 31);
            fresh = !(atomicOr(&expl[my_choice >> 5], m) & m);
        }
        const int n_fresh = __popc(__ballot_sync(FULL, fresh));
        const int64_t c_bad = __shfl_sync(FULL, (long long)my_choice, first_bad & 31);
        __syncwarp();
        if (lane == 0) {
            rs.ns = ns0 + nrec;
            rs.n_expl += n_fresh;
            if (first_bad < first_stop && first_bad < made) {
                rs.st = CT_STATUS_ERROR; rs.err = -4;
                if (rs.ns < a.max_steps) out_idx[rs.ns] = (int32_t)c_bad;
            } else if (first_stop < made) {
                rs.st = CT_STATUS_STOPPED;
            }
        }
        if (first_bad < made || first_stop < made) {
            done = 1;
        } else if (made > 0) {
            double mn = lane < made ? rt : INFINITY;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) mn = fmin(mn, __shfl_xor_sync(FULL, mn, d));
            if (mn <= t_best) {
                const unsigned at = __ballot_sync(FULL, lane < made && rt == mn);
                const int jw = 31 - __clz(at);
                const int64_t cw = __shfl_sync(FULL, (long long)my_choice, jw);
                t_best = mn;
                if (lane == 0) rs.c_prof = cw;
            }
        }
        if (!done && exhausted) {
            if (lane == 0) rs.st = CT_STATUS_EXHAUSTED;
            done = 1;
        }
        CT_SUB(5);
    }
    if (lane == 0) rs.rng.state = g.state;
    if (lane == 0) ctl.done = done;
    __syncwarp();
}

// ---------------------------------------------------------------------------
// score_top_k (search.py:133-140): only the K unexplored configurations
// nearest to the profile in Euclidean parameter distance are scored, ties in
// distance taken in index order (np.argsort(kind="stable")).  The CTA
// writes each configuration's distance as an order-preserving 64-bit key
// (the float64 bits; explored -> all ones) over its weight slots, finds the
// K-th smallest key with an 8-pass radix select (8-bit digits, shared-memory
// histograms), and builds an exclusion bitmask: explored, farther than the
// K-th key, or equal to it beyond the K - (number nearer) lowest indices.
// Eq. 16 / Eq. 17 then read that mask in place of the explored bits, so the
// pool (scoreable & ~explored) and its extrema are the reference's.  The
// weights overwrite the keys afterwards.
__host__ __device__ constexpr size_t topk_bytes(int64_t nwords) {
    return ((4 * (size_t)nwords + 15) & ~(size_t)15) + 256 * 4 + 32;
}

template <int NT>
__device__ __forceinline__ void topk_phase(const SearchArgs& a, int64_t cp, int64_t K,
                                           const uint32_t* expl, uint32_t* excl, uint32_t* hist,
                                           unsigned long long* tkv, double* w, int tid) {
    constexpr int NW = NT / 32;
    const int lane = tid & 31, warp = tid >> 5;
    const int64_t N = a.n;
    const int P = a.n_params < 64 ? a.n_params : 64;
    unsigned long long* key = reinterpret_cast<unsigned long long*>(w);
    const double* prof = a.assign + (size_t)cp * a.n_params;
    for (int64_t e = tid; e < N; e += NT) {
        unsigned long long k = ~0ull;
        if (!bit_get(expl, e)) {
            // np_row_sum (ct_hd.cuh) of the squared differences, streamed:
            // the eight pairwise accumulators stay in registers
            const double* row = a.assign + (size_t)e * a.n_params;
            auto sq = [&](int j) {
                const double d = sub(__ldg(row + j), __ldg(prof + j));
                return mul(d, d);
            };
            double res;
            if (P < 8) {
                res = -0.0;
                for (int j = 0; j < P; ++j) res = add(res, sq(j));
            } else {
                double r[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = sq(j);
                int i = 8;
                for (; i < P - (P % 8); i += 8) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) r[j] = add(r[j], sq(i + j));
                }
                res = add(add(add(r[0], r[1]), add(r[2], r[3])), add(add(r[4], r[5]), add(r[6], r[7])));
                for (; i < P; ++i) res = add(res, sq(i));
            }
            k = (unsigned long long)dbits(dsqrt(res));   // >= 0: bits order as values
        }
        key[e] = k;
    }
    unsigned long long prefix = 0, mask = 0;
    unsigned long long krem = (unsigned long long)K;      // rank wanted among the matching keys
    unsigned long long cnt_eq = 0;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += NT) hist[i] = 0u;
        __syncthreads();
        for (int64_t e = tid; e < N; e += NT) {
            const unsigned long long k = key[e];
            if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            unsigned c[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { c[j] = hist[8 * lane + j]; sum += c[j]; }
            unsigned incl = sum;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned v = __shfl_up_sync(FULL, incl, d);
                if (lane >= d) incl += v;
            }
            const int L = __ffs(__ballot_sync(FULL, incl >= krem)) - 1;   // K <= pool: exists
            if (lane == L) {
                unsigned long long cum = incl - sum;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (cum + c[j] >= krem) {
                        tkv[0] = prefix | ((unsigned long long)(8 * lane + j) << shift);
                        tkv[1] = krem - cum;
                        tkv[2] = c[j];
                        break;
                    }
                    cum += c[j];
                }
            }
        }
        __syncthreads();
        prefix = tkv[0];
        krem = tkv[1];
        cnt_eq = tkv[2];
        mask |= 255ull << shift;
    }
    // prefix is the K-th smallest key; krem of the cnt_eq keys equal to it
    // are in (the lowest indices)
    const bool all_eq = cnt_eq == krem;
    for (int64_t t = warp; t < a.nwords; t += NW) {
        const int64_t e = 32 * t + lane;
        const unsigned long long k = e < N ? key[e] : ~0ull;
        const unsigned word = __ballot_sync(FULL, k > prefix || (k == prefix && !all_eq));
        if (lane == 0) excl[t] = word;
    }
    __syncthreads();
    if (!all_eq && warp == 0) {
        unsigned long long carry = 0;
        for (int64_t t = 0; t < a.nwords && carry < krem; ++t) {
            const int64_t e = 32 * t + lane;
            const bool eq = e < N && key[e] == prefix;
            const unsigned bal = __ballot_sync(FULL, eq);
            if (!bal) continue;
            const unsigned long long rank = carry + __popc(bal & ((1u << lane) - 1u));
            const unsigned in = __ballot_sync(FULL, eq && rank < krem);
            if (lane == 0) excl[t] &= ~in;
            carry += __popc(bal);
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// k_profile_search: one CTA runs one repetition end to end (then the next one
// of its persistent slice); the serial phases run on warp 0 while the other
// warps wait at the CTA barrier.
template <int NT, bool SMEM, bool PRE, bool TOPK, bool HG = false>
__global__ void __launch_bounds__(NT, (NT <= 64) ? 8 : ((NT == 128) ? 7 : (896 / NT)))
k_profile_search(const SearchArgs a) {
    static_assert(!HG || (!SMEM && !TOPK), "global row index: weights in global scratch, no top-K");
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ Ctl<NW> ctl;
    __shared__ RepState rs;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    __shared__ uint32_t seed_sh[SEED_INLINE_WORDS];
    // PCG64 jump-ahead tables: k steps = (A_k, C_k), k = 0..32
    __shared__ u128 jA[33], jC[33];
    if (tid == 0) Pcg64::jump_tables(jA, jC, 32);
    load_seed_words(a.seed, seed_sh);

    // dynamic shared memory: row totals | explored bits | [top-K: exclusion
    // bits | radix histogram | select state] | [weights | in-row prefixes]
    const size_t head = (16 * (size_t)a.nrows + 4 * (size_t)a.nwords + 15) & ~(size_t)15;
    // HG (spaces whose row index outgrows shared memory, >~ 300k
    // configurations): row totals and explored bits in a per-CTA slice of
    // global scratch as well
    unsigned char* head_base = HG ? reinterpret_cast<unsigned char*>(a.scratch_head) +
                                        (size_t)blockIdx.x * head
                                  : smem;
    double* row_tot = reinterpret_cast<double*>(head_base);
    uint32_t* expl = reinterpret_cast<uint32_t*>(head_base + 16 * (size_t)a.nrows);
    const size_t tk_b = TOPK ? topk_bytes(a.nwords) : 0;
    uint32_t* excl_k = reinterpret_cast<uint32_t*>(smem + head);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + head + ((4 * (size_t)a.nwords + 15) & ~(size_t)15));
    unsigned long long* tkv = reinterpret_cast<unsigned long long*>(hist + 256);
    double* w;
    if (SMEM) {
        w = reinterpret_cast<double*>(smem + head + tk_b);
    } else {
        w = a.scratch_w + (size_t)blockIdx.x * 64 * (size_t)a.nrows;
    }
    double* pre = w + 32 * (size_t)a.nrows;

#ifdef CT_PHASE_CLOCKS
    long long clk_p1 = 0, clk_score = 0, clk_weight = 0, clk_p4 = 0, clk_t = 0;
#define CT_CLK(acc) do { if (tid == 0) { long long n_ = clock64(); acc += n_ - clk_t; clk_t = n_; } } while (0)
#else
#define CT_CLK(acc) do { } while (0)
#endif
    const int pcol = (lane < N_COMP) ? a.delta_col[lane] : -1;
    for (int rep = blockIdx.x; rep < a.n_reps; rep += gridDim.x) {
        int32_t* out_idx = a.step_index + (size_t)rep * a.max_steps;
        uint8_t* out_prof = a.step_profiled + (size_t)rep * a.max_steps;
        if (warp == 0) rep_begin(a, seed_sh, rep, rs, ctl, expl, lane);
        __syncthreads();

        // warp 0 runs the draws and, without a CTA barrier in between, the
        // next iteration's profile step (the other warps have nothing to do)
#ifdef CT_PHASE_CLOCKS
        if (tid == 0) clk_t = clock64();
#endif
        if (warp == 0 && a.outer > 0) profile_step(a, rs, ctl, expl, out_idx, out_prof, lane, pcol);
        __syncthreads();
        CT_CLK(clk_p1);
        for (int it = 0; it < a.outer; ++it) {
            if (ctl.done) break;
            const uint32_t* excl = expl;     // configurations outside the pool
            if constexpr (TOPK) {
                if (a.topk < a.n - rs.n_expl) {
                    if (a.topk == 0) {
                        // an empty pool: normalize_scores raises (search.py:155)
                        if (tid == 0) { rs.st = CT_STATUS_ERROR; rs.err = -3; }
                        break;
                    }
                    topk_phase<NT>(a, rs.c_prof, a.topk, expl, excl_k, hist, tkv, w, tid);
                    excl = excl_k;
                }
            }
            score_phase<NT>(a, ctl, excl, w, tid);
            __syncthreads();
            CT_CLK(clk_score);
            weight_phase<PRE>(a, ctl, excl, w, pre, row_tot, warp);
            __syncthreads();
            CT_CLK(clk_weight);
            if (warp == 0) {
                draw_step<PRE, NW, (NT >= 512)>(a, rs, ctl, expl, w, pre, row_tot, jA, jC, out_idx,
                                                out_prof, lane);
                CT_CLK(clk_p4);
                if (!ctl.done && it + 1 < a.outer)
                    profile_step(a, rs, ctl, expl, out_idx, out_prof, lane, pcol);
            }
            __syncthreads();
            CT_CLK(clk_p1);
        }
        if (tid == 0) rep_end(a, rep, rs);
        __syncthreads();
    }
#ifdef CT_PHASE_CLOCKS
    if (tid == 0 && (blockIdx.x % 37) == 0)
        printf("[clk] cta %d: profile+expert %lld score %lld weights %lld draws %lld cycles\n",
               blockIdx.x, clk_p1, clk_score, clk_weight, clk_p4);
    if (tid == 0 && blockIdx.x == 0)
        printf("[clk-draw] all CTAs so far: setup %llu jump-ahead %llu locate %llu zero %llu "
               "lookup %llu bookkeeping %llu\n", g_subclk[0], g_subclk[1], g_subclk[2],
               g_subclk[3], g_subclk[4], g_subclk[5]);
#endif
}

// ---------------------------------------------------------------------------
// k_profile_search_ws: warp-specialised, two repetitions per CTA.
//
// In k_profile_search the serial phases (profile step + expert system, the n
// draws) keep NW-1 warps idle at the CTA barrier.  Here warp 0 is the serial
// warp and warps 1..PW the parallel warps, and the CTA interleaves two
// repetitions (slots 0 and 1): while the serial warp runs slot s's draws and
// its next profile step, the parallel warps score and weight slot s^1.
// Hand-off through named barriers (bar.arrive by the producer, bar.sync by
// the consumer; both order shared-memory accesses):
//   READY_s (1 + s): the serial warp has set up slot s (ctl[s].cmd says
//                    RUN / SKIP / EXIT)
//   DONE_s  (3 + s): the parallel warps have finished slot s
//   barrier 5      : among the parallel warps, between Eq. 16 and Eq. 17
// Every repetition executes exactly the phases k_profile_search executes,
// in the same order, so its trajectory is identical.
enum : int { WS_RUN = 0, WS_SKIP = 1, WS_EXIT = 2 };

__device__ __forceinline__ void bar_sync_n(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int PW, bool SMEM>
__global__ void __launch_bounds__(32 * (PW + 1), (PW <= 4) ? 4 : (PW <= 6 ? 4 : 3))
k_profile_search_ws(const SearchArgs a) {
    constexpr int PT = 32 * PW, NTT = PT + 32;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ Ctl<PW> ctl[2];
    __shared__ RepState rs[2];
    __shared__ uint32_t seed_sh[SEED_INLINE_WORDS];
    __shared__ u128 jA[33], jC[33];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) Pcg64::jump_tables(jA, jC, 32);
    load_seed_words(a.seed, seed_sh);      // ends with __syncthreads()

    // dynamic shared memory, per slot: row totals | explored bits |
    // [weights | in-row prefixes]
    const size_t head = (16 * (size_t)a.nrows + 4 * (size_t)a.nwords + 15) & ~(size_t)15;
    const size_t per_slot = head + (SMEM ? 16 * 32 * (size_t)a.nrows : 0);
    double* row_tot[2];
    uint32_t* expl[2];
    double* w[2];
    double* pre[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        unsigned char* base = smem + per_slot * s;
        row_tot[s] = reinterpret_cast<double*>(base);
        expl[s] = reinterpret_cast<uint32_t*>(base + 16 * (size_t)a.nrows);
        w[s] = SMEM ? reinterpret_cast<double*>(base + head)
                    : a.scratch_w + (size_t)(2 * blockIdx.x + s) * 64 * (size_t)a.nrows;
        pre[s] = w[s] + 32 * (size_t)a.nrows;
    }
    const int stride = 2 * gridDim.x;

    if (warp == 0) {
        // ------------------------------ serial warp ------------------------
        int rep[2] = {0, 0}, it[2] = {-1, -1};
        const int pcol = (lane < N_COMP) ? a.delta_col[lane] : -1;
#ifdef CT_PHASE_CLOCKS
        long long clk_wait = 0, clk_work = 0, clk_t = clock64();
#endif
        // set up slot s with its next repetition that still has a parallel
        // phase to run (a repetition can end at its first profile step)
        auto next_run = [&](int s) {
            while (rep[s] < a.n_reps) {
                int32_t* out_idx = a.step_index + (size_t)rep[s] * a.max_steps;
                uint8_t* out_prof = a.step_profiled + (size_t)rep[s] * a.max_steps;
                if (it[s] < 0) { rep_begin(a, seed_sh, rep[s], rs[s], ctl[s], expl[s], lane); it[s] = 0; }
                profile_step(a, rs[s], ctl[s], expl[s], out_idx, out_prof, lane, pcol);
                if (!ctl[s].done) { if (lane == 0) ctl[s].cmd = WS_RUN; __syncwarp(); return; }
                if (lane == 0) rep_end(a, rep[s], rs[s]);
                rep[s] += stride; it[s] = -1;
            }
            if (lane == 0) ctl[s].cmd = WS_SKIP;
            __syncwarp();
        };
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            rep[s] = 2 * blockIdx.x + s; it[s] = -1;
            next_run(s);
            bar_arrive_n(1 + s, NTT);
        }
        int cur = 0;
        for (;;) {
#ifdef CT_PHASE_CLOCKS
            long long t_ = clock64(); clk_work += t_ - clk_t; clk_t = t_;
#endif
            bar_sync_n(3 + cur, NTT);
#ifdef CT_PHASE_CLOCKS
            t_ = clock64(); clk_wait += t_ - clk_t; clk_t = t_;
#endif
            if (ctl[cur].cmd == WS_RUN) {
                int32_t* out_idx = a.step_index + (size_t)rep[cur] * a.max_steps;
                uint8_t* out_prof = a.step_profiled + (size_t)rep[cur] * a.max_steps;
                draw_step<true>(a, rs[cur], ctl[cur], expl[cur], w[cur], pre[cur], row_tot[cur], jA, jC,
                          out_idx, out_prof, lane);
                ++it[cur];
                if (ctl[cur].done || it[cur] >= a.outer) {
                    if (lane == 0) rep_end(a, rep[cur], rs[cur]);
                    rep[cur] += stride; it[cur] = -1;
                }
                next_run(cur);
            }
            if (ctl[0].cmd == WS_SKIP && ctl[1].cmd == WS_SKIP) {
                if (lane == 0) ctl[cur].cmd = WS_EXIT;
                __syncwarp();
                bar_arrive_n(1 + cur, NTT);
                bar_sync_n(3 + (cur ^ 1), NTT);
                break;
            }
            bar_arrive_n(1 + cur, NTT);
            cur ^= 1;
        }
#ifdef CT_PHASE_CLOCKS
        if (lane == 0 && (blockIdx.x % 37) == 0)
            printf("[clk-ws] cta %d: serial warp busy %lld waiting %lld cycles\n", blockIdx.x,
                   clk_work, clk_wait);
#endif
    } else {
        // ------------------------------ parallel warps ---------------------
        const int ptid = tid - 32, pw = warp - 1;
        int cur = 0;
#ifdef CT_PHASE_CLOCKS
        long long clk_wait = 0, clk_work = 0, clk_t = clock64();
#endif
        for (;;) {
            bar_sync_n(1 + cur, NTT);
#ifdef CT_PHASE_CLOCKS
            long long t_ = clock64(); clk_wait += t_ - clk_t; clk_t = t_;
#endif
            const int cmd = ctl[cur].cmd;
            if (cmd == WS_EXIT) break;
            if (cmd == WS_RUN) {
                score_phase<PT>(a, ctl[cur], expl[cur], w[cur], ptid);
                bar_sync_n(5, PT);
                weight_phase<true>(a, ctl[cur], expl[cur], w[cur], pre[cur], row_tot[cur], pw);
            }
#ifdef CT_PHASE_CLOCKS
            t_ = clock64(); clk_work += t_ - clk_t; clk_t = t_;
#endif
            bar_arrive_n(3 + cur, NTT);
            cur ^= 1;
        }
#ifdef CT_PHASE_CLOCKS
        if (tid == 32 && (blockIdx.x % 37) == 0)
            printf("[clk-ws] cta %d: parallel warps busy %lld waiting %lld cycles\n", blockIdx.x,
                   clk_work, clk_wait);
#endif
    }
}

// ---------------------------------------------------------------------------
// run_random_search (search.py:317-335): one thread per repetition shuffles
// arange(N) with numpy's Fisher-Yates (random_interval) in a scratch slice and
// emits the prefix up to the first stop configuration.
struct RandomArgs {
    int64_t n;
    const uint8_t* has_record;
    const uint32_t* stop_bits;     // nullable
    int64_t max_steps_req;         // < 0: None
    SeedInline seed;
    int32_t n_reps;
    int32_t* perm_scratch;         // n_slots * n
    int32_t n_slots;
    int32_t* step_index;
    uint8_t* step_profiled;
    int64_t max_steps;
    int32_t* n_steps;
    int32_t* status;
    int32_t* rep_error;
};

__global__ void k_random_search(const RandomArgs a) {
    __shared__ uint32_t seed_sh[SEED_INLINE_WORDS];
    load_seed_words(a.seed, seed_sh);
    for (int rep = blockIdx.x * blockDim.x + threadIdx.x; rep < a.n_reps;
         rep += gridDim.x * blockDim.x) {
        int slot = (blockIdx.x * blockDim.x + threadIdx.x);
        int32_t* perm = a.perm_scratch + (size_t)slot * a.n;
        const int64_t N = a.n;
        Pcg64 rng;
        rng.seed(seed_pool(seed_words_of(a.seed, seed_sh, rep)));
        for (int64_t i = 0; i < N; ++i) perm[i] = (int32_t)i;
        for (int64_t i = N - 1; i > 0; --i) {
            int64_t j = (int64_t)rng.interval((uint64_t)i);
            int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
        }
        int64_t lim = N;
        if (a.max_steps_req >= 0 && a.max_steps_req < N) lim = a.max_steps_req;
        int st = (a.max_steps_req < 0 || a.max_steps_req >= N) ? CT_STATUS_EXHAUSTED : CT_STATUS_BUDGET;
        int err = 0;
        int64_t ns = 0;
        int32_t* out_idx = a.step_index + (size_t)rep * a.max_steps;
        uint8_t* out_prof = a.step_profiled + (size_t)rep * a.max_steps;
        for (int64_t pos = 0; pos < lim; ++pos) {
            int32_t idx = perm[pos];
            if (!a.has_record[idx]) { st = CT_STATUS_ERROR; err = -4; out_idx[ns] = idx; break; }
            out_idx[ns] = idx; out_prof[ns] = 0; ++ns;
            if (a.stop_bits && bit_get(a.stop_bits, idx)) { st = CT_STATUS_STOPPED; break; }
        }
        a.n_steps[rep] = (int32_t)ns;
        a.status[rep] = st;
        a.rep_error[rep] = err;
    }
}

}  // namespace ct
