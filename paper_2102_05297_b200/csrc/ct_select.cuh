// ct_select.cuh -- certified inverse-CDF draw (weighted_select, search.py:175-185).
//
// The reference draws r = u * cumsum(w)[-1] and returns the first index whose
// *sequential* float64 cumsum exceeds r.  On the device the weights are
// summed exactly (2^-66 fixed point, so the prefix is associative and can be
// taken in any order), the index is located with two warp scans (tile totals,
// then the 32-element rows of the hit tile), and the decision is certified:
// if r sits farther from both neighbouring prefix boundaries than the
// worst-case disagreement between the exact prefix and the reference's
// sequential float prefix (incl. a 1-ulp pow difference per weight), both
// pick the same index.  Otherwise the draw is re-decided with the sequential
// float64 cumsum itself.
#pragma once
#include "ct_warp.cuh"

namespace ct {

struct Located {
    int64_t idx;      // chosen configuration (-1: r beyond the exact total)
    int tile;
    u128 before;      // exact prefix strictly before idx
    u128 wfx;         // fixed-point weight of idx
};

// In-tile part of a draw (one full warp): rows of 32 consecutive elements,
// one exact warp scan per row until the row containing r is found.  carry
// is the exact prefix before the tile.
__device__ __forceinline__ Located warp_locate_rows(int tile, u128 carry, const double* w,
                                                    int64_t n, int rows, u128 r_fx, int lane) {
    Located out;
    out.idx = -1; out.tile = -1; out.before = 0; out.wfx = 0;
    const int64_t base = (int64_t)tile * (32LL * rows);
    for (int j = 0; j < rows; ++j) {
        int64_t e = base + 32LL * j + lane;
        double wv = (e < n) ? w[e] : 0.0;
        u128 f = 0;
        to_fx(wv, &f);
        u128 in = warp_incl_scan(f, lane);
        u128 tot = shfl_u128(in, 31);
        if (carry + tot > r_fx) {
            unsigned b2 = __ballot_sync(FULL, carry + in > r_fx);
            int l2 = __ffs(b2) - 1;
            out.before = carry + shfl_u128(in - f, l2);
            out.wfx = shfl_u128(f, l2);
            out.idx = base + 32LL * j + l2;
            out.tile = tile;
            return out;
        }
        carry += tot;
    }
    return out;
}

// Tile part with a per-lane inclusive prefix kept by the caller: lane L owns
// tiles [t0, t1) (a contiguous chunk), mine is their exact sum and
// lane_pref the inclusive prefix over lanes.  A ballot finds the lane whose
// chunk holds r, that lane walks its chunk.
__device__ __forceinline__ Located warp_locate_pref(const u128* tile_tot, int t0, int t1,
                                                    u128 lane_pref, u128 mine, const double* w,
                                                    int64_t n, int rows, u128 r_fx, int lane) {
    unsigned bal = __ballot_sync(FULL, lane_pref > r_fx);
    if (bal == 0) {
        Located out;
        out.idx = -1; out.tile = -1; out.before = 0; out.wfx = 0;
        return out;
    }
    int L = __ffs(bal) - 1;
    int tile = -1;
    u128 carry = lane_pref - mine;
    if (lane == L) {
        for (int t = t0; t < t1; ++t) {
            u128 nxt = carry + tile_tot[t];
            if (nxt > r_fx) { tile = t; break; }
            carry = nxt;
        }
    }
    tile = __shfl_sync(FULL, tile, L);
    carry = shfl_u128(carry, L);
    return warp_locate_rows(tile, carry, w, n, rows, r_fx, lane);
}

// Stateless form (single-call API): the lane prefix is built on the spot.
__device__ __forceinline__ Located warp_locate(const u128* tile_tot, int ntiles,
                                               const double* w, int64_t n, int rows,
                                               u128 r_fx, int lane) {
    int cpl = (ntiles + 31) >> 5;
    int t0 = lane * cpl;
    int t1 = min(t0 + cpl, ntiles);
    u128 mine = 0;
    for (int t = t0; t < t1; ++t) mine += tile_tot[t];
    u128 incl = warp_incl_scan(mine, lane);
    return warp_locate_pref(tile_tot, t0, t1, incl, mine, w, n, rows, r_fx, lane);
}

// Certification: |c_seq(i) - S(i)| + |r_ref - r| <= (2N + 7) 2^-53 T for the
// reference's sequential prefix c_seq over weights within 1 ulp of ours
// (SURVEY hard part 3); 16 instead of 7 leaves slack for a pow8 that misses
// correct rounding by a hair.
__device__ __forceinline__ bool certify(const Located& p, u128 r_fx, double total_d, int64_t n) {
    if (p.idx < 0) return false;
    double bound = (double)(2 * n + 16) * 1.1102230246251565e-16 * total_d;   // 2^-53
    u128 b_fx = floor_fx(bound) + 1;
    u128 lo = r_fx - p.before;                       // r_fx >= before
    u128 after = p.before + p.wfx;                   // > r_fx
    u128 hi = after - r_fx - 1;
    return lo > b_fx && hi > b_fx;
}

// Sequential float64 re-decision (np.cumsum + searchsorted 'right'), one
// thread.  Returns n when r reaches the total (the reference would then index
// past the end).
__device__ __noinline__ int64_t sequential_select(const double* w, int64_t n, double u) {
    double c = 0.0;
    for (int64_t i = 0; i < n; ++i) c = add(c, w[i]);
    double r = mul(u, c);
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        s = add(s, w[i]);
        if (s > r) return i;
    }
    return n;
}

}  // namespace ct
