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

// The same re-decision by one warp, for large spaces: lane 0 still performs
// every add of np.cumsum in order, while the whole warp fetches the weights
// (one coalesced 32-element chunk per load, four chunks ahead) and hands
// them to lane 0 by shuffle, so the chain runs at the add latency instead of
// a dependent load per element.  The running sum before every per-th chunk
// is kept as a checkpoint (<= 256, eight per lane), so finding r needs one
// interval of the second pass instead of the whole array.  Returns the same
// index as sequential_select.
__device__ __forceinline__ double seq_fetch(const double* w, int64_t n, int64_t ch, int lane) {
    const int64_t e = ch * 32 + lane;
    return (e < n) ? w[e] : 0.0;
}

__device__ __noinline__ int64_t sequential_select_warp(const double* w, int64_t n, double u, int lane) {
    constexpr int CK = 8;
    const int64_t nchunks = (n + 31) / 32;
    const int64_t per = max((int64_t)1, (nchunks + 32 * CK - 1) / (32 * CK));
    double ck[CK];
#pragma unroll
    for (int s = 0; s < CK; ++s) ck[s] = 0.0;
    double c = 0.0;                  // lane 0's running sum (+0.0 padding adds are exact)
    double v[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) v[d] = seq_fetch(w, n, d, lane);
    for (int64_t k = 0; k < nchunks; k += 4) {
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int64_t ch = k + d;
            if (ch < nchunks) {
                if (ch % per == 0) {
                    const int64_t slot = ch / per;
                    const double cb = __shfl_sync(FULL, c, 0);
#pragma unroll
                    for (int s = 0; s < CK; ++s)
                        if (slot == 32 * s + lane) ck[s] = cb;
                }
                const double x = v[d];
                v[d] = seq_fetch(w, n, ch + 4, lane);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const double xj = __shfl_sync(FULL, x, j);
                    if (lane == 0) c = add(c, xj);
                }
            }
        }
    }
    const double total = __shfl_sync(FULL, c, 0);
    const double r = mul(u, total);
    // the last checkpoint at or below r (slot 0 holds 0 <= r)
    const int64_t nslots = (nchunks + per - 1) / per;
    int64_t best = -1;
    double from = 0.0;
#pragma unroll
    for (int s = 0; s < CK; ++s) {
        const int64_t slot = 32 * s + lane;
        if (slot < nslots && ck[s] <= r && slot > best) { best = slot; from = ck[s]; }
    }
    int64_t slot = best;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) slot = max(slot, (int64_t)__shfl_xor_sync(FULL, (long long)slot, m));
    if (slot < 0) slot = 0;
    const int owner = (int)(slot & 31);
    c = __shfl_sync(FULL, from, owner);      // the owner's best is this slot
    int64_t found = n;
#pragma unroll
    for (int d = 0; d < 4; ++d) v[d] = seq_fetch(w, n, slot * per + d, lane);
    for (int64_t k = slot * per; k < nchunks; k += 4) {
        bool done = false;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int64_t ch = k + d;
            if (ch < nchunks && !done) {
                const double x = v[d];
                v[d] = seq_fetch(w, n, ch + 4, lane);
                int hit = -1;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const double xj = __shfl_sync(FULL, x, j);
                    if (lane == 0 && hit < 0) {
                        c = add(c, xj);
                        if (c > r) hit = j;
                    }
                }
                hit = __shfl_sync(FULL, hit, 0);
                if (hit >= 0) {
                    found = min(n, ch * 32 + hit);
                    done = true;
                }
            }
        }
        if (done) break;
    }
    return found;
}

}  // namespace ct
