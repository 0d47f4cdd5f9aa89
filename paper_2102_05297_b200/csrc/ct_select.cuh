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

// The same re-decision by one warp, for large spaces, without a chain of N
// dependent adds.  np.cumsum's running value c_k = fl(c_(k-1) + w_k) is
// emulated EXACTLY in integer arithmetic while c stays in one binade
// [2^E, 2^(E+1)): there c = g C with the grid g = 2^(E-52) and an integer
// C in [2^52, 2^53), and for w >= 0 with c + w still below 2^(E+1),
// fl(c + w) = g (C + n), n = round-to-nearest-even(w / g) -- w / g is an
// exact power-of-two scaling, and n does not depend on C unless w / g is a
// tie (fraction exactly 1/2, parity of C decides).  So a block of 256
// weights (8 per lane) is one exact int64 warp scan of the n's; the first
// element whose sum would leave the binade (C + n >= 2^53), or is a tie, or
// (c = 0) starts the sum, is added by the hardware's own fl add instead,
// and the scan resumes after it in the new binade.  Every c_k is therefore
// bit-identical to the sequential loop's, at ~1-2 cycles per element
// instead of one add latency.
//
// seq_scan: from element k0 with running value c (c_(k0-1)), through n
// elements, stopping at the first k with c_k > r (r < 0: never); returns k
// (n if none) and leaves c = c_(k) / c_(n-1).
__device__ __forceinline__ double pow2d(int e) {          // 2^e, e in [-1022, 1023]
    return bitsd((uint64_t)(1023 + e) << 52);
}

constexpr int SEQ_EPL = 16, SEQ_BLK = 32 * SEQ_EPL;  // elements per lane, per block
constexpr int SEQ_CK = 8;                          // checkpoints per lane (256 in all)

// increment of one element in the binade grid (see above); stop = the
// element must take the hardware's fl add (a tie, alone past the binade, or
// the first nonzero while c = 0)
__device__ __forceinline__ int64_t seq_inc(double x, bool lin, double to_grid, bool& stop) {
    // n = round-to-nearest-even(x / g) without a float-to-integer
    // conversion (slow on the FP64 units): t + 2^52 rounds t to an integer
    // (RNE) for 0 <= t < 2^52 and holds it in its low mantissa bits.
    // Branch-free (lin is warp-uniform, but the selects keep the unrolled
    // block loop straight-line).
    const double t = x * to_grid;                                // exact
    const double big = 4503599627370496.0;                       // 2^52
    const double s = t + big;
    const double rne = s - big;                                  // exact
    const double d = t - rne;                                    // exact, |d| <= 1/2
    stop = lin ? ((t >= big) | (fabs(d) == 0.5)) : (x != 0.0);   // too large, a tie; or c = 0
    return lin ? (int64_t)(dbits(s) & ((1ull << 52) - 1)) : 0;
}

// ck / per: with ck != nullptr the running value at the start of every
// per-th block is kept (lane L, slot s: block (32 s + L) per).
//
// A block's common path is one increment per element, one exact int64 warp
// scan of the lane totals and one ballot: an event -- a stop, leaving the
// binade, passing r -- can only lie in the first lane whose running total
// shows one (the increments are >= 0), and only that lane then walks its
// elements to find it.
__device__ __forceinline__ int64_t seq_scan(const double* w, int64_t n, int64_t k0, double& c,
                                            double r, int lane, double* ck = nullptr,
                                            int64_t per = 1) {
    constexpr int EPL = SEQ_EPL, BLK = SEQ_BLK;
    const int64_t TWO53 = 1ll << 53;
    // this lane's EPL weights of a block: elements base + EPL lane + j (0.0
    // outside [k0, n): adding +0.0 is exact and never an event); the next
    // block's are fetched while this one is scanned
    auto fetch = [&](int64_t base, double* x) {
        if (base >= k0 && base + BLK <= n) {            // a whole block: 8 x 16-byte loads
            const double2* q = reinterpret_cast<const double2*>(w + base + EPL * lane);
#pragma unroll
            for (int j = 0; j < EPL / 2; ++j) { const double2 v = q[j]; x[2 * j] = v.x; x[2 * j + 1] = v.y; }
        } else {
#pragma unroll
            for (int j = 0; j < EPL; ++j) {
                const int64_t e = base + EPL * lane + j;
                x[j] = (e >= k0 && e < n) ? w[e] : 0.0;
            }
        }
    };
    double xn[EPL];
    const int64_t first = k0 & ~(int64_t)(BLK - 1);
    fetch(first, xn);
    int64_t blk = first / BLK, next_ck = 0, slot = 0;   // checkpoint bookkeeping, no division
    // the next block's lane total and stop flag, computed while this block's
    // scan is in flight, under this block's binade (key: E, or -9999 for
    // c = 0); reused when the next block starts in the same binade
    int spec_key = 0x7fffffff;
    int64_t spec_run = 0;
    bool spec_st = false;
    int rint_key = 0x7fffffff;
    int64_t Rint = (int64_t)1 << 62;
    for (int64_t base = first; base < n; base += BLK, ++blk) {
        double x[EPL];
#pragma unroll
        for (int j = 0; j < EPL; ++j) x[j] = xn[j];
        fetch(base + BLK, xn);
        {
            // one warp streams the weights: each lane also pulls its 128-byte
            // segment of the block 16 ahead into L2
            const int64_t e = base + 16 * (int64_t)BLK + EPL * lane;
            if (e < n) asm volatile("prefetch.L2 [%0];" ::"l"(w + e));   // generic: w may be shared memory
        }
        if (ck && blk == next_ck) {
#pragma unroll
            for (int q = 0; q < SEQ_CK; ++q)
                if (slot == 32 * q + lane) ck[q] = c;        // c is warp-uniform here
            ++slot;
            next_ck += per;
        }
        const int64_t mine0 = base + EPL * lane;
        bool fresh = true;                  // no event yet in this block
        for (;;) {
            // binade state of c; c == 0 (or subnormal): every nonzero element
            // is a scalar step until the sum is normal
            const bool lin = c >= 2.2250738585072014e-308;
            const int E = lin ? (int)((dbits(c) >> 52) & 0x7ff) - 1023 : 0;
            const int64_t C = lin ? (int64_t)((dbits(c) & ((1ull << 52) - 1)) | (1ull << 52)) : 0;
            const double to_grid = lin ? pow2d(52 - E) : 0.0, from_grid = lin ? pow2d(E - 52) : 0.0;
            // c_k > r  <=>  C_k > floor(r / g) (C_k integer); r / g exact.
            // Recomputed only when the binade changes (the float-to-integer
            // conversion is slow, and the binade changes ~40 times in a pass)
            const int key = lin ? E : -9999;
            if (key != rint_key) {
                const double rg = (lin && r >= 0.0) ? r * to_grid : 1.0e300;
                Rint = (rg < 9007199254740992.0) ? (int64_t)floor(rg) : (int64_t)1 << 62;
                rint_key = key;
            }
            int64_t run = 0;
            bool st_any = false;
            if (fresh && key == spec_key) {
                run = spec_run;
                st_any = spec_st;
            } else {
#pragma unroll
                for (int j = 0; j < EPL; ++j) {
                    bool sj = false;
                    run += seq_inc(x[j], lin, to_grid, sj);
                    st_any |= sj;
                }
            }
            if (fresh) {                            // speculate the next block
                spec_key = key;
                spec_run = 0;
                spec_st = false;
#pragma unroll
                for (int j = 0; j < EPL; ++j) {
                    bool sj = false;
                    spec_run += seq_inc(xn[j], lin, to_grid, sj);
                    spec_st |= sj;
                }
            }
            int64_t incl = run;                     // exact int64 warp scan
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int64_t v = __shfl_up_sync(FULL, (long long)incl, d);
                if (lane >= d) incl += v;
            }
            const bool leave = lin && C + incl >= TWO53;
            const bool hit = lin && C + incl > Rint;
            const unsigned bal = __ballot_sync(FULL, st_any || leave || hit);
            if (!bal) {                             // the rest of the block stays in the binade
                if (lin) c = (double)(C + __shfl_sync(FULL, (long long)incl, 31)) * from_grid;
                break;
            }
            // the first flagged lane walks its elements to the event
            const int L = __ffs(bal) - 1;
            int kind = 0, jev = EPL;                // kind: 1 stop, 2 hit
            int64_t pre = 0;                        // increments before the event
            if (lane == L) {
                int64_t acc = incl - run;           // exclusive prefix of this lane
#pragma unroll
                for (int j = 0; j < EPL; ++j) {
                    if (kind == 0) {
                        bool sj = false;
                        const int64_t nj = seq_inc(x[j], lin, to_grid, sj);
                        if (sj || (lin && C + acc + nj >= TWO53)) {
                            kind = 1; jev = j; pre = acc;
                        } else if (lin && C + acc + nj > Rint) {
                            kind = 2; jev = j;
                        } else {
                            acc += nj;
                        }
                    }
                }
            }
            kind = __shfl_sync(FULL, kind, L);
            jev = __shfl_sync(FULL, jev, L);
            pre = __shfl_sync(FULL, (long long)pre, L);
            const int64_t p = base + EPL * L + jev;
            if (kind == 2) return p;                // c_p > r inside the binade
            // kind == 1: the elements before p are final, then the hardware add
            if (lin) c = (double)(C + pre) * from_grid;
            c = add(c, w[p]);
            if (r >= 0.0 && c > r) return p;
            // the elements up to p are added: they no longer take part
#pragma unroll
            for (int j = 0; j < EPL; ++j)
                if (mine0 + j <= p) x[j] = 0.0;
            fresh = false;
        }
    }
    return n;
}

// np.cumsum + searchsorted(side='right') by one warp: the total, r = u c_N,
// then the first k with c_k > r (n when r reaches the total).
__device__ __noinline__ int64_t sequential_select_warp(const double* w, int64_t n, double u, int lane) {
    // pass 1: the total, keeping the exact running value at <= 256 block
    // boundaries; pass 2 starts from the last boundary at or below r
    const int64_t nblocks = (n + SEQ_BLK - 1) / SEQ_BLK;
    const int64_t per = max((int64_t)1, (nblocks + 32 * SEQ_CK - 1) / (32 * SEQ_CK));
    double ck[SEQ_CK];
#pragma unroll
    for (int q = 0; q < SEQ_CK; ++q) ck[q] = 0.0;
    double c = 0.0;
    seq_scan(w, n, 0, c, -1.0, lane, ck, per);
    const double r = mul(u, c);
    const int64_t nslots = (nblocks + per - 1) / per;
    int64_t best = 0;
    double from = 0.0;
#pragma unroll
    for (int q = 0; q < SEQ_CK; ++q) {
        const int64_t slot = 32 * q + lane;
        if (slot < nslots && ck[q] <= r && slot > best) { best = slot; from = ck[q]; }
    }
    int64_t slot = best;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) slot = max(slot, (int64_t)__shfl_xor_sync(FULL, (long long)slot, m));
    double c2 = __shfl_sync(FULL, from, (int)(slot & 31));   // the owner's best is this slot
    if (slot == 0) c2 = 0.0;
    return seq_scan(w, n, slot * per * SEQ_BLK, c2, r, lane);
}

}  // namespace ct
