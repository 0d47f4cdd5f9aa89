// ct_warp.cuh -- warp / block primitives on 128-bit fixed-point sums.
#pragma once
#include "ct_hd.cuh"

namespace ct {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ u128 shfl_u128(u128 v, int src) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    lo = __shfl_sync(FULL, lo, src);
    hi = __shfl_sync(FULL, hi, src);
    return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ u128 shfl_up_u128(u128 v, int d) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    lo = __shfl_up_sync(FULL, lo, d);
    hi = __shfl_up_sync(FULL, hi, d);
    return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ u128 shfl_xor_u128(u128 v, int m) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    lo = __shfl_xor_sync(FULL, lo, m);
    hi = __shfl_xor_sync(FULL, hi, m);
    return ((u128)hi << 64) | lo;
}

// inclusive prefix over the 32 lanes (exact: integer addition)
__device__ __forceinline__ u128 warp_incl_scan(u128 v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        u128 t = shfl_up_u128(v, d);
        if (lane >= d) v += t;
    }
    return v;
}

__device__ __forceinline__ u128 warp_sum(u128 v) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v += shfl_xor_u128(v, m);
    return v;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(FULL, v, m);
    return v;
}

// ---- three-limb form of an Eq. 17 weight's fixed point -------------------
// A weight is 0 or a double in [2^-14, 2^8]; as a multiple of 2^-66 it is
// f = m 2^sh with a 53-bit mantissa m and sh = e - 1009 in [0, 22], so
// f < 2^75.  Split in 26/26/23-bit limbs, a sum of 32 limbs fits 32 bits:
// warp reductions are three REDUX.SUM, warp scans three 32-bit scans.
struct Limbs { uint32_t l0, l1, l2; };

// Limbs of w's fixed point; false for a value outside {0} U [2^-14, 2^8]
// (the general to_fx handles those: never an Eq. 17 weight of finite scores).
__device__ __forceinline__ bool weight_limbs(double w, Limbs* out) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(w);
    const int e = (int)(b >> 52);                      // sign bit included: w >= 0 only
    const int sh = e - 1009;
    const unsigned long long m = (b & 0xFFFFFFFFFFFFFull) | 0x10000000000000ull;
    const bool zero = ((b << 1) == 0ull);             // +0.0 or -0.0
    const bool ok = zero || (sh >= 0 && sh <= 22);
    const int s = (sh < 0) ? 0 : (sh > 22 ? 22 : sh);
    const unsigned long long lo = m << s;               // bits 0..63 of f
    out->l0 = zero ? 0u : (uint32_t)(lo & 0x3FFFFFFull);
    out->l1 = zero ? 0u : (uint32_t)((lo >> 26) & 0x3FFFFFFull);
    out->l2 = zero ? 0u : (uint32_t)(m >> (52 - s));     // f >> 52
    return ok;
}

__device__ __forceinline__ u128 limbs_value(uint32_t l0, uint32_t l1, uint32_t l2) {
    return (u128)l0 + ((u128)l1 << 26) + ((u128)l2 << 52);
}

// Warp sum of the lanes' limbs (exact, 32-bit per limb).
__device__ __forceinline__ u128 warp_sum_limbs(const Limbs& x) {
    return limbs_value(__reduce_add_sync(0xffffffffu, x.l0), __reduce_add_sync(0xffffffffu, x.l1),
                       __reduce_add_sync(0xffffffffu, x.l2));
}

// Inclusive warp scan of the lanes' limbs, recombined (exact).
__device__ __forceinline__ u128 warp_incl_scan_limbs(Limbs x, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t a = __shfl_up_sync(0xffffffffu, x.l0, d);
        const uint32_t b = __shfl_up_sync(0xffffffffu, x.l1, d);
        const uint32_t c = __shfl_up_sync(0xffffffffu, x.l2, d);
        if (lane >= d) { x.l0 += a; x.l1 += b; x.l2 += c; }
    }
    return limbs_value(x.l0, x.l1, x.l2);
}

// NaN-propagating max/min, as numpy's ndarray.max()/min()
__device__ __forceinline__ double nmax(double a, double b) { return (a > b || a != a) ? a : b; }
__device__ __forceinline__ double nmin(double a, double b) { return (a < b || a != a) ? a : b; }

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v = nmax(v, __shfl_xor_sync(FULL, v, m));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v = nmin(v, __shfl_xor_sync(FULL, v, m));
    return v;
}

}  // namespace ct
