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
