// Tunable all-pairs N-body acceleration step:
//   a_i = sum_j m_j (p_j - p_i) / (|p_j - p_i|^2 + eps^2)^(3/2)
// NVRTC source; tuning parameters arrive as -D<NAME>=<v>.
//
//   BLOCK       threads per block
//   OUTER       bodies per thread (strided by the launch's thread count)
//   UNROLL      unroll factor of the j loop
//   USE_SMEM    stage BLOCK bodies at a time in shared memory
//   VEC         j bodies per load step (SoA: float2/float4 vector loads)
//   FAST_RSQRT  rsqrtf (MUFU) instead of 1/sqrtf (IEEE sqrt + division)
//   SOA         positions/masses as four float arrays instead of float4
//
// 20 flops per interaction (the customary count); FP32/MUFU-bound.
#ifndef BLOCK
#define BLOCK 256
#endif
#ifndef OUTER
#define OUTER 1
#endif
#ifndef UNROLL
#define UNROLL 4
#endif
#ifndef USE_SMEM
#define USE_SMEM 1
#endif
#ifndef VEC
#define VEC 1
#endif
#ifndef FAST_RSQRT
#define FAST_RSQRT 1
#endif
#ifndef SOA
#define SOA 0
#endif

constexpr int kUnroll = UNROLL;

template <int V> struct vec_t;
template <> struct vec_t<1> { typedef float T; };
template <> struct vec_t<2> { typedef float2 T; };
template <> struct vec_t<4> { typedef float4 T; };
typedef vec_t<VEC>::T vec;
__device__ __forceinline__ float get(const vec& v, int k) { return reinterpret_cast<const float*>(&v)[k]; }

struct Body {
    float px, py, pz, ax, ay, az;
    __device__ __forceinline__ void interact(float qx, float qy, float qz, float m, float eps2) {
        const float dx = qx - px, dy = qy - py, dz = qz - pz;
        const float r2 = dx * dx + dy * dy + dz * dz + eps2;
#if FAST_RSQRT
        const float inv = rsqrtf(r2);
#else
        const float inv = 1.0f / sqrtf(r2);
#endif
        const float s = m * (inv * inv * inv);
        ax += dx * s; ay += dy * s; az += dz * s;
    }
};

extern "C" __global__ void __launch_bounds__(BLOCK)
nbody(const float4* __restrict__ pm, const float* __restrict__ x, const float* __restrict__ y,
      const float* __restrict__ z, const float* __restrict__ m, int n, float eps2,
      float4* __restrict__ acc) {
    const int nthreads = gridDim.x * BLOCK;
    const int t = blockIdx.x * BLOCK + threadIdx.x;
    Body b[OUTER];
#pragma unroll
    for (int o = 0; o < OUTER; ++o) {
        const int i = min(t + o * nthreads, n - 1);
#if SOA
        b[o].px = x[i]; b[o].py = y[i]; b[o].pz = z[i];
#else
        const float4 q = pm[i];
        b[o].px = q.x; b[o].py = q.y; b[o].pz = q.z;
#endif
        b[o].ax = b[o].ay = b[o].az = 0.0f;
    }
#if USE_SMEM
#if SOA
    __shared__ __align__(16) float sx[BLOCK], sy[BLOCK], sz[BLOCK], sm[BLOCK];
#else
    __shared__ float4 sp[BLOCK];
#endif
    for (int base = 0; base < n; base += BLOCK) {
        __syncthreads();
        const int j = base + threadIdx.x;
#if SOA
        if (j < n) { sx[threadIdx.x] = x[j]; sy[threadIdx.x] = y[j]; sz[threadIdx.x] = z[j]; sm[threadIdx.x] = m[j]; }
#else
        if (j < n) sp[threadIdx.x] = pm[j];
#endif
        __syncthreads();
        const int cnt = min(BLOCK, n - base);
#pragma unroll kUnroll
        for (int jj = 0; jj < cnt; jj += VEC) {
#if SOA
            const vec vx = *reinterpret_cast<const vec*>(sx + jj);
            const vec vy = *reinterpret_cast<const vec*>(sy + jj);
            const vec vz = *reinterpret_cast<const vec*>(sz + jj);
            const vec vm = *reinterpret_cast<const vec*>(sm + jj);
#pragma unroll
            for (int k = 0; k < VEC; ++k)
#pragma unroll
                for (int o = 0; o < OUTER; ++o) b[o].interact(get(vx, k), get(vy, k), get(vz, k), get(vm, k), eps2);
#else
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                const float4 q = sp[jj + k];
#pragma unroll
                for (int o = 0; o < OUTER; ++o) b[o].interact(q.x, q.y, q.z, q.w, eps2);
            }
#endif
        }
    }
#else
#pragma unroll kUnroll
    for (int j = 0; j < n; j += VEC) {
#if SOA
        const vec vx = __ldg(reinterpret_cast<const vec*>(x + j));
        const vec vy = __ldg(reinterpret_cast<const vec*>(y + j));
        const vec vz = __ldg(reinterpret_cast<const vec*>(z + j));
        const vec vm = __ldg(reinterpret_cast<const vec*>(m + j));
#pragma unroll
        for (int k = 0; k < VEC; ++k)
#pragma unroll
            for (int o = 0; o < OUTER; ++o) b[o].interact(get(vx, k), get(vy, k), get(vz, k), get(vm, k), eps2);
#else
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const float4 q = __ldg(pm + j + k);
#pragma unroll
            for (int o = 0; o < OUTER; ++o) b[o].interact(q.x, q.y, q.z, q.w, eps2);
        }
#endif
    }
#endif
#pragma unroll
    for (int o = 0; o < OUTER; ++o) {
        const int i = t + o * nthreads;
        if (i < n) acc[i] = make_float4(b[o].ax, b[o].ay, b[o].az, 0.0f);
    }
}
