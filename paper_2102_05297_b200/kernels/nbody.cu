// Tunable all-pairs N-body acceleration step:
//   a_i = sum_j m_j (p_j - p_i) / (|p_j - p_i|^2 + eps^2)^(3/2)
// NVRTC source; tuning parameters arrive as -D<NAME>=<v>.
//
//   BLOCK       bodies per block (threads along x)
//   OUTER       bodies per thread (strided by the launch's x extent)
//   UNROLL      unroll factor of the j loop
//   USE_SMEM    stage BLOCK bodies at a time in shared memory
//   VEC         j bodies per load step (SoA: float2/float4 vector loads)
//   FAST_RSQRT  MUFU rsqrt (rsqrt.approx.ftz) instead of 1/sqrtf (IEEE sqrt +
//               division)
//   SOA         positions/masses as four float arrays instead of float4
//
// JS and gridDim.y = JB (set by the host, not tuning parameters): the j range
// is split over JB blocks and, inside a block, over blockDim.y = JS thread
// rows, so that n = 16,384 bodies still fill the 148 SMs (one thread per body
// would be 512 warps) -- in one wave of resident blocks (live.py split()).  A body's JS partial sums are reduced in shared
// memory, its JB block partials by the last block to finish (fixed order,
// deterministic; the arrival counters reset themselves, so a launch is
// idempotent under timing and profiler replay).
//
// 20 flops per interaction (the customary count); FP32/MUFU-bound.
//
// With OUTER even, a thread's bodies are processed in pairs with Blackwell's
// packed FP32 instructions (FADD2 / FMUL2 / FFMA2, PTX add/mul/fma.rn.f32x2,
// sm_100): one instruction advances two interactions, the j body's
// coordinates enter as a broadcast scalar operand, and each lane's
// operation is the scalar path's IEEE operation, so the sums are identical.
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
#ifndef JS
#define JS 1
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
        const float r2 = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, eps2)));
#if FAST_RSQRT
        // MUFU.RSQ alone: r2 >= eps2 > 0 is never denormal, so rsqrtf's
        // denormal scaling (a compare and two multiplies) is dropped
        float inv;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(r2));
#else
        const float inv = 1.0f / sqrtf(r2);
#endif
        const float s = (m * inv) * (inv * inv);
        ax = fmaf(dx, s, ax); ay = fmaf(dy, s, ay); az = fmaf(dz, s, az);
    }
};

#if OUTER % 2 == 0
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
    f2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r;
}
__device__ __forceinline__ void upk(f2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
    f2 d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}

// two of the thread's bodies, lane k of every register pair = body 2p + k
struct BodyPair {
    f2 px, py, pz, ax, ay, az;
    __device__ __forceinline__ void interact(float qx, float qy, float qz, float m, float eps2) {
        const f2 dx = sub2(pk(qx, qx), px), dy = sub2(pk(qy, qy), py), dz = sub2(pk(qz, qz), pz);
        const f2 r2 = fma2(dz, dz, fma2(dy, dy, fma2(dx, dx, pk(eps2, eps2))));
        float r0, r1;
        upk(r2, r0, r1);
#if FAST_RSQRT
        float i0, i1;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(i0) : "f"(r0));
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(i1) : "f"(r1));
#else
        const float i0 = 1.0f / sqrtf(r0), i1 = 1.0f / sqrtf(r1);
#endif
        const f2 inv = pk(i0, i1);
        const f2 s = mul2(mul2(pk(m, m), inv), mul2(inv, inv));
        ax = fma2(dx, s, ax); ay = fma2(dy, s, ay); az = fma2(dz, s, az);
    }
};
#endif

// at most 64 registers: 1024 resident threads per SM, which the host's
// choice of JS / JB fills in one wave (live.NBodyBenchmark.split)
extern "C" __global__ void __launch_bounds__(BLOCK * JS, (1024 / (BLOCK * JS)) > 0 ? 1024 / (BLOCK * JS) : 1)
nbody(const float4* __restrict__ pm, const float* __restrict__ x, const float* __restrict__ y,
      const float* __restrict__ z, const float* __restrict__ m, int n, float eps2,
      float4* __restrict__ acc, float4* __restrict__ partial, unsigned* __restrict__ arrivals) {
    const int nthreads = gridDim.x * BLOCK;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int t = blockIdx.x * BLOCK + tx;
    const int JB = gridDim.y;
    // this thread row's share of the j range (a multiple of BLOCK)
    const int splits = JB * JS;
    const int span = ((n + splits - 1) / splits + BLOCK - 1) / BLOCK * BLOCK;
    const int j0 = min(n, (blockIdx.y * JS + ty) * span), j1 = min(n, j0 + span);
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
#if OUTER % 2 == 0
    // the interaction loops run on packed pairs; the scalar bodies are
    // rebuilt from them for the reductions below
    BodyPair bp[OUTER / 2];
#pragma unroll
    for (int p = 0; p < OUTER / 2; ++p) {
        bp[p].px = pk(b[2 * p].px, b[2 * p + 1].px);
        bp[p].py = pk(b[2 * p].py, b[2 * p + 1].py);
        bp[p].pz = pk(b[2 * p].pz, b[2 * p + 1].pz);
        bp[p].ax = bp[p].ay = bp[p].az = 0ull;
    }
#define INTERACT_ALL(qx, qy, qz, qm) \
    _Pragma("unroll") for (int p = 0; p < OUTER / 2; ++p) bp[p].interact(qx, qy, qz, qm, eps2)
#else
#define INTERACT_ALL(qx, qy, qz, qm) \
    _Pragma("unroll") for (int o = 0; o < OUTER; ++o) b[o].interact(qx, qy, qz, qm, eps2)
#endif
#if USE_SMEM
#if SOA
    __shared__ __align__(16) float sx[JS][BLOCK], sy[JS][BLOCK], sz[JS][BLOCK], sm[JS][BLOCK];
#else
    __shared__ float4 sp[JS][BLOCK];
#endif
    // every thread row walks the same number of tiles (barriers stay uniform)
    for (int base = 0; base < span; base += BLOCK) {
        __syncthreads();
        const int j = j0 + base + tx;
#if SOA
        if (j < j1) { sx[ty][tx] = x[j]; sy[ty][tx] = y[j]; sz[ty][tx] = z[j]; sm[ty][tx] = m[j]; }
#else
        if (j < j1) sp[ty][tx] = pm[j];
#endif
        __syncthreads();
        const int cnt = max(0, min(BLOCK, j1 - j0 - base));
#pragma unroll kUnroll
        for (int jj = 0; jj < cnt; jj += VEC) {
#if SOA
            const vec vx = *reinterpret_cast<const vec*>(&sx[ty][jj]);
            const vec vy = *reinterpret_cast<const vec*>(&sy[ty][jj]);
            const vec vz = *reinterpret_cast<const vec*>(&sz[ty][jj]);
            const vec vm = *reinterpret_cast<const vec*>(&sm[ty][jj]);
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                INTERACT_ALL(get(vx, k), get(vy, k), get(vz, k), get(vm, k));
            }
#else
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                const float4 q = sp[ty][jj + k];
                INTERACT_ALL(q.x, q.y, q.z, q.w);
            }
#endif
        }
    }
#else
#pragma unroll kUnroll
    for (int j = j0; j < j1; j += VEC) {
#if SOA
        const vec vx = __ldg(reinterpret_cast<const vec*>(x + j));
        const vec vy = __ldg(reinterpret_cast<const vec*>(y + j));
        const vec vz = __ldg(reinterpret_cast<const vec*>(z + j));
        const vec vm = __ldg(reinterpret_cast<const vec*>(m + j));
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            INTERACT_ALL(get(vx, k), get(vy, k), get(vz, k), get(vm, k));
        }
#else
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const float4 q = __ldg(pm + j + k);
            INTERACT_ALL(q.x, q.y, q.z, q.w);
        }
#endif
    }
#endif
#if OUTER % 2 == 0
#pragma unroll
    for (int p = 0; p < OUTER / 2; ++p) {
        upk(bp[p].ax, b[2 * p].ax, b[2 * p + 1].ax);
        upk(bp[p].ay, b[2 * p].ay, b[2 * p + 1].ay);
        upk(bp[p].az, b[2 * p].az, b[2 * p + 1].az);
    }
#endif
#if JS > 1
    // partial sums of the JS thread rows, reduced in row order
    __shared__ float3 part[JS][BLOCK];
#pragma unroll
    for (int o = 0; o < OUTER; ++o) {
        __syncthreads();
        part[ty][tx] = make_float3(b[o].ax, b[o].ay, b[o].az);
        __syncthreads();
        if (ty == 0) {
            float3 s = part[0][tx];
#pragma unroll
            for (int r = 1; r < JS; ++r) { s.x += part[r][tx].x; s.y += part[r][tx].y; s.z += part[r][tx].z; }
            b[o].ax = s.x; b[o].ay = s.y; b[o].az = s.z;
        }
    }
#endif
    // thread row 0 holds the block's sums (the other rows stay for the barriers)
    if (JB == 1) {
        if (ty == 0) {
#pragma unroll
            for (int o = 0; o < OUTER; ++o) {
                const int i = t + o * nthreads;
                if (i < n) acc[i] = make_float4(b[o].ax, b[o].ay, b[o].az, 0.0f);
            }
        }
        return;
    }
    // block partials; the last of the JB blocks of this body group sums them
    if (ty == 0) {
#pragma unroll
        for (int o = 0; o < OUTER; ++o) {
            const int i = t + o * nthreads;
            if (i < n) partial[(size_t)blockIdx.y * n + i] = make_float4(b[o].ax, b[o].ay, b[o].az, 0.0f);
        }
    }
    __threadfence();
    __shared__ int last;
    __syncthreads();
    if (tx == 0 && ty == 0) last = (atomicAdd(&arrivals[blockIdx.x], 1u) == (unsigned)JB - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (ty == 0) {
#pragma unroll
        for (int o = 0; o < OUTER; ++o) {
            const int i = t + o * nthreads;
            if (i < n) {
                float4 sum = __ldcg(partial + i);
                for (int r = 1; r < JB; ++r) {
                    const float4 q = __ldcg(partial + (size_t)r * n + i);
                    sum.x += q.x; sum.y += q.y; sum.z += q.z;
                }
                acc[i] = make_float4(sum.x, sum.y, sum.z, 0.0f);
            }
        }
    }
    if (tx == 0 && ty == 0) arrivals[blockIdx.x] = 0u;
}
