// Tunable SGEMM in the style of CLBlast's xgemm: C = A B with A stored
// K-major (AT[K][M], i.e. column-major A), B[K][N] and C[M][N] row-major.
// NVRTC source; tuning parameters arrive as -D<NAME>=<v>.
//
//   MWG, NWG     block tile of C (rows x columns)
//   KWG          k-slice per main-loop step
//   MDIMC, NDIMC threads per block along m / n (block = MDIMC * NDIMC)
//   VWM, VWN     vector width of A / B loads (and of C stores along n)
//   SA, SB       stage the A / B slice in shared memory (else each thread
//                reads its operands through L1)
//   TC           tensor-core path (needs SA = SB = 1): mma.sync m16n8k8
//                TF32 with the 3xTF32 split (big*big + big*small +
//                small*big), accurate to fp32 level; warps take 16x8 tiles
//                of the block tile round-robin
//
// Thread (tm, tn) owns MWI = MWG/MDIMC rows and NWI = NWG/NDIMC columns of
// the block tile, in groups of VWM (VWN) contiguous elements interleaved
// across threads, so that operand loads and C stores are vectors.
// Sizes must be multiples of the block tile (M % MWG == N % NWG == K % KWG == 0).
#ifndef MWG
#define MWG 64
#endif
#ifndef NWG
#define NWG 64
#endif
#ifndef KWG
#define KWG 16
#endif
#ifndef MDIMC
#define MDIMC 16
#endif
#ifndef NDIMC
#define NDIMC 16
#endif
#ifndef VWM
#define VWM 2
#endif
#ifndef VWN
#define VWN 2
#endif
#ifndef SA
#define SA 1
#endif
#ifndef SB
#define SB 1
#endif
#ifndef TC
#define TC 0
#endif

#if TC && !(SA && SB)
#error "the tensor-core path stages both operands in shared memory"
#endif

constexpr int NT = MDIMC * NDIMC;
constexpr int MWI = MWG / MDIMC, NWI = NWG / NDIMC;
static_assert(MWG % (MDIMC * VWM) == 0 && NWG % (NDIMC * VWN) == 0, "tile / thread / vector mismatch");

template <int V> struct vec_t;
template <> struct vec_t<1> { typedef float T; };
template <> struct vec_t<2> { typedef float2 T; };
template <> struct vec_t<4> { typedef float4 T; };
template <> struct vec_t<8> { struct __align__(32) T { float4 a, b; }; };
typedef vec_t<VWM>::T vecm;
typedef vec_t<VWN>::T vecn;

template <typename V> __device__ __forceinline__ float el(const V& v, int k) { return reinterpret_cast<const float*>(&v)[k]; }

// local row of the thread's i-th value (groups of VW contiguous, interleaved)
__device__ __forceinline__ int local_m(int i, int tm) { return (i / VWM) * (MDIMC * VWM) + tm * VWM + (i % VWM); }
__device__ __forceinline__ int local_n(int j, int tn) { return (j / VWN) * (NDIMC * VWN) + tn * VWN + (j % VWN); }

// cooperative copy of a KWG x W slice (row stride ld) into shared memory
template <int W, int V, typename VT>
__device__ __forceinline__ void stage(const float* __restrict__ src, int ld, float* dst, int tid) {
    constexpr int NV = KWG * W / V;
#pragma unroll
    for (int v = tid; v < NV; v += NT) {
        const int k = v / (W / V), c = (v % (W / V)) * V;
        *reinterpret_cast<VT*>(dst + k * W + c) = *reinterpret_cast<const VT*>(src + (size_t)k * ld + c);
    }
}

#if TC
__device__ __forceinline__ unsigned tf32(float x) {
    unsigned r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mma(float* c, const unsigned* a, const unsigned* b) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 "
                 "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
constexpr int NWARP = NT / 32;
constexpr int TILES = (MWG / 16) * (NWG / 8);
constexpr int MAXT = (TILES + NWARP - 1) / NWARP;
#endif

extern "C" __global__ void __launch_bounds__(NT)
gemm(const float* __restrict__ at, const float* __restrict__ b, float* __restrict__ c, int M, int N,
     int K) {
    const int tid = threadIdx.x;
    const int m0 = blockIdx.x * MWG, n0 = blockIdx.y * NWG;
#if SA
    __shared__ __align__(32) float As[KWG * MWG];
#endif
#if SB
    __shared__ __align__(32) float Bs[KWG * NWG];
#endif
#if TC
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    float acc[MAXT][4];
#pragma unroll
    for (int s = 0; s < MAXT; ++s) acc[s][0] = acc[s][1] = acc[s][2] = acc[s][3] = 0.0f;
#else
    const int tm = tid % MDIMC, tn = tid / MDIMC;
    float acc[MWI][NWI];
#pragma unroll
    for (int i = 0; i < MWI; ++i)
#pragma unroll
        for (int j = 0; j < NWI; ++j) acc[i][j] = 0.0f;
#endif

    for (int k0 = 0; k0 < K; k0 += KWG) {
#if SA || SB
        __syncthreads();
#endif
#if SA
        stage<MWG, VWM, vecm>(at + (size_t)k0 * M + m0, M, As, tid);
#endif
#if SB
        stage<NWG, VWN, vecn>(b + (size_t)k0 * N + n0, N, Bs, tid);
#endif
#if SA || SB
        __syncthreads();
#endif
#if TC
#pragma unroll
        for (int kk = 0; kk < KWG; kk += 8) {
#pragma unroll
            for (int s = 0; s < MAXT; ++s) {
                const int tile = warp + s * NWARP;
                if (tile < TILES) {
                    const int tmm = (tile % (MWG / 16)) * 16, tnn = (tile / (MWG / 16)) * 8;
                    float af[4], bf[2];
                    af[0] = As[(kk + t4) * MWG + tmm + g];
                    af[1] = As[(kk + t4) * MWG + tmm + g + 8];
                    af[2] = As[(kk + t4 + 4) * MWG + tmm + g];
                    af[3] = As[(kk + t4 + 4) * MWG + tmm + g + 8];
                    bf[0] = Bs[(kk + t4) * NWG + tnn + g];
                    bf[1] = Bs[(kk + t4 + 4) * NWG + tnn + g];
                    unsigned ab[4], as[4], bb[2], bs[2];
#pragma unroll
                    for (int q = 0; q < 4; ++q) { ab[q] = tf32(af[q]); as[q] = tf32(af[q] - __uint_as_float(ab[q])); }
#pragma unroll
                    for (int q = 0; q < 2; ++q) { bb[q] = tf32(bf[q]); bs[q] = tf32(bf[q] - __uint_as_float(bb[q])); }
                    mma(acc[s], as, bb);
                    mma(acc[s], ab, bs);
                    mma(acc[s], ab, bb);
                }
            }
        }
#else
#pragma unroll
        for (int kk = 0; kk < KWG; ++kk) {
            float av[MWI], bv[NWI];
#pragma unroll
            for (int i = 0; i < MWI; i += VWM) {
#if SA
                const vecm v = *reinterpret_cast<const vecm*>(As + kk * MWG + local_m(i, tm));
#else
                const vecm v = *reinterpret_cast<const vecm*>(at + (size_t)(k0 + kk) * M + m0 + local_m(i, tm));
#endif
#pragma unroll
                for (int q = 0; q < VWM; ++q) av[i + q] = el(v, q);
            }
#pragma unroll
            for (int j = 0; j < NWI; j += VWN) {
#if SB
                const vecn v = *reinterpret_cast<const vecn*>(Bs + kk * NWG + local_n(j, tn));
#else
                const vecn v = *reinterpret_cast<const vecn*>(b + (size_t)(k0 + kk) * N + n0 + local_n(j, tn));
#endif
#pragma unroll
                for (int q = 0; q < VWN; ++q) bv[j + q] = el(v, q);
            }
#pragma unroll
            for (int i = 0; i < MWI; ++i)
#pragma unroll
                for (int j = 0; j < NWI; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
#endif
    }

#if TC
#pragma unroll
    for (int s = 0; s < MAXT; ++s) {
        const int tile = warp + s * NWARP;
        if (tile < TILES) {
            const int tmm = (tile % (MWG / 16)) * 16, tnn = (tile / (MWG / 16)) * 8;
            float* r0 = c + (size_t)(m0 + tmm + g) * N + n0 + tnn + 2 * t4;
            float* r1 = r0 + (size_t)8 * N;
            *reinterpret_cast<float2*>(r0) = make_float2(acc[s][0], acc[s][1]);
            *reinterpret_cast<float2*>(r1) = make_float2(acc[s][2], acc[s][3]);
        }
    }
#else
#pragma unroll
    for (int i = 0; i < MWI; ++i) {
        float* row = c + (size_t)(m0 + local_m(i, tm)) * N + n0;
#pragma unroll
        for (int j = 0; j < NWI; j += VWN) {
            vecn v;
#pragma unroll
            for (int q = 0; q < VWN; ++q) reinterpret_cast<float*>(&v)[q] = acc[i][j + q];
            *reinterpret_cast<vecn*>(row + local_n(j, tn)) = v;
        }
    }
#endif
}
