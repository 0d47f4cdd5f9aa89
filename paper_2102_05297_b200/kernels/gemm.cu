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
//   TC           tensor-core path (needs SA = SB = 1), TF32 with the 3xTF32
//                split (big*big + big*small + small*big), accurate to fp32
//                level:
//                  MWG = 128 and >= 4 warps: 5th-generation tensor cores --
//                    one thread issues tcgen05.mma (M = 128, N = NWG, K = 8)
//                    from K-major canonical shared-memory tiles into a TMEM
//                    accumulator, completion through tcgen05.commit on an
//                    mbarrier, epilogue by tcgen05.ld (warp q reads TMEM
//                    lanes 32q..32q+31 = rows of C);
//                  otherwise: mma.sync m16n8k8, warps take 16x8 tiles of the
//                    block tile round-robin
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

#if TC && MWG == 128 && MDIMC * NDIMC >= 128
#define TC5 1
#else
#define TC5 0
#endif

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

#if TC5
// K-major canonical (no swizzle) layout of a ROWS x KWG fp32 tile: 8x16-byte
// core matrices; element (r, k) at (r/8)*SBO + (k/4)*128 + (r%8)*16 + (k%4)*4
// bytes with LBO = 128 (next 4 k) and SBO = KWG*32 (next 8 rows).
constexpr int SBO = KWG * 32;
__device__ __forceinline__ int kmaj(int r, int k) {
    return (r >> 3) * (SBO / 4) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}
// shared-memory matrix descriptor (sm_100 UMMA): start >> 4 | LBO >> 4 << 16 |
// SBO >> 4 << 32 | version 1 << 46, layout type 0 (SWIZZLE_NONE)
__device__ __forceinline__ unsigned long long sdesc(const void* p) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    return (unsigned long long)((a >> 4) & 0x3FFF) | ((unsigned long long)(128 >> 4) << 16) |
           ((unsigned long long)(SBO >> 4) << 32) | (1ull << 46);
}
// instruction descriptor: D f32, A/B tf32, both K-major, N = NWG, M = 128
constexpr unsigned IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(NWG >> 3) << 17) |
                           ((unsigned)(128 >> 4) << 24);
constexpr unsigned TMEM_COLS = NWG < 32 ? 32 : NWG;

__device__ __forceinline__ void umma(unsigned tmem_d, unsigned long long da,
                                     unsigned long long db, unsigned acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(tmem_d), "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
#endif

#if TC5
// 5th-generation tensor-core path (see the header), a TMA-fed pipeline:
//   * TMA (cp.async.bulk.tensor.2d) brings the fp32 slices A^T[k0:k0+KWG,
//     m0:m0+128] and B[k0:k0+KWG, n0:n0+NWG] into a two-stage ring of raw
//     tiles; an mbarrier per stage counts their bytes (expect_tx);
//   * all threads split a landed slice into tf32 big / small halves in the
//     K-major canonical operand layout (thread = one row x 4 k: four
//     conflict-free scalar shared loads, two 16-byte shared stores), into a
//     two-stage ring of operand buffers;
//   * one thread issues the slice's 3 x KWG/8 tcgen05.mma into the TMEM
//     accumulator and commits them to the stage's MMA mbarrier, then
//     launches the TMA of slice s+2 into the raw stage just consumed.
// The tensor core therefore works on slice s while the threads split slice
// s+1 and the copy engine fetches slice s+2; an operand stage is rewritten
// only after its MMAs completed (the MMA mbarrier of slice s-2).
struct __align__(64) TensorMap { unsigned long long w[16]; };

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_wait(const unsigned long long* bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void tma_2d(void* dst, const TensorMap* map, int c0, int c1,
                                       unsigned long long* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
                 "[%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(dst)), "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0),
                    "r"(c1), "r"(smem_u32(bar))
                 : "memory");
}

constexpr int RAW_A = KWG * 128, RAW_B = KWG * NWG;          // floats per raw stage
constexpr int OPS = 2 * 128 * KWG + 2 * NWG * KWG;           // big+small A, big+small B
constexpr unsigned SLICE_BYTES = 4u * (RAW_A + RAW_B);

// split raw [k][r] (row stride W floats) rows x KWG into big/small K-major
template <int ROWS>
__device__ __forceinline__ void split(const float* raw, float* big, float* small, int tid) {
    constexpr int TASKS = ROWS * (KWG / 4);
#pragma unroll
    for (int t = tid; t < TASKS; t += NT) {
        const int r = t % ROWS, kg = t / ROWS;
        float v[4], hi[4], lo[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = raw[(4 * kg + j) * ROWS + r];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            hi[j] = __uint_as_float(tf32(v[j]));
            lo[j] = __uint_as_float(tf32(v[j] - hi[j]));
        }
        const int o = kmaj(r, 4 * kg);
        *reinterpret_cast<float4*>(big + o) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<float4*>(small + o) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
}

extern "C" __global__ void __launch_bounds__(NT)
gemm(const float* __restrict__ at, const float* __restrict__ b, float* __restrict__ c, int M, int N,
     int K, const __grid_constant__ TensorMap tmA, const __grid_constant__ TensorMap tmB) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.x * MWG, n0 = blockIdx.y * NWG;
    extern __shared__ __align__(1024) float dsm[];
    float* raw = dsm;                          // [2][RAW_A + RAW_B]
    float* ops = dsm + 2 * (RAW_A + RAW_B);    // [2][OPS]
    __shared__ __align__(8) unsigned long long full[2], done[2];
    __shared__ unsigned tmem_base;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&tmem_base)), "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const int nk = K / KWG;
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&done[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
        for (int s = 0; s < 2 && s < nk; ++s) {
            float* rs = raw + s * (RAW_A + RAW_B);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         :: "r"(smem_u32(&full[s])), "r"(SLICE_BYTES) : "memory");
            tma_2d(rs, &tmA, m0, s * KWG, &full[s]);
            tma_2d(rs + RAW_A, &tmB, n0, s * KWG, &full[s]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem_d = tmem_base;
    for (int s = 0; s < nk; ++s) {
        const int st = s & 1;
        const unsigned ph = (unsigned)(s >> 1) & 1u;
        float* rs = raw + st * (RAW_A + RAW_B);
        float* os = ops + st * OPS;
        float* a_big = os;
        float* a_small = a_big + 128 * KWG;
        float* b_big = a_small + 128 * KWG;
        float* b_small = b_big + NWG * KWG;
        mbar_wait(&full[st], ph);                       // slice s landed
        if (s >= 2) mbar_wait(&done[st], ph ^ 1u);      // MMAs of slice s-2 done: stage free
        split<128>(rs, a_big, a_small, tid);
        split<NWG>(rs + RAW_A, b_big, b_small, tid);
        // generic-proxy shared stores -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;");
        __syncthreads();
        if (tid == 0) {
            if (s + 2 < nk) {      // every thread is done reading this raw stage
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             :: "r"(smem_u32(&full[st])), "r"(SLICE_BYTES) : "memory");
                tma_2d(rs, &tmA, m0, (s + 2) * KWG, &full[st]);
                tma_2d(rs + RAW_A, &tmB, n0, (s + 2) * KWG, &full[st]);
            }
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int kk = 0; kk < KWG / 8; ++kk) {
                const int off = kk * 64;   // 8 k = two 4-k core-matrix columns = 256 B
                const unsigned acc0 = (s > 0 || kk > 0) ? 1u : 0u;
                umma(tmem_d, sdesc(a_small + off), sdesc(b_big + off), acc0);
                umma(tmem_d, sdesc(a_big + off), sdesc(b_small + off), 1u);
                umma(tmem_d, sdesc(a_big + off), sdesc(b_big + off), 1u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         :: "r"(smem_u32(&done[st])) : "memory");
        }
    }
    // the last commit completes after every earlier MMA
    mbar_wait(&done[(nk - 1) & 1], (unsigned)((nk - 1) >> 1) & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // epilogue: warps 0..3 read rows 32q + lane of the accumulator
    if (warp < 4) {
        const int row = warp * 32 + lane;
        float* crow = c + (size_t)(m0 + row) * N + n0;
#pragma unroll
        for (int c0 = 0; c0 < NWG; c0 += 8) {
            unsigned v[8];
            const unsigned taddr = tmem_d + ((unsigned)(warp * 32) << 16) + (unsigned)c0;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                           "=r"(v[6]), "=r"(v[7])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            *reinterpret_cast<float4*>(crow + c0) =
                make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]),
                            __uint_as_float(v[3]));
            *reinterpret_cast<float4*>(crow + c0 + 4) =
                make_float4(__uint_as_float(v[4]), __uint_as_float(v[5]), __uint_as_float(v[6]),
                            __uint_as_float(v[7]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                     :: "r"(tmem_d), "n"(TMEM_COLS));
}
#else
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
#endif  // TC5
