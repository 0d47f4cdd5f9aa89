// Tunable 2D convolution (FILTER x FILTER taps, zero padding), fp32:
//   out[y][x] = sum_{fy, fx} in[y + fy - R][x + fx - R] * filt[fy][fx]
// NVRTC source; tuning parameters arrive as -D<NAME>=<v>.
//
//   TBX, TBY    threads per block in x / y
//   WPTX, WPTY  outputs per thread in x (contiguous) / y (strided by TBY;
//               contiguous with LOCAL = 2)
//   VW          floats per output store (WPTX % VW == 0)
//   LOCAL       0: input straight from global memory
//               1: block's input tile (+ halo) staged in shared memory
//               2: as 1, and each thread owns WPTY contiguous output rows:
//                  every input row it needs is read from shared memory once
//                  into a register window (WPTX + FILTER - 1 values) and
//                  feeds all the thread's output rows it touches (2D
//                  register blocking: (WPTX+F-1)(WPTY+F-1) loads per
//                  WPTX*WPTY*F*F FMAs)
//   PAD         +1 float per shared-memory tile row (LOCAL > 0)
//   UNROLL_F    fully unroll the filter loops
//   CACHE_F     1: filter staged in shared memory; 0: filter passed by value
//               in the kernel parameters (the constant bank: FFMA takes it
//               as an operand, no load instruction at all)
//   REVERSE     filter traversal order (fx outer instead of fy outer)
//
// With LOCAL = 2 and WPTX even, each thread's output columns are processed in
// adjacent pairs with Blackwell's packed FP32 FMA (FFMA2, PTX fma.rn.f32x2,
// sm_100): output pair (2h, 2h+1) with filter column fx reads the window
// pair (win[2h+fx], win[2h+fx+1]) and takes the filter tap as a broadcast
// operand.  Every lane's FMA is the scalar path's, in the same order:
// outputs are identical.  The tile is staged twice, the second copy shifted
// by one float, so every window pair is one aligned 8-byte load (no register
// moves); the row stride is then even (PAD pads by two floats).
//
// The tile lives in dynamic shared memory: the host passes
// smem_bytes() = 4 * ((TH + F - 1) * (TW + 8 + PAD) + CACHE_F * F * F), and
// with the packed path two tile copies and (CACHE_F) the duplicated taps.
#ifndef TBX
#define TBX 32
#endif
#ifndef TBY
#define TBY 8
#endif
#ifndef WPTX
#define WPTX 2
#endif
#ifndef WPTY
#define WPTY 2
#endif
#ifndef VW
#define VW 2
#endif
#ifndef LOCAL
#define LOCAL 1
#endif
#ifndef PAD
#define PAD 0
#endif
#ifndef UNROLL_F
#define UNROLL_F 1
#endif
#ifndef CACHE_F
#define CACHE_F 1
#endif
#ifndef REVERSE
#define REVERSE 0
#endif
#ifndef FILTER
#define FILTER 7
#endif

constexpr int F = FILTER, R = FILTER / 2;
constexpr int TW = TBX * WPTX, TH = TBY * WPTY;
constexpr int LH = TH + F - 1;                    // tile rows incl. halo
constexpr int V4 = (TW + 8) / 4;                  // float4 per staged row: x0-4 .. x0+TW+3
// packed-FMA path (see above): two copies of the tile, the second shifted by
// one float, so that every window pair is one aligned 8-byte shared load
// (only where the doubled tile still fits the 227 KB per-block limit; a
// preprocessor test, since it also selects the packed code path below)
#define CONV_PAIRED_SMEM (4 * (2 * (TBY * WPTY + FILTER - 1) * ((TBX * WPTX + 8) / 4 * 4 + 2 * PAD) \
                              + (CACHE_F ? (FILTER * FILTER + 1) / 2 * 2 + 2 * FILTER * FILTER : 0)))
#if LOCAL == 2 && WPTX % 2 == 0 && CONV_PAIRED_SMEM <= 227 * 1024
#define CONV_PAIRED 1
#else
#define CONV_PAIRED 0
#endif
constexpr bool PAIRED = CONV_PAIRED;
constexpr int SW = PAIRED ? 4 * V4 + 2 * PAD : 4 * V4 + PAD;   // shared row stride (even if PAIRED)
static_assert(F <= 9, "the staged row holds a halo of at most 4 columns per side");
constexpr int NT = TBX * TBY;
constexpr int kUnrollF = UNROLL_F ? F : 1;

template <int V> struct vec_t;
template <> struct vec_t<1> { typedef float T; };
template <> struct vec_t<2> { typedef float2 T; };
template <> struct vec_t<4> { typedef float4 T; };
typedef vec_t<VW>::T vec;

__device__ __forceinline__ float load_global(const float* __restrict__ in, int width, int height,
                                             int gx, int gy) {
    return (gx >= 0 && gx < width && gy >= 0 && gy < height) ? __ldg(in + (size_t)gy * width + gx)
                                                             : 0.0f;
}

// the filter by value: the taps, then each tap duplicated as a packed pair
// (the broadcast operand of the FFMA2 path, read straight from the
// parameter bank instead of being packed into a register pair per use)
struct Filter { float f[FILTER * FILTER]; unsigned long long f2[FILTER * FILTER]; };

extern "C" __global__ void __launch_bounds__(NT)
conv(const float* __restrict__ in, const float* __restrict__ filt, const Filter kf,
     float* __restrict__ out,
     int width, int height) {
    extern __shared__ __align__(16) float dsm[];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TBX + tx;
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
#if CACHE_F
    float* sf = dsm + (LOCAL ? (PAIRED ? 2 : 1) * LH * SW : 0);
    for (int i = tid; i < F * F; i += NT) sf[i] = filt[i];
#if CONV_PAIRED
    // pairs (f, f) after the taps, 8-byte aligned
    unsigned long long* sf2 = reinterpret_cast<unsigned long long*>(sf + ((F * F + 1) & ~1));
    for (int i = tid; i < F * F; i += NT) {
        const float f = filt[i];
        unsigned long long p;
        asm("mov.b64 %0, {%1, %1};" : "=l"(p) : "f"(f));
        sf2[i] = p;
    }
#endif
#define FILT(fy, fx) sf[(fy) * F + (fx)]
#define FILT2(fy, fx) sf2[(fy) * F + (fx)]
#else
#define FILT2(fy, fx) kf.f2[(fy) * F + (fx)]
#define FILT(fy, fx) kf.f[(fy) * F + (fx)]
#endif
#if LOCAL
    // the tile starts at column x0 - 4 (16-byte aligned: x0 is a multiple of
    // TW >= 8, the image width a multiple of 4), so it is read with float4
    // loads that are either wholly inside the image or wholly outside; the
    // R = FILTER/2 halo columns the filter needs begin at tile column 4 - R
    float* tile = dsm;
    for (int i = tid; i < LH * V4; i += NT) {
        const int ry = i / V4, c4 = i - ry * V4;
        const int gx = x0 - 4 + 4 * c4, gy = y0 + ry - R;
        float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (gx >= 0 && gx < width && gy >= 0 && gy < height)
            v = __ldg(reinterpret_cast<const float4*>(in + (size_t)gy * width + gx));
        float* d = tile + ry * SW + 4 * c4;
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
        if (PAIRED) {       // tile2[i] = tile[i + 1]
            float* d2 = dsm + LH * SW + ry * SW + 4 * c4 - 1;
            if (c4 > 0) d2[0] = v.x;
            d2[1] = v.y; d2[2] = v.z; d2[3] = v.w;
        }
    }
#define INPUT(ly, lx) tile[(ly) * SW + (lx) + (4 - R)]
#else
#define INPUT(ly, lx) load_global(in, width, height, x0 - R + (lx), y0 - R + (ly))
#endif
#if CACHE_F || LOCAL
    __syncthreads();
#endif
    float acc[WPTY][WPTX];
#pragma unroll
    for (int wy = 0; wy < WPTY; ++wy)
#pragma unroll
        for (int i = 0; i < WPTX; ++i) acc[wy][i] = 0.0f;

#if CONV_PAIRED
    {
        // output pairs (2h, 2h + 1); the window row as overlapping pairs
        // pr[k] = (in[k], in[k + 1]), each one 8-byte shared load
        constexpr int H = WPTX / 2, L = WPTX + F - 1;
        typedef unsigned long long f2;
        const int ly0 = ty * WPTY;
        const int lx = tx * WPTX;
        f2 accp[WPTY][H];
#pragma unroll
        for (int wy = 0; wy < WPTY; ++wy)
#pragma unroll
            for (int h = 0; h < H; ++h) accp[wy][h] = 0ull;
        const float* tile2 = dsm + LH * SW;
#pragma unroll
        for (int iy = 0; iy < WPTY + F - 1; ++iy) {
            // pair k = (in[k], in[k+1]) of this input row: tile index
            // row + lx + k + (4 - R) has the parity of k + 4 - R (row and lx
            // are even), an odd index is read from the shifted copy
            const int rowi = (ly0 + iy) * SW + lx + (4 - R);
            f2 pr[L - 1];
#pragma unroll
            for (int k = 0; k < L - 1; ++k) {
                const float* src = ((k + 4 - R) & 1) ? tile2 + rowi + k - 1 : tile + rowi + k;
                pr[k] = *reinterpret_cast<const f2*>(src);
            }
#pragma unroll
            for (int wy = 0; wy < WPTY; ++wy) {
                const int fy = iy - wy;
                if (fy >= 0 && fy < F) {
#if REVERSE
#pragma unroll
                    for (int h = 0; h < H; ++h)
#pragma unroll kUnrollF
                        for (int fx = 0; fx < F; ++fx) {
                            const f2 fp = FILT2(fy, fx);
                            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(accp[wy][h]) : "l"(pr[2 * h + fx]), "l"(fp));
                        }
#else
#pragma unroll kUnrollF
                    for (int fx = 0; fx < F; ++fx) {
                        const f2 fp = FILT2(fy, fx);
#pragma unroll
                        for (int h = 0; h < H; ++h)
                            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(accp[wy][h]) : "l"(pr[2 * h + fx]), "l"(fp));
                    }
#endif
                }
            }
        }
#pragma unroll
        for (int wy = 0; wy < WPTY; ++wy)
#pragma unroll
            for (int h = 0; h < H; ++h)
                asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[wy][2 * h]), "=f"(acc[wy][2 * h + 1]) : "l"(accp[wy][h]));
    }
#elif LOCAL == 2
    {
        const int ly0 = ty * WPTY;         // first output row inside the tile
        const int lx = tx * WPTX;          // first output column inside the tile
        // input row iy feeds output row wy through filter row fy = iy - wy;
        // per output the taps still go fy ascending, fx ascending
#pragma unroll
        for (int iy = 0; iy < WPTY + F - 1; ++iy) {
            float win[WPTX + F - 1];
#pragma unroll
            for (int k = 0; k < WPTX + F - 1; ++k) win[k] = INPUT(ly0 + iy, lx + k);
#pragma unroll
            for (int wy = 0; wy < WPTY; ++wy) {
                const int fy = iy - wy;
                if (fy >= 0 && fy < F) {
#if REVERSE
#pragma unroll
                    for (int i = 0; i < WPTX; ++i)
#pragma unroll kUnrollF
                        for (int fx = 0; fx < F; ++fx) acc[wy][i] += win[i + fx] * FILT(fy, fx);
#else
#pragma unroll kUnrollF
                    for (int fx = 0; fx < F; ++fx) {
                        const float f = FILT(fy, fx);
#pragma unroll
                        for (int i = 0; i < WPTX; ++i) acc[wy][i] += win[i + fx] * f;
                    }
#endif
                }
            }
        }
    }
#else
#pragma unroll
    for (int wy = 0; wy < WPTY; ++wy) {
        const int ly = wy * TBY + ty;      // output row inside the tile
        const int lx = tx * WPTX;          // first output column inside the tile
#if REVERSE
#pragma unroll kUnrollF
        for (int fx = 0; fx < F; ++fx)
#pragma unroll kUnrollF
            for (int fy = 0; fy < F; ++fy) {
#else
#pragma unroll kUnrollF
        for (int fy = 0; fy < F; ++fy)
#pragma unroll kUnrollF
            for (int fx = 0; fx < F; ++fx) {
#endif
                const float f = FILT(fy, fx);
#pragma unroll
                for (int i = 0; i < WPTX; ++i) acc[wy][i] += INPUT(ly + fy, lx + i + fx) * f;
            }
    }
#endif
#pragma unroll
    for (int wy = 0; wy < WPTY; ++wy) {
        const int y = y0 + (LOCAL == 2 ? ty * WPTY + wy : wy * TBY + ty);
        float* row = out + (size_t)y * width + x0 + tx * WPTX;
#pragma unroll
        for (int i = 0; i < WPTX; i += VW) {
            vec v;
#pragma unroll
            for (int k = 0; k < VW; ++k) reinterpret_cast<float*>(&v)[k] = acc[wy][i + k];
            *reinterpret_cast<vec*>(row + i) = v;
        }
    }
}
