// Tunable fp32 matrix transpose, out[x][y] = in[y][x] (in: HEIGHT x WIDTH,
// row-major).  NVRTC source: every tuning parameter arrives as -D<NAME>=<v>.
//
//   TILE      square tile edge (8..64)
//   VEC       floats per load/store (float, float2, float4)
//   PAD       +1 float per shared-memory row (bank-conflict-free column reads)
//   BLOCK_Y   thread rows; the block is (TILE/VEC) x BLOCK_Y, each thread
//             walks TILE/BLOCK_Y rows of the tile
//   USE_SMEM  stage the tile in shared memory (coalesced loads AND stores)
//             or store straight from registers (strided stores)
//   DIAG      diagonal block order (spreads concurrent blocks over memory
//             partitions)
//   UNROLL    unroll factor of the per-thread row loop
//   WORK_X    tiles per block along x (one launch covers WIDTH/(TILE WORK_X)
//             block columns)
//
// HBM-bound: 2 * 4 * WIDTH * HEIGHT algorithmic bytes per launch.
#ifndef TILE
#define TILE 32
#endif
#ifndef VEC
#define VEC 4
#endif
#ifndef PAD
#define PAD 1
#endif
#ifndef BLOCK_Y
#define BLOCK_Y 8
#endif
#ifndef USE_SMEM
#define USE_SMEM 1
#endif
#ifndef DIAG
#define DIAG 0
#endif
#ifndef UNROLL
#define UNROLL 4
#endif
#ifndef WORK_X
#define WORK_X 1
#endif

template <int V> struct vec_t;
template <> struct vec_t<1> { typedef float T; };
template <> struct vec_t<2> { typedef float2 T; };
template <> struct vec_t<4> { typedef float4 T; };
typedef vec_t<VEC>::T vec;

__device__ __forceinline__ float get(const vec& v, int k) { return reinterpret_cast<const float*>(&v)[k]; }
__device__ __forceinline__ void set(vec& v, int k, float x) { reinterpret_cast<float*>(&v)[k] = x; }

constexpr int TX = TILE / VEC;
constexpr int kUnroll = UNROLL;

extern "C" __global__ void __launch_bounds__(TX * BLOCK_Y)
transpose(const float* __restrict__ in, float* __restrict__ out, int width, int height) {
    int bx = blockIdx.x, by = blockIdx.y;
    if (DIAG) {
        // diagonal reordering for any grid shape (linear id -> diagonal)
        const int bid = blockIdx.x + gridDim.x * blockIdx.y;
        by = bid % gridDim.y;
        bx = ((bid / gridDim.y) + by) % gridDim.x;
    }
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int y0 = by * TILE;
#if USE_SMEM
    __shared__ float tile[TILE][TILE + PAD];
#endif
    for (int wx = 0; wx < WORK_X; ++wx) {
        const int x0 = (bx * WORK_X + wx) * TILE;
#if USE_SMEM
#pragma unroll kUnroll
        for (int r = ty; r < TILE; r += BLOCK_Y) {
            const vec v = *reinterpret_cast<const vec*>(in + (size_t)(y0 + r) * width + x0 + tx * VEC);
#pragma unroll
            for (int k = 0; k < VEC; ++k) tile[r][tx * VEC + k] = get(v, k);
        }
        __syncthreads();
#pragma unroll kUnroll
        for (int r = ty; r < TILE; r += BLOCK_Y) {
            vec v;
#pragma unroll
            for (int k = 0; k < VEC; ++k) set(v, k, tile[tx * VEC + k][r]);
            *reinterpret_cast<vec*>(out + (size_t)(x0 + r) * height + y0 + tx * VEC) = v;
        }
        __syncthreads();
#else
#pragma unroll kUnroll
        for (int r = ty; r < TILE; r += BLOCK_Y) {
            const vec v = *reinterpret_cast<const vec*>(in + (size_t)(y0 + r) * width + x0 + tx * VEC);
#pragma unroll
            for (int k = 0; k < VEC; ++k) out[(size_t)(x0 + tx * VEC + k) * height + y0 + r] = get(v, k);
        }
#endif
    }
}
