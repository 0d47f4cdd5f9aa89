// Known-answer kernel for validating the CUPTI collector (tests/test_cupti_gpu.py).
// Every thread executes, in straight-line inline PTX (no compiler freedom):
//   NFMA  dependent fma.rn.f32 (SASS FFMA)           -> INST_F32 = threads * NFMA
//   NLDS  ld.shared.u32 of its own word (conflict-free, one wavefront per warp)
//   one st.shared.u32, a __syncthreads, and two global stores
// Launch with 1-D blocks of a multiple of 32 threads and a grid that covers
// `out` exactly (no bounds test, no divergence).
#ifndef NFMA
#define NFMA 64
#endif
#ifndef NLDS
#define NLDS 8
#endif

extern "C" __global__ void probe(float* __restrict__ out, unsigned* __restrict__ tag, float a,
                                 float b) {
    __shared__ unsigned sh[1024];
    const unsigned t = threadIdx.x;
    unsigned s_addr = (unsigned)__cvta_generic_to_shared(&sh[t]);
    asm volatile("st.shared.u32 [%0], %1;" :: "r"(s_addr), "r"(t));
    __syncthreads();
    unsigned acc_u = 0;
#pragma unroll
    for (int i = 0; i < NLDS; ++i) {
        unsigned v;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(s_addr));
        acc_u ^= v + i;
    }
    float x = a;
#pragma unroll
    for (int i = 0; i < NFMA; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(b), "f"(a));
    out[blockIdx.x * blockDim.x + t] = x;
    tag[blockIdx.x * blockDim.x + t] = acc_u;
}
