// FFMA vs FFMA2 (fma.rn.f32x2, sm_100) issue/throughput on one B200:
// 8 independent chains per thread, 148*8 blocks x 256 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_rate.cu -o ffma2_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

__global__ void k_ffma(float* out, int iters, float s) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 0.001f + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], s, 0.5f * k + 0.1f);
    float r = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) r += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_ffma3(float* out, int iters, float s, float t) {
    float a[8];
    float c = t * threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 0.001f + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], s, c);   // 3-register form
    float r = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) r += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_ffma2(float* out, int iters, float s, float t) {
    unsigned long long a[8], b, c;
    float c0 = t * threadIdx.x;
    asm("mov.b64 %0, {%1, %1};" : "=l"(b) : "f"(s));
    asm("mov.b64 %0, {%1, %1};" : "=l"(c) : "f"(c0));
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float lo = threadIdx.x * 0.001f + k, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a[k]) : "f"(lo), "f"(hi));
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma2(a[k], b, c);
    float r = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[k]));
        r += lo + hi;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    float* out;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int pass = 0; pass < 2; ++pass) {
        for (int which = 0; which < 3; ++which) {
            cudaEventRecord(e0);
            if (which == 0) k_ffma<<<blocks, threads>>>(out, iters, 0.999f);
            if (which == 1) k_ffma3<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
            if (which == 2) k_ffma2<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double lanes = (double)blocks * threads * iters * 8 * (which == 2 ? 2 : 1);
            if (pass == 1)
                printf("%s: %.3f ms, %.1f TFLOP/s (2 flop per fma lane-op)\n",
                       which == 0 ? "FFMA imm" : (which == 1 ? "FFMA 3-reg" : "FFMA2"), ms,
                       2.0 * lanes / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
