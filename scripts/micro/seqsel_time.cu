// Time the re-decision (sequential_select_warp, ct_select.cuh) on one warp
// against the one-thread sequential loop, same weights, same answer.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <cmath>
#include "ct_select.cuh"
using namespace ct;
__global__ void k_warp(const double* w, int64_t n, double u, int64_t* out) {
    int64_t a = sequential_select_warp(w, n, u, threadIdx.x & 31);
    if (threadIdx.x == 0) out[0] = a;
}
__global__ void k_pass(const double* w, int64_t n, int64_t* out) {   // one seq_scan pass
    double c = 0.0;
    int64_t a = seq_scan(w, n, 0, c, -1.0, threadIdx.x & 31);
    if (threadIdx.x == 0) { out[0] = a; out[1] = (int64_t)c; }
}
__global__ void k_pass_ck(const double* w, int64_t n, int64_t* out) {   // pass 1 with checkpoints
    double ck[SEQ_CK];
    for (int q = 0; q < SEQ_CK; ++q) ck[q] = 0.0;
    const int64_t nblocks = (n + SEQ_BLK - 1) / SEQ_BLK;
    const int64_t per = max((int64_t)1, (nblocks + 32 * SEQ_CK - 1) / (32 * SEQ_CK));
    double c = 0.0;
    int64_t a = seq_scan(w, n, 0, c, -1.0, threadIdx.x & 31, ck, per);
    if (threadIdx.x == 0) { out[0] = a; out[1] = (int64_t)ck[1]; }
}
__global__ void k_seq(const double* w, int64_t n, double u, int64_t* out) {
    if (threadIdx.x == 0) out[0] = sequential_select(w, n, u);
}
int main() {
    const int64_t n = 1 << 20;
    std::vector<double> h(n);
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> d(0.3, 2.0);
    for (auto& x : h) { double y = std::pow(d(g), 8); x = y > 256 ? 256 : (y < 1e-4 ? 1e-4 : y); }
    double* w; int64_t* o;
    cudaMalloc(&w, n * 8); cudaMalloc(&o, 16);
    cudaMemcpy(w, h.data(), n * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms; int64_t r1, r2;
    k_warp<<<1, 32>>>(w, n, 0.37, o); cudaDeviceSynchronize();
    cudaEventRecord(a); k_warp<<<1, 32>>>(w, n, 0.37, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); cudaMemcpy(&r1, o, 8, cudaMemcpyDeviceToHost);
    printf("warp select: %.3f ms -> %lld\n", ms, (long long)r1);
    cudaEventRecord(a); k_pass<<<1, 32>>>(w, n, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("one binade pass: %.3f ms\n", ms);
    cudaEventRecord(a); k_pass_ck<<<1, 32>>>(w, n, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("one pass with checkpoints: %.3f ms\n", ms);
    cudaEventRecord(a); k_seq<<<1, 32>>>(w, n, 0.37, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); cudaMemcpy(&r2, o, 8, cudaMemcpyDeviceToHost);
    printf("scalar select: %.3f ms -> %lld (%s)\n", ms, (long long)r2, r1 == r2 ? "same" : "DIFFERENT");
    return r1 == r2 ? 0 : 1;
}
