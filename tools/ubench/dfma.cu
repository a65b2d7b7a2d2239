// Microbenchmark: DFMA throughput on sm_100a vs warps per SM and independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double *out, int iters, double a, double b) {
    double acc[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 12345.678) out[0] = s;
}
template <int CH>
void run(int warps, double *d) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<CH><<<148, warps * 32>>>(d, 16, 0.999, 1e-3);
    cudaEventRecord(e0);
    k<CH><<<148, warps * 32>>>(d, iters, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = 148.0 * warps * 32 * (double)iters * 8 * CH;
    printf("warps/SM %2d chains %2d: %.2f TFMA/s  (%.1f FMA/clk/SM @1.965GHz)\n", warps, CH, fma / ms / 1e9,
           fma / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
    double *d; cudaMalloc(&d, 8);
    for (int w : {2, 4, 8, 16, 32}) { run<1>(w, d); run<2>(w, d); run<4>(w, d); run<8>(w, d); }
    return 0;
}
