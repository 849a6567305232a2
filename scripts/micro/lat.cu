// Latency microbenchmarks on B200: dependent DFMA chain, LDS chain, SHFL chain, LDG (L1 hit) chain.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double *out, double a, double b, int iters, long long *cyc) {
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_lds(double *out, int iters, long long *cyc) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
    __syncthreads();
    int j = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) j = idx[j];
    }
    long long t1 = clock64();
    out[threadIdx.x] = j;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_shfl(double *out, int iters, long long *cyc) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = __shfl_up_sync(0xffffffffu, x, 1) + 1.0;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_ldg(const int *__restrict__ p, double *out, int iters, long long *cyc) {
    int j = threadIdx.x & 255;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) j = __ldg(p + j);
    }
    long long t1 = clock64();
    out[threadIdx.x] = j;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double *out; long long *cyc, h; int *p;
    cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8); cudaMalloc(&p, 4096 * 4);
    int hp[4096]; for (int i = 0; i < 4096; ++i) hp[i] = (i + 1) & 255;
    cudaMemcpy(p, hp, sizeof hp, cudaMemcpyHostToDevice);
    const int it = 1000;
    for (int w : {1, 4, 8}) {
        k_dfma<<<1, 32 * w>>>(out, 0.999, 1e-3, it, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA dependent chain, %d warp(s)/SM: %.2f cycles per DFMA\n", w, (double)h / (it * 16));
    }
    k_lds<<<1, 32>>>(out, it, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS dependent chain: %.2f cycles\n", (double)h / (it * 16));
    k_shfl<<<1, 32>>>(out, it, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("SHFL.64 (2x SHFL) + DADD chain: %.2f cycles\n", (double)h / (it * 16));
    k_ldg<<<1, 32>>>(p, out, it, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDG L1-hit dependent chain: %.2f cycles\n", (double)h / (it * 16));
    // DFMA throughput: many warps
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k_dfma<<<148 * 8, 256>>>(out, 0.999, 1e-3, 4000, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA throughput: %.1f TFLOP/s (fp64 FMA = 2 flop)\n", 2.0 * 148 * 8 * 256 * 4000.0 * 16 / ms / 1e9);
    return 0;
}
