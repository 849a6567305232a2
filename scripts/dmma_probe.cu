// FP64 tensor-core probe for sm_100a: fragment layout check and throughput of
// mma.sync.aligned.m8n8k4.row.col.f64 (one warp instruction = 8x8x4 = 256 FMAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe scripts/dmma_probe.cu
// Layout assumed (PTX ISA, m8n8k4 .f64): lane l holds A[l/4][l%4], B[l%4][l/4],
// C/D[l/4][2(l%4)], C/D[l/4][2(l%4)+1].
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void layout_kernel(const double *A, const double *B, double *D) {
    const int l = threadIdx.x;
    double d0 = 0, d1 = 0;
    dmma(d0, d1, A[(l / 4) * 4 + l % 4], B[(l % 4) * 8 + l / 4]);
    D[(l / 4) * 8 + 2 * (l % 4)] = d0;
    D[(l / 4) * 8 + 2 * (l % 4) + 1] = d1;
}

template <int NACC>
__global__ void tput_kernel(double *out, int iters, double a, double b) {
    double d[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(d[i][0], d[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += d[i][0] + d[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
    double d[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) d[i] = fma(a, d[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// mixed: every warp interleaves NACC DMMA chains with 16 DFMA chains (are the FP64 tensor and the
// FP64 vector pipes separate?)
__global__ void mixed_kernel(double *out, int iters, double a, double b) {
    double d[8][2], f[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            dmma(d[i][0], d[i][1], a, b);
            f[2 * i] = fma(a, f[2 * i], b);
            f[2 * i + 1] = fma(a, f[2 * i + 1], b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double hA[32], hB[32], hD[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i * 0.37; hB[i] = 2.0 - i * 0.11; }
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c];
            ref[r * 8 + c] = s;
        }
    double *dA, *dB, *dD, *dO;
    cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    layout_kernel<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hD[i] - ref[i]) / fabs(ref[i]));
    printf("layout: max rel err %.3e (%s)\n", err, err < 1e-13 ? "layout as assumed (differences are rounding order)" : "MISMATCH");

    const int blocks = 148 * 4, threads = 256, iters = 4096;
    cudaMalloc(&dO, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch, double flops) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-22s %8.3f ms  %7.2f TFLOP/s\n", name, ms, flops / (ms * 1e-3) / 1e12);
    };
    const double warps = blocks * threads / 32.0;
    run("dmma 4 acc", [&] { tput_kernel<4><<<blocks, threads>>>(dO, iters, 1.0000001, 0.9999999); },
        warps * iters * 4 * 512.0);
    run("dmma 8 acc", [&] { tput_kernel<8><<<blocks, threads>>>(dO, iters, 1.0000001, 0.9999999); },
        warps * iters * 8 * 512.0);
    run("dfma 16 chains", [&] { dfma_kernel<<<blocks, threads>>>(dO, iters, 1.0000001, 1e-9); },
        (double)blocks * threads * iters * 16 * 2.0);
    // mixed: 8 DMMA (8*512 flops per warp) + 16 DFMA (16*32*2 flops per warp) per iteration
    run("mixed 8 dmma+16 dfma", [&] { mixed_kernel<<<blocks, threads>>>(dO, iters, 1.0000001, 0.9999999); },
        warps * iters * (8 * 512.0 + 16 * 64.0));
    run("dmma 8 acc (alone)", [&] { tput_kernel<8><<<blocks, threads>>>(dO, iters, 1.0000001, 0.9999999); },
        warps * iters * 8 * 512.0);
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
