// Microbenchmark: achievable HBM bandwidth of the sweep access patterns as pure copies.
// Field n^3 doubles (n = 515).  A CTA owns XW adjacent x-lines x C chunks of L elements
// along the sweep axis (stride st elements), like sweep_kernel; loads all, stores all.
#include <cstdio>
#include <cuda_runtime.h>
template <int XW, int L>
__global__ void __launch_bounds__(XW * 32) pat(const double *__restrict__ in, double *__restrict__ out, int n, long sa,
                                               long sb, long st, int na, int C) {
    const int xl = threadIdx.x, c = threadIdx.y;
    const long base = (long)blockIdx.y * sb + (long)(blockIdx.x * XW) * sa;
    const bool valid = blockIdx.x * XW + xl < na;
    const int s = c * L, len = min(L, n - s);
    double v[L];
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = (valid && j < len) ? __ldg(in + base + xl + (long)(s + j) * st) : 0.0;
#pragma unroll
    for (int j = 0; j < L; ++j)
        if (valid && j < len) out[base + xl + (long)(s + j) * st] = v[j] * 1.0000001;
}
__global__ void copy_flat(const double *__restrict__ in, double *__restrict__ out, long N) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < N; i += (long)gridDim.x * blockDim.x) out[i] = in[i] * 1.0000001;
}
template <int XW, int L>
float run(const double *in, double *out, int n, int dir) {
    const long sy = n, sz = (long)n * n;
    long st = dir == 1 ? sy : sz, sb = dir == 1 ? sz : sy;
    int C = (n + L - 1) / L;
    dim3 blk(XW, C), grd((n + XW - 1) / XW, n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 2; ++w) pat<XW, L><<<grd, blk>>>(in, out, n, 1, sb, st, n, C);
    cudaEventRecord(e0);
    for (int w = 0; w < 5; ++w) pat<XW, L><<<grd, blk>>>(in, out, n, 1, sb, st, n, C);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e) printf("err %s\n", cudaGetErrorString(e));
    return ms / 5;
}
int main() {
    const int n = 515;
    const long N = (long)n * n * n;
    double *a, *b;
    cudaMalloc(&a, N * 8); cudaMalloc(&b, N * 8);
    cudaMemset(a, 0, N * 8); cudaMemset(b, 0, N * 8);
    const double GB = 2.0 * N * 8 / 1e9;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    copy_flat<<<148 * 8, 256>>>(a, b, N);
    cudaEventRecord(e0);
    for (int w = 0; w < 5; ++w) copy_flat<<<148 * 8, 256>>>(a, b, N);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("flat copy          %.3f ms  %.0f GB/s\n", ms, GB / ms * 1e3);
    for (int dir = 1; dir <= 2; ++dir) {
        const char *d = dir == 1 ? "y" : "z";
        ms = run<8, 17>(a, b, n, dir);  printf("%s XW=8  L=17 %.3f ms  %.0f GB/s\n", d, ms, GB / ms * 1e3);
        ms = run<16, 17>(a, b, n, dir); printf("%s XW=16 L=17 %.3f ms  %.0f GB/s\n", d, ms, GB / ms * 1e3);
        ms = run<32, 17>(a, b, n, dir); printf("%s XW=32 L=17 %.3f ms  %.0f GB/s\n", d, ms, GB / ms * 1e3);
        ms = run<8, 33>(a, b, n, dir);  printf("%s XW=8  L=33 %.3f ms  %.0f GB/s\n", d, ms, GB / ms * 1e3);
        ms = run<16, 33>(a, b, n, dir); printf("%s XW=16 L=33 %.3f ms  %.0f GB/s\n", d, ms, GB / ms * 1e3);
        ms = run<32, 9>(a, b, n, dir);  printf("%s XW=32 L=9  %.3f ms  %.0f GB/s\n", d, ms, GB / ms * 1e3);
    }
    return 0;
}
