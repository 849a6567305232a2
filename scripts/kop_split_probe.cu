// Probe for the next-round operator split: K P = Kx A + Mx B with
//   A = (My (x) Mz) P,   B = (Ky (x) Mz + My (x) Kz) P,   P = U + tau V,
// computed by a y/z-only kernel (no x-pass, no shared-memory Y tile): thread = (column, 2 rows),
// register window of 2 + 2p rows of P per plane, scatter rings of A and B over 2p + 1 pending
// planes, 16-byte zero-filling cp.async copies of the raw U, V planes, one barrier per plane.
// HBM: read U, V; write P, A, B = 40 B/DOF.  Interior Toeplitz rows (p = 3, uniform mesh); the
// domain edges are zero-filled (the probe measures the streaming kernel, not boundary rows).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o kop_split_probe scripts/kop_split_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int P = 3, W = 2 * P + 1;
constexpr int TX = 32, TY = 16, RY = 2, THREADS = TX * TY / RY, NPF = 4;
constexpr int HY = TY + 2 * P, HN = TX * HY;  // raw plane tile (no x halo: no x-pass)
__constant__ double cM[W], cK[W];              // Toeplitz rows (the same in y and z here)

__device__ __forceinline__ void cp16(unsigned s, const double *g, unsigned nb) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(nb) : "memory");
}

__global__ void __launch_bounds__(THREADS, 2)
    yz_kernel(const double *__restrict__ U, const double *__restrict__ V, double *__restrict__ Pout,
              double *__restrict__ A, double *__restrict__ B, double tau, int n0, int n1, int n2, long sy, long sz,
              int zlen) {
    __shared__ __align__(16) double ring[NPF][2][HN];
    const int tid = threadIdx.x, cx = tid % TX, g = tid / TX;  // rows 2g, 2g + 1 of the tile
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int z0 = blockIdx.z * zlen, z1 = min(n2, z0 + zlen), kk0 = z0 - P, npl = z1 - z0 + 2 * P;
    // copies: 16-byte pieces e = tid + THREADS m of the [HY][TX/2] plane
    constexpr int NPC = HN / 2, NS = (NPC + THREADS - 1) / THREADS;
    int goff[NS];
    unsigned ok = 0;
    for (int m = 0; m < NS; ++m) {
        const int e = tid + m * THREADS, hy = e / (TX / 2), hx = 2 * (e % (TX / 2));
        const int X = x0 + hx, Y = y0 - P + hy;
        const bool in = e < NPC && X < n0 && Y >= 0 && Y < n1;
        goff[m] = in ? (int)(Y * sy + X) : 0;
        if (in) ok |= 1u << m;
    }
    const unsigned rs = (unsigned)__cvta_generic_to_shared(&ring[0][0][0]) + 16u * tid;
    auto issue = [&](int ii) {
        if (ii < npl) {
            const int kk = kk0 + ii;
            const bool kv = kk >= 0 && kk < n2;
            const unsigned su = rs + 8u * (unsigned)((ii % NPF) * 2 * HN);
            for (int m = 0; m < NS; ++m) {
                if (tid + m * THREADS >= NPC) break;
                const unsigned nb = (kv && (ok >> m & 1)) ? 16u : 0u;
                const long o = kv ? (long)kk * sz + goff[m] : 0;
                cp16(su + 16u * m * THREADS, U + o, nb);
                cp16(su + 16u * m * THREADS + 8u * HN, V + o, nb);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    const int X = x0 + cx, Y0 = y0 + RY * g;
    const bool own0 = X < n0 && Y0 < n1, own1 = X < n0 && Y0 + 1 < n1;
    const long oxy = (long)Y0 * sy + X;
    double a0[W], a1[W], b0[W], b1[W];  // pending planes kk - p .. kk + p (slot c = plane kk - p + c)
    for (int c = 0; c < W; ++c) a0[c] = a1[c] = b0[c] = b1[c] = 0.0;
    for (int i = 0; i < NPF - 1; ++i) issue(i);
    for (int ii = 0; ii < npl; ++ii) {
        const int kk = kk0 + ii;
        asm volatile("cp.async.wait_group %0;\n" ::"n"(NPF - 2) : "memory");
        __syncthreads();  // plane ii landed; slot (ii - 1) % NPF free
        issue(ii + NPF - 1);
        const double *bu = &ring[ii % NPF][0][0] + (RY * g) * TX + cx, *bv = bu + HN;
        double pr[RY + 2 * P];
#pragma unroll
        for (int r = 0; r < RY + 2 * P; ++r) pr[r] = fma(tau, bv[r * TX], bu[r * TX]);
        if (kk >= z0 && kk < z1) {
            if (own0) Pout[(long)kk * sz + oxy] = pr[P];
            if (own1) Pout[(long)kk * sz + oxy + sy] = pr[P + 1];
        }
        double y1[RY], y2[RY];  // My P, Ky P of rows 2g, 2g + 1 (pair-sum form of the symmetric rows)
#pragma unroll
        for (int r = 0; r < RY; ++r) {
            y1[r] = cM[P] * pr[r + P];
            y2[r] = cK[P] * pr[r + P];
#pragma unroll
            for (int d = 1; d <= P; ++d) {
                const double sp = pr[r + P - d] + pr[r + P + d];
                y1[r] = fma(cM[P + d], sp, y1[r]);
                y2[r] = fma(cK[P + d], sp, y2[r]);
            }
        }
        // z scatter: output plane kk - p + c gets Mz(k, kk) y1 (A) and Mz y2 + Kz y1 (B)
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const double m = cM[c], k = cK[c];
            a0[c] = fma(m, y1[0], a0[c]);
            a1[c] = fma(m, y1[1], a1[c]);
            b0[c] = fma(k, y1[0], fma(m, y2[0], b0[c]));
            b1[c] = fma(k, y1[1], fma(m, y2[1], b1[c]));
        }
        const int ko = kk - P;  // slot 0 is complete
        if (ko >= z0 && ko < z1) {
            const long o = (long)ko * sz + oxy;
            if (own0) { A[o] = a0[0]; B[o] = b0[0]; }
            if (own1) { A[o + sy] = a1[0]; B[o + sy] = b1[0]; }
        }
#pragma unroll
        for (int c = 0; c < W - 1; ++c) {
            a0[c] = a0[c + 1]; a1[c] = a1[c + 1]; b0[c] = b0[c + 1]; b1[c] = b1[c + 1];
        }
        a0[W - 1] = a1[W - 1] = b0[W - 1] = b1[W - 1] = 0.0;
    }
}

static void run(int n, int zlen, double tau, const double *dU, const double *dV, double *dP, double *dA, double *dB,
                long sy, long sz, cudaStream_t s) {
    dim3 grd((n + TX - 1) / TX, (n + TY - 1) / TY, (n + zlen - 1) / zlen);
    yz_kernel<<<grd, THREADS, 0, s>>>(dU, dV, dP, dA, dB, tau, n, n, n, sy, sz, zlen);
}

int main(int argc, char **argv) {
    const double h = 1.0 / 512;
    double m[W] = {1, 120, 1191, 2416, 1191, 120, 1}, k[W] = {-1, -24, -15, 80, -15, -24, -1};
    for (int c = 0; c < W; ++c) { m[c] *= h / 5040.0; k[c] /= 120.0 * h; }
    cudaMemcpyToSymbol(cM, m, sizeof m);
    cudaMemcpyToSymbol(cK, k, sizeof k);
    const double tau = 5e-4;
    // ---- correctness on a small grid against a plain CPU evaluation of the definitions
    {
        const int n = 45;
        const long sy = 48, sz = sy * n, N = sz * n;
        std::vector<double> u(N, 0.0), v(N, 0.0);
        srand(3);
        for (int z = 0; z < n; ++z)
            for (int y = 0; y < n; ++y)
                for (int x = 0; x < n; ++x) {
                    u[z * sz + y * sy + x] = rand() / (double)RAND_MAX - 0.5;
                    v[z * sz + y * sy + x] = rand() / (double)RAND_MAX - 0.5;
                }
        double *dU, *dV, *dP, *dA, *dB;
        for (double **p : {&dU, &dV, &dP, &dA, &dB}) { cudaMalloc(p, N * 8); cudaMemset(*p, 0, N * 8); }
        cudaMemcpy(dU, u.data(), N * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(dV, v.data(), N * 8, cudaMemcpyHostToDevice);
        run(n, 13, tau, dU, dV, dP, dA, dB, sy, sz, 0);
        std::vector<double> A(N), B(N);
        cudaMemcpy(A.data(), dA, N * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(B.data(), dB, N * 8, cudaMemcpyDeviceToHost);
        auto Pv = [&](int x, int y, int z) {
            if (y < 0 || y >= n || z < 0 || z >= n) return 0.0;
            const long o = z * sz + y * sy + x;
            return u[o] + tau * v[o];
        };
        double err = 0.0, ref = 0.0;
        for (int z = 0; z < n; ++z)
            for (int y = 0; y < n; ++y)
                for (int x = 0; x < n; ++x) {
                    double ea = 0.0, eb = 0.0;  // A = My Mz P, B = Ky Mz P + My Kz P (rows extended by zero)
                    for (int dy = -P; dy <= P; ++dy)
                        for (int dz = -P; dz <= P; ++dz) {
                            const double pv = Pv(x, y + dy, z + dz);
                            ea += m[dy + P] * m[dz + P] * pv;
                            eb += (k[dy + P] * m[dz + P] + m[dy + P] * k[dz + P]) * pv;
                        }
                    const long o = z * sz + y * sy + x;
                    err = fmax(err, fmax(fabs(A[o] - ea), fabs(B[o] - eb)));
                    ref = fmax(ref, fmax(fabs(ea), fabs(eb)));
                }
        printf("check n=%d: max |err| / max |ref| = %.3e (%s)\n", n, err / ref, err / ref < 1e-13 ? "ok" : "FAIL");
        for (double *p : {dU, dV, dP, dA, dB}) cudaFree(p);
    }
    // ---- throughput at c4 (515^3, pitch 520)
    const int n = 515;
    const long sy = 520, sz = sy * n, N = sz * n;
    double *dU, *dV, *dP, *dA, *dB;
    for (double **p : {&dU, &dV, &dP, &dA, &dB}) { cudaMalloc(p, N * 8); cudaMemset(*p, 0, N * 8); }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int zl : {129, 104, 86, 65, 52}) {
        run(n, zl, tau, dU, dV, dP, dA, dB, sy, sz, 0);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) run(n, zl, tau, dU, dV, dP, dA, dB, sy, sz, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 10;
        const double bytes = 40.0 * (double)n * n * n;
        printf("515^3 zlen %3d: %.3f ms per launch, %.0f GB/s at 40 B/DOF (%s)\n", zl, ms, bytes / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
