// Phase timing of sweep_kernel (clock64 per phase, CTAs 0..7, first tile, threads 0 and last).
#define ADS_PHASE_TIMING
#include "../../paper_1911_08158_b200/csrc/kernels.cu"
#include "../../paper_1911_08158_b200/csrc/host_setup.h"
#include <vector>
using namespace ads;
template <class T> T *up(const std::vector<T> &v) { T *d; cudaMalloc(&d, sizeof(T) * std::max<size_t>(v.size(), 1)); cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice); return d; }
int main(int argc, char **argv) {
    int nel = argc > 1 ? atoi(argv[1]) : 127, p = argc > 2 ? atoi(argv[2]) : 3, dir = argc > 3 ? atoi(argv[3]) : 1;
    double tau = 5e-4;
    Space1D s; build_space(p, nel, 1, s);
    int n = s.n;
    Band A(n, p); for (size_t q = 0; q < A.v.size(); ++q) A.v[q] = s.M.v[q] + tau * tau / 4 * s.K.v[q];
    A.at(0, 0) = 1; A.at(n - 1, n - 1) = 1;
    LUFactors f; banded_lu(A, f, true);
    std::vector<int> cs; int L = choose_chunks(n, p, 32, cs);
    const int C = (int)cs.size() - 1, npad = C * L;
    LUFactors fp = f; fp.n = npad; fp.l.resize((size_t)npad * p, 0.0); fp.us.resize((size_t)npad * p, 0.0); fp.dinv.resize(npad, 1.0);
    std::vector<int> csp(cs); csp[C] = npad;
    PartTables pt; build_part_tables(fp, csp, pt); f = fp;
    SweepArgs a;
    a.t.l = up(f.l); a.t.us = up(f.us); a.t.dinv = up(f.dinv); a.t.phif = up(pt.phif); a.t.phib = up(pt.phib); a.t.cs = up(pt.cs);
    a.t.n = n; a.t.C = pt.C; a.t.levels = pt.levels; a.t.L = L;
    int c_lo = (f.i_lo + L - 1) / L, c_hi = f.i_hi / L;
    a.t.i_lo = c_hi > c_lo ? c_lo * L : 0; a.t.i_hi = c_hi > c_lo ? c_hi * L : 0;
    for (int k = 0; k < p; ++k) { a.t.lc[k] = f.l[a.t.i_lo * p + k]; a.t.usc[k] = f.us[a.t.i_lo * p + k]; }
    a.t.dic = f.dinv[a.t.i_lo];
    long N = (long)n * n * n;
    double *x, *y; cudaMalloc(&x, N * 8); cudaMalloc(&y, N * 8); cudaMemset(x, 0, N * 8);
    a.in = x; a.out = y; a.geo.n0 = a.geo.n1 = a.geo.n2 = n; a.geo.sy = n; a.geo.sz = (long)n * n; a.dir = dir; a.mode = 0;
    printf("n=%d p=%d L=%d C=%d levels=%d uniform rows [%d,%d)\n", n, p, L, pt.C, pt.levels, a.t.i_lo, a.t.i_hi);
    for (int it = 0; it < 3; ++it) launch_sweep(p, a, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); for (int it = 0; it < 10; ++it) launch_sweep(p, a, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("sweep dir %d: %.3f ms  (%s)\n", dir, ms / 10, cudaGetErrorString(cudaGetLastError()));
    long long h[64][16]; cudaMemcpyFromSymbol(h, g_phase, sizeof(h));
    const char *nm[] = {"start", "loaded", "solved", "stored"};
    for (int b = 0; b < 6; ++b) {
        if (b % 3 == 2) continue;
        printf("CTA %d thr %s:", b / 3, b % 3 == 0 ? "0 " : "80");
        for (int k = 1; k <= 3; ++k) printf("  %s %lld", nm[k], h[b][k] - h[b][k - 1]);
        printf("  | total %lld cycles\n", h[b][3] - h[b][0]);
    }
    long long sub[4][8]; cudaMemcpyFromSymbol(sub, g_sub, sizeof(sub));
    const char *sn[] = {"", "pass1", "scanf", "pass2", "pass3", "scanb", "pass4"};
    for (int b = 0; b < 2; ++b) { printf("solve sub-phases (CTA0, last tile, %s):", b ? "warp2 lane10" : "warp0 lane0");
        for (int k = 1; k <= 6; ++k) printf(" %s %lld", sn[k], sub[b][k] - sub[b][k-1]); printf("\n"); }
    return 0;
}
