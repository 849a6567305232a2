// modal_tc.cu -- the f3 modal transforms (the paper's §3
// eigen-decomposition) as hand-written FP64 tensor-core GEMMs (sm_100a DMMA,
// mma.sync.m8n8k4.f64) with the mirror fold / unfold fused into the operand loads / the epilogue.
//
// Along an axis of length n (h = n / 2, H = h + n % 2) every line u is mapped by the even / odd
// halves of the 1D maps (host_setup modal_basis: each eigenvector has an exact parity):
//   forward  c_even = Q_e t_e,  c_odd = Q_o t_o,   t_e(k) = u(k) + u(n-1-k) (k < h), u(h) (k = h, n odd),
//                                                    t_o(k) = u(k) - u(n-1-k);
//            modal slots along the axis: [even (ne) | odd (no) | zero];
//   inverse  t_e = P_e c_even, t_o = P_o c_odd;  u(i) = t_e(i) + t_o(i), u(n-1-i) = t_e(i) - t_o(i),
//            u(h) = t_e(h) (n odd).
// Q_*, P_* are column-major (the layout ads_modal_basis builds).  A line is addressed as
// element k at k ks + l ls + b bs (line l of batch b): x lines are contiguous (ks = 1), y / z
// lines are adjacent (ls = 1).  The fold costs one add per loaded operand and no HBM pass.
//
// Tiles: forward BM x BN = 64 x 64 per CTA (4 warps of 32 x 32, 4 x 4 DMMA tiles each), inverse
// 32 x 64 per CTA for both halves at once (4 warps of 32 x 16 per half; the unfold needs the even
// and odd results of the same rows), BK = 16, double-buffered shared memory filled from registers
// (the loads of the next K tile are in flight during the current tile's DMMAs).  Rows beyond the
// last full M tile (n = 515: one or two) take a CUDA-core tail path.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ads {

namespace {

constexpr int MG_BN = 64, MG_BK = 16, MG_THREADS = 128;
constexpr int MG_PA = MG_BK + 4;  // A tile pitch: m rows of BK (+4: conflict-free fragment reads)
constexpr int MG_PT = MG_BN + 4;  // T tile pitch: k rows of BN

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// u(k) of line l, batch b
__device__ __forceinline__ double el(const ModalGemmArgs &g, const double *base, int k, long loff) {
    return __ldg(base + (long)k * g.ks + loff);
}

// folded operand t(k) of half q for the line at loff (0 beyond K)
__device__ __forceinline__ double fold(const ModalGemmArgs &g, int q, int k, long loff) {
    const int h = g.n / 2;
    if (q == 0) {
        if (k < h) return el(g, g.in, k, loff) + el(g, g.in, g.n - 1 - k, loff);
        return (k == h && (g.n & 1)) ? el(g, g.in, h, loff) : 0.0;
    }
    return k < h ? el(g, g.in, k, loff) - el(g, g.in, g.n - 1 - k, loff) : 0.0;
}

// ---- forward: one half q, rows [m0, m0 + 64) of C = A t (A = Q_q, M x K, column-major)
template <bool KX>
__global__ void __launch_bounds__(MG_THREADS) modal_fwd_kernel(const ModalGemmArgs g) {
    __shared__ __align__(16) double As[2][64 * MG_PA];
    __shared__ __align__(16) double Ts[2][MG_BK * MG_PT];
    const int q = blockIdx.z & 1, b = blockIdx.z >> 1;
    const int M = q ? g.no : g.ne, K = q ? g.hh : g.H;
    const double *A = q ? g.Qo : g.Qe;
    const int slot0 = q ? g.ne : 0;
    const int mt = blockIdx.x, l0 = blockIdx.y * MG_BN;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long boff = (long)b * g.bs;
    const int mfull = M / 64;
    if (mt > mfull || M == 0) return;
    if (mt == mfull) {  // tail rows [64 mfull, M) on CUDA cores: thread per line, 8 rows at a time
        const int r0 = 64 * mfull;
        if (r0 >= M) return;
        for (int li = tid; li < MG_BN; li += MG_THREADS) {
            const int l = l0 + li;
            if (l >= g.nl) break;
            const long loff = (long)l * g.ls + boff;
            for (int rc = r0; rc < M; rc += 8) {
                double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int k = 0; k < K; ++k) {
                    const double t = fold(g, q, k, loff);
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (rc + r < M) acc[r] = fma(__ldg(A + (rc + r) + (long)k * M), t, acc[r]);
                }
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    if (rc + r < M) g.out[(long)(slot0 + rc + r) * g.ks + loff] = acc[r];
            }
        }
        return;
    }
    const int m0 = 64 * mt;
    // zero the unused slots [ne + no, n) of these lines once (one CTA per line tile)
    if (q == 1 && mt == 0)
        for (int e = tid; e < MG_BN * (g.n - g.ne - g.no); e += MG_THREADS) {
            const int l = l0 + e % MG_BN, s = g.ne + g.no + e / MG_BN;
            if (l < g.nl) g.out[(long)s * g.ks + (long)l * g.ls + boff] = 0.0;
        }
    // operand staging: A (64 x BK) 8 values per thread, t (BK x 64) 8 folded values per thread
    double ra[8], rt[8];
    auto load = [&](int k0) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int mm = tid & 63, kk = (tid >> 6) + 2 * r;
            const int k = k0 + kk;
            ra[r] = k < K ? __ldg(A + (m0 + mm) + (long)k * M) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int kk, nn;
            if (KX) {  // x lines: consecutive k contiguous
                kk = tid & 15;
                nn = (tid >> 4) + 8 * r;
            } else {   // y / z: consecutive lines contiguous
                nn = tid & 63;
                kk = (tid >> 6) + 2 * r;
            }
            const int k = k0 + kk, l = l0 + nn;
            rt[r] = (k < K && l < g.nl) ? fold(g, q, k, (long)l * g.ls + boff) : 0.0;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int mm = tid & 63, kk = (tid >> 6) + 2 * r;
            As[buf][mm * MG_PA + kk] = ra[r];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int kk, nn;
            if (KX) {
                kk = tid & 15;
                nn = (tid >> 4) + 8 * r;
            } else {
                nn = tid & 63;
                kk = (tid >> 6) + 2 * r;
            }
            Ts[buf][kk * MG_PT + nn] = rt[r];
        }
    };
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int wm = (w >> 1) * 32, wn = (w & 1) * 32;
    const int nk = (K + MG_BK - 1) / MG_BK;
    load(0);
    store(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) load((kt + 1) * MG_BK);
#pragma unroll
        for (int s = 0; s < MG_BK / 4; ++s) {
            double a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][(wm + 8 * i + (lane >> 2)) * MG_PA + 4 * s + (lane & 3)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = Ts[buf][(4 * s + (lane & 3)) * MG_PT + wn + 8 * j + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], bb[j]);
        }
        if (kt + 1 < nk) store(buf ^ 1);
        __syncthreads();
    }
    // epilogue: acc[i][j][e] = C(m0 + wm + 8 i + lane/4, l0 + wn + 8 j + 2 (lane%4) + e)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + wm + 8 * i + (lane >> 2);
        const long ro = (long)(slot0 + m) * g.ks + boff;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int l = l0 + wn + 8 * j + 2 * (lane & 3) + e;
                if (l < g.nl) g.out[ro + (long)l * g.ls] = acc[i][j][e];
            }
    }
}

// ---- inverse: rows [i0, i0 + 32) of t_e = P_e c_e and t_o = P_o c_o, unfolded into u
template <bool KX>
__global__ void __launch_bounds__(MG_THREADS) modal_inv_kernel(const ModalGemmArgs g) {
    __shared__ __align__(16) double As[2][32 * MG_PA];
    __shared__ __align__(16) double Ts[2][MG_BK * MG_PT];
    const int b = blockIdx.z, mt = blockIdx.x, l0 = blockIdx.y * MG_BN;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long boff = (long)b * g.bs;
    const int H = g.H, hh = g.hh, n = g.n;
    const int mfull = H / 32;
    if (mt > mfull) return;
    if (mt == mfull) {  // tail rows [32 mfull, H): thread per line
        const int r0 = 32 * mfull;
        if (r0 >= H) return;
        for (int li = tid; li < MG_BN; li += MG_THREADS) {
            const int l = l0 + li;
            if (l >= g.nl) break;
            const long loff = (long)l * g.ls + boff;
            for (int i = r0; i < H; ++i) {
                double te = 0.0, to = 0.0;
                for (int k = 0; k < g.ne; ++k) te = fma(__ldg(g.Pe + i + (long)k * H), el(g, g.in, k, loff), te);
                if (i < hh)
                    for (int k = 0; k < g.no; ++k) to = fma(__ldg(g.Po + i + (long)k * hh), el(g, g.in, g.ne + k, loff), to);
                if (i < hh) {
                    g.out[(long)i * g.ks + loff] = te + to;
                    g.out[(long)(n - 1 - i) * g.ks + loff] = te - to;
                } else {
                    g.out[(long)i * g.ks + loff] = te;  // the middle position of an odd axis
                }
            }
        }
        return;
    }
    const int i0 = 32 * mt;
    double ra[4], rt[8];
    // half q: A = q ? P_o (hh x no) : P_e (H x ne); operand rows c(k) at slot (q ? ne : 0) + k
    auto load = [&](int q, int k0) {
        const int MR = q ? hh : H, K = q ? g.no : g.ne;
        const double *A = q ? g.Po : g.Pe;
        const int s0 = q ? g.ne : 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int mm = tid & 31, kk = (tid >> 5) + 4 * r;
            const int k = k0 + kk, m = i0 + mm;
            ra[r] = (k < K && m < MR) ? __ldg(A + m + (long)k * MR) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int kk, nn;
            if (KX) {
                kk = tid & 15;
                nn = (tid >> 4) + 8 * r;
            } else {
                nn = tid & 63;
                kk = (tid >> 6) + 2 * r;
            }
            const int k = k0 + kk, l = l0 + nn;
            rt[r] = (k < K && l < g.nl) ? el(g, g.in, s0 + k, (long)l * g.ls + boff) : 0.0;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int mm = tid & 31, kk = (tid >> 5) + 4 * r;
            As[buf][mm * MG_PA + kk] = ra[r];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int kk, nn;
            if (KX) {
                kk = tid & 15;
                nn = (tid >> 4) + 8 * r;
            } else {
                nn = tid & 63;
                kk = (tid >> 6) + 2 * r;
            }
            Ts[buf][kk * MG_PT + nn] = rt[r];
        }
    };
    double acc[2][4][2][2];  // [half][m tile][n tile][e]: warp tile 32 x 16 per half
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;
    const int wn = w * 16;
    // one K loop over the even half's tiles followed by the odd half's (tile index kt over both)
    const int nke = (g.ne + MG_BK - 1) / MG_BK, nko = (g.no + MG_BK - 1) / MG_BK, nk = nke + nko;
    if (nk == 0) return;
    auto tile_q = [&](int kt) { return kt < nke ? 0 : 1; };
    auto tile_k0 = [&](int kt) { return (kt < nke ? kt : kt - nke) * MG_BK; };
    load(tile_q(0), tile_k0(0));
    store(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1, q = tile_q(kt);
        if (kt + 1 < nk) load(tile_q(kt + 1), tile_k0(kt + 1));
#pragma unroll
        for (int s = 0; s < MG_BK / 4; ++s) {
            double a[4], bb[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][(8 * i + (lane >> 2)) * MG_PA + 4 * s + (lane & 3)];
#pragma unroll
            for (int j = 0; j < 2; ++j) bb[j] = Ts[buf][(4 * s + (lane & 3)) * MG_PT + wn + 8 * j + (lane >> 2)];
            if (q == 0) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) dmma(acc[0][i][j], a[i], bb[j]);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) dmma(acc[1][i][j], a[i], bb[j]);
            }
        }
        if (kt + 1 < nk) store(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = i0 + 8 * i + (lane >> 2);
        if (r >= H) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int l = l0 + wn + 8 * j + 2 * (lane & 3) + e;
                if (l >= g.nl) continue;
                const long lo = (long)l * g.ls + boff;
                const double te = acc[0][i][j][e], to = acc[1][i][j][e];
                if (r < hh) {
                    g.out[(long)r * g.ks + lo] = te + to;
                    g.out[(long)(n - 1 - r) * g.ks + lo] = te - to;
                } else {
                    g.out[(long)r * g.ks + lo] = te;
                }
            }
    }
}

}  // namespace

int launch_modal_gemm(const ModalGemmArgs &g, cudaStream_t s) {
    if (g.nl <= 0 || g.nb <= 0) return 0;
    const unsigned ny = (unsigned)((g.nl + MG_BN - 1) / MG_BN);
    if (ny > 65535u || g.nb > 32767) return -1;
    if (!g.inverse) {
        const int mt = std::max(g.ne, g.no) / 64 + 1;
        dim3 grd(mt, ny, 2 * g.nb);
        if (g.ks == 1) modal_fwd_kernel<true><<<grd, MG_THREADS, 0, s>>>(g);
        else modal_fwd_kernel<false><<<grd, MG_THREADS, 0, s>>>(g);
    } else {
        dim3 grd(g.H / 32 + 1, ny, g.nb);
        if (g.ks == 1) modal_inv_kernel<true><<<grd, MG_THREADS, 0, s>>>(g);
        else modal_inv_kernel<false><<<grd, MG_THREADS, 0, s>>>(g);
    }
    return 0;
}

}  // namespace ads
