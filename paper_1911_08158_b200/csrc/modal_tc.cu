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

#include <algorithm>

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
    const int mfull = M / 64;
    const int mt = g.tail_only ? mfull : (int)blockIdx.x, l0 = blockIdx.y * MG_BN;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long boff = (long)b * g.bs;
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
    const int H = g.H, hh = g.hh, n = g.n;
    const int mfull = H / 32;
    const int b = blockIdx.z, mt = g.tail_only ? mfull : (int)blockIdx.x, l0 = blockIdx.y * MG_BN;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long boff = (long)b * g.bs;
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

// ---------------------------------------------------------------------------------------------
// TMA-fed versions of the full tiles: the A tile (the map) and the operand tiles move by TMA into a
// MT_S-stage shared-memory ring (mbarrier completion, one refill per K tile after a CTA barrier);
// the forward operand is loaded twice, as u(k) and as the mirrored block u(n-1-k) (a second box
// whose rows run backwards), and folded while the DMMA fragments are read.  Tile rows are padded
// (+4 doubles: the boxes load 4 extra rows / columns) so every fragment read is conflict-free.
// ---------------------------------------------------------------------------------------------
constexpr int MT_S = 3, MT_THREADS = 128;
constexpr int MT_TSZ = 1280;  // operand tile: 16 k x 68 lines (y, z) or 64 lines x 20 k (x)

__device__ __forceinline__ void mt_wait(unsigned mb, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n MTW_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra MTW_%=;\n}\n" ::"r"(mb), "r"(parity) : "memory");
    __syncwarp();  // lanes leave the spin at different times; the DMMAs (.aligned) need the whole warp
}
__device__ __forceinline__ void mt_load(unsigned dst, const CUtensorMap *tm, int c0, int c1, int c2, unsigned mb) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
        "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(mb)
        : "memory");
}

extern __shared__ __align__(128) double mt_smem[];

template <bool KX>
__global__ void __launch_bounds__(MT_THREADS) modal_fwd_tma(const ModalGemmArgs g, const __grid_constant__ CUtensorMap tA0,
                                                            const __grid_constant__ CUtensorMap tA1,
                                                            const __grid_constant__ CUtensorMap tT) {
    constexpr int AP = 68, ASZ = 16 * AP, STAGE = ASZ + 2 * MT_TSZ;
    const int q = blockIdx.z & 1, b = blockIdx.z >> 1;
    const int M = q ? g.no : g.ne, K = q ? g.hh : g.H;
    const int mt = blockIdx.x, m0 = 64 * mt, l0 = blockIdx.y * 64;
    if (mt >= M / 64) return;
    // the last full tile's CTA also computes the tail rows [64 (M / 64), M) (<= 4: the A box's 4
    // extra rows hold them) on CUDA cores from the same staged operand tiles
    const int TR = M - 64 * (M / 64);
    const bool tail = g.fuse_tail && mt == M / 64 - 1 && TR > 0;
    double tacc[2] = {0.0, 0.0};  // tail rows tr, tr + 2 of line tn
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int sh = (int)(((128 - (__cvta_generic_to_shared(mt_smem) & 127)) & 127) / sizeof(double));
    double *sm = mt_smem + sh;
    const unsigned s0 = (unsigned)__cvta_generic_to_shared(sm), mb0 = s0 + 8u * MT_S * STAGE;
    const int nk = (K + 15) / 16;
    constexpr unsigned BYTES = 8u * (ASZ + 2 * (KX ? 64 * 20 : 16 * 68));
    auto issue = [&](int kt) {  // thread 0
        if (kt >= nk) return;
        // the mirrored block starts at n - k0 - 16; along x (the box's contiguous dimension) the
        // start must be 16-byte aligned, so an odd start is moved down by one (read with offset mo)
        const int slot = kt % MT_S, k0 = 16 * kt, km = g.n - k0 - 16 - (KX ? (g.n & 1) : 0);
        const unsigned mb = mb0 + 8u * slot, d = s0 + 8u * slot * STAGE;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(BYTES) : "memory");
        // (the map operand is the kernel parameter itself: a runtime-selected pointer to one of two
        // __grid_constant__ maps could be materialised in local memory, which TMA cannot read)
        if (q) mt_load(d, &tA1, m0, k0, 0, mb);
        else mt_load(d, &tA0, m0, k0, 0, mb);
        if (KX) {
            mt_load(d + 8u * ASZ, &tT, k0, l0, 0, mb);
            mt_load(d + 8u * (ASZ + MT_TSZ), &tT, km, l0, 0, mb);
        } else {
            mt_load(d + 8u * ASZ, &tT, l0, k0, b, mb);
            mt_load(d + 8u * (ASZ + MT_TSZ), &tT, l0, km, b, mb);
        }
    };
    if (tid == 0) {
        for (int i = 0; i < MT_S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb0 + 8u * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int i = 0; i < MT_S; ++i) issue(i);
    }
    __syncthreads();
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int wm = (w >> 1) * 32, wn = (w & 1) * 32;
    const double sg = q ? -1.0 : 1.0;
    const int mo = KX ? (g.n & 1) : 0;
    for (int kt = 0; kt < nk; ++kt) {
        const int slot = kt % MT_S;
        mt_wait(mb0 + 8u * slot, (unsigned)((kt / MT_S) & 1));
        const double *As = sm + slot * STAGE, *Ts = As + ASZ, *Tm = Ts + MT_TSZ;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int kk = 4 * s + (lane & 3);
            double a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk * AP + wm + 8 * i + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int nn = wn + 8 * j + (lane >> 2);
                bb[j] = KX ? fma(sg, Tm[nn * 20 + 15 - kk + mo], Ts[nn * 20 + kk])
                           : fma(sg, Tm[(15 - kk) * 68 + nn], Ts[kk * 68 + nn]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], bb[j]);
        }
        if (tail) {
            const int tn = tid & 63, tr = tid >> 6;
#pragma unroll 4
            for (int kk = 0; kk < 16; ++kk) {
                const double t = KX ? fma(sg, Tm[tn * 20 + 15 - kk + mo], Ts[tn * 20 + kk])
                                    : fma(sg, Tm[(15 - kk) * 68 + tn], Ts[kk * 68 + tn]);
                if (tr < TR) tacc[0] = fma(As[kk * AP + 64 + tr], t, tacc[0]);
                if (tr + 2 < TR) tacc[1] = fma(As[kk * AP + 64 + tr + 2], t, tacc[1]);
            }
        }
        __syncthreads();  // every warp is done with this slot
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(kt + MT_S);
        }
    }
    const int slot0 = q ? g.ne : 0;
    const long boff = (long)b * g.bs;
    if (tail) {
        const int tn = tid & 63, tr = tid >> 6, l = l0 + tn;
        if (l < g.nl)
#pragma unroll
            for (int u = 0; u < 2; ++u)
                if (tr + 2 * u < TR) g.out[(long)(slot0 + 64 * (M / 64) + tr + 2 * u) * g.ks + boff + (long)l * g.ls] = tacc[u];
    }
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
    // the unused slots [ne + no, n) of these lines are zero (one CTA per line tile writes them)
    if (q == 1 && mt == 0)
        for (int e = tid; e < 64 * (g.n - g.ne - g.no); e += MT_THREADS) {
            const int l = l0 + e % 64, sl = g.ne + g.no + e / 64;
            if (l < g.nl) g.out[(long)sl * g.ks + (long)l * g.ls + boff] = 0.0;
        }
}

template <bool KX>
__global__ void __launch_bounds__(MT_THREADS) modal_inv_tma(const ModalGemmArgs g, const __grid_constant__ CUtensorMap tA0,
                                                            const __grid_constant__ CUtensorMap tA1,
                                                            const __grid_constant__ CUtensorMap tT) {
    constexpr int AP = 36, ASZ = 16 * AP, STAGE = ASZ + MT_TSZ, S = 4;
    const int b = blockIdx.z, mt = blockIdx.x, i0 = 32 * mt, l0 = blockIdx.y * 64;
    const int H = g.H, hh = g.hh, n = g.n;
    if (mt >= H / 32) return;
    // the last full tile's CTA also computes the tail rows [32 (H / 32), H) (<= 4: the A box's 4
    // extra rows hold them; rows >= hh of P_o are zero padding)
    const int TR = H - 32 * (H / 32);
    const bool tail = g.fuse_tail && mt == H / 32 - 1 && TR > 0;
    double tte[2] = {0.0, 0.0}, tto[2] = {0.0, 0.0};  // tail rows tr, tr + 2 of line tn
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int sh = (int)(((128 - (__cvta_generic_to_shared(mt_smem) & 127)) & 127) / sizeof(double));
    double *sm = mt_smem + sh;
    const unsigned s0 = (unsigned)__cvta_generic_to_shared(sm), mb0 = s0 + 8u * S * STAGE;
    const int nke = (g.ne + 15) / 16, nk = nke + (g.no + 15) / 16;
    constexpr unsigned BYTES = 8u * (ASZ + (KX ? 64 * 20 : 16 * 68));
    auto issue = [&](int kt) {  // thread 0
        if (kt >= nk) return;
        const int slot = kt % S, q = kt < nke ? 0 : 1, k0 = 16 * (kt < nke ? kt : kt - nke);
        // operand rows: the half's modal slots; along x an odd start moves down by one (16-byte
        // aligned box rows), read back with the offset ko below
        const int kc0 = (q ? g.ne : 0) + k0, kc = KX ? kc0 - (kc0 & 1) : kc0;
        const unsigned mb = mb0 + 8u * slot, d = s0 + 8u * slot * STAGE;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(BYTES) : "memory");
        if (q) mt_load(d, &tA1, i0, k0, 0, mb);
        else mt_load(d, &tA0, i0, k0, 0, mb);
        if (KX) mt_load(d + 8u * ASZ, &tT, kc, l0, 0, mb);
        else mt_load(d + 8u * ASZ, &tT, l0, kc, b, mb);
    };
    if (tid == 0) {
        for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb0 + 8u * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int i = 0; i < S; ++i) issue(i);
    }
    __syncthreads();
    double acc[2][4][2][2];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[h2][i][j][0] = acc[h2][i][j][1] = 0.0;
    const int wn = 16 * w;
    auto body = [&](double (&ac)[4][2][2], const double *As, const double *Ts, int ko) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int kk = 4 * s + (lane & 3);
            double a[4], bb[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk * AP + 8 * i + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int nn = wn + 8 * j + (lane >> 2);
                bb[j] = KX ? Ts[nn * 20 + kk + ko] : Ts[kk * 68 + nn];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma(ac[i][j], a[i], bb[j]);
        }
    };
    for (int kt = 0; kt < nk; ++kt) {
        const int slot = kt % S;
        mt_wait(mb0 + 8u * slot, (unsigned)((kt / S) & 1));
        const double *As = sm + slot * STAGE, *Ts = As + ASZ;
        if (kt < nke) body(acc[0], As, Ts, 0);
        else body(acc[1], As, Ts, KX ? (g.ne & 1) : 0);
        if (tail) {
            const int tn = tid & 63, tr = tid >> 6, ko = kt < nke ? 0 : (KX ? (g.ne & 1) : 0);
            double(&ta)[2] = kt < nke ? tte : tto;
#pragma unroll 4
            for (int kk = 0; kk < 16; ++kk) {
                const double c = KX ? Ts[tn * 20 + kk + ko] : Ts[kk * 68 + tn];
                if (tr < TR) ta[0] = fma(As[kk * AP + 32 + tr], c, ta[0]);
                if (tr + 2 < TR) ta[1] = fma(As[kk * AP + 32 + tr + 2], c, ta[1]);
            }
        }
        __syncthreads();
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(kt + S);
        }
    }
    const long boff = (long)b * g.bs;
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
    if (tail) {
        const int tn = tid & 63, tr = tid >> 6, l = l0 + tn;
        if (l < g.nl) {
            const long lo = (long)l * g.ls + boff;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int r = 32 * (H / 32) + tr + 2 * u;
                if (tr + 2 * u >= TR) continue;
                if (r < hh) {
                    g.out[(long)r * g.ks + lo] = tte[u] + tto[u];
                    g.out[(long)(n - 1 - r) * g.ks + lo] = tte[u] - tto[u];
                } else {
                    g.out[(long)r * g.ks + lo] = tte[u];
                }
            }
        }
    }
}

}  // namespace

int launch_modal_gemm(const ModalGemmArgs &g, cudaStream_t s) {
    if (g.nl <= 0 || g.nb <= 0) return 0;
    const unsigned ny = (unsigned)((g.nl + MG_BN - 1) / MG_BN);
    if (ny > 65535u || g.nb > 32767) return -1;
    const bool kx = g.kdim == 0;
    // full tiles on the TMA-fed tensor-core kernels (when the maps are available), the rest on
    // the register-staged kernels (tail rows, or everything)
    const bool tma = g.Qe2 && g.td[0] > 0;
    // the tail rows ride in the TMA kernels' last full-tile CTAs when there are at most 4 of them
    // (ADS_MODAL_FUSE_TAIL=0: the separate CUDA-core tail kernel, experiment switch)
    static const bool fuse_ok = [] {
        const char *e = std::getenv("ADS_MODAL_FUSE_TAIL");
        return !(e && e[0] == '0');
    }();
    auto fits = [](int M, int T) { return M >= T && M % T <= 4; };
    const bool fuse = tma && fuse_ok &&
                      (g.inverse ? fits(g.H, 32) : (fits(g.ne, 64) && (g.no == 0 || fits(g.no, 64))));
    ModalGemmArgs gf = g;
    gf.fuse_tail = fuse ? 1 : 0;
    if (tma) {
        CUtensorMap tA0, tA1, tT;
        const unsigned tb0 = kx ? 20 : 68, tb1 = kx ? 64 : 16;
        if (encode_map_3d(&tT, g.in, g.td[0], g.td[1], g.td[2], g.ts1, g.ts2, tb0, tb1, 1)) return -2;
        if (!g.inverse) {
            const int mt = std::max(g.ne, g.no) / 64;
            if (mt > 0) {
                if (encode_map_3d(&tA0, g.Qe2, g.lqe, g.H, 1, g.lqe, (long)g.lqe * g.H, 68, 16, 1) ||
                    encode_map_3d(&tA1, g.Qo2, g.lqo, std::max(g.hh, 1), 1, g.lqo, (long)g.lqo * std::max(g.hh, 1), 68,
                                  16, 1))
                    return -2;
                const size_t sm = sizeof(double) * (MT_S * (16 * 68 + 2 * MT_TSZ) + 16 + 16);
                auto fn = kx ? modal_fwd_tma<true> : modal_fwd_tma<false>;
                cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                dim3 grd(mt, ny, 2 * g.nb);
                fn<<<grd, MT_THREADS, sm, s>>>(gf, tA0, tA1, tT);
            }
        } else if (g.H / 32 > 0) {
            if (encode_map_3d(&tA0, g.Pe2, g.lpe, std::max(g.ne, 1), 1, g.lpe, (long)g.lpe * std::max(g.ne, 1), 36, 16,
                              1) ||
                encode_map_3d(&tA1, g.Po2, g.lpo, std::max(g.no, 1), 1, g.lpo, (long)g.lpo * std::max(g.no, 1), 36, 16,
                              1))
                return -2;
            const size_t sm = sizeof(double) * (4 * (16 * 36 + MT_TSZ) + 16 + 16);
            auto fn = kx ? modal_inv_tma<true> : modal_inv_tma<false>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            dim3 grd(g.H / 32, ny, g.nb);
            fn<<<grd, MT_THREADS, sm, s>>>(gf, tA0, tA1, tT);
        }
    }
    if (fuse) return 0;
    ModalGemmArgs t = g;
    t.tail_only = tma ? 1 : 0;
    if (!g.inverse) {
        const int mt = tma ? 1 : std::max(g.ne, g.no) / 64 + 1;
        dim3 grd(mt, ny, 2 * g.nb);
        if (kx) modal_fwd_kernel<true><<<grd, MG_THREADS, 0, s>>>(t);
        else modal_fwd_kernel<false><<<grd, MG_THREADS, 0, s>>>(t);
    } else {
        dim3 grd(tma ? 1 : g.H / 32 + 1, ny, g.nb);
        if (kx) modal_inv_kernel<true><<<grd, MG_THREADS, 0, s>>>(t);
        else modal_inv_kernel<false><<<grd, MG_THREADS, 0, s>>>(t);
    }
    return 0;
}

}  // namespace ads
