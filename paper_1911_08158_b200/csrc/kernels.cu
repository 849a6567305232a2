// kernels.cu -- sm_100a fp64 kernels of the ADS wave step (arXiv:1911.08158).
//
//   kop4_kernel  : drift P = U + tau V, source, and the sum-factorised
//                  Kronecker operator K P (Eq. 14, 3D) in ONE
//                  pass, every stiffness factor on P itself (K first; Kz in
//                  plane-difference form): a 32x16 (x,y) tile marches along z;
//                  per plane the x- and y-passes run from shared memory and the
//                  z-pass from a register ring of 2p+1 planes.  HBM: reads U, V;
//                  writes P, r.
//   sweep_kernel : batched banded LU solves A_d^-1 along x, y or z
//                  (PAPER.md:533-618).  Each line is split into C chunks; every
//                  chunk runs the p-term recurrences twice (zero incoming state
//                  -> boundary state; exact incoming state -> result), the chunk
//                  boundary states are coupled by an exact Kogge-Stone scan of
//                  the affine chunk maps in shared memory (partitioned / SPIKE-
//                  style elimination).  Lines are kept in registers: one HBM read
//                  and one write per element.  x-lines are staged through shared
//                  memory (coalesced); y/z lines are loaded coalesced across 8
//                  adjacent x-lines.  The z sweep fuses the kick V += tau a.
#include <cstdlib>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "kernels.cuh"

namespace ads {

// Programmatic dependent launch (sm_90+): the step's kernels are launched with programmatic stream
// serialisation (launch_pdl), let their successor launch as soon as they start, and wait for their
// predecessor's completion (and memory flush) before touching any field the step reads or writes;
// only constant tables are staged before the wait, so the successor's launch and prologue overlap
// the predecessor's tail.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Per-device launch facts of a kernel at a dynamic shared-memory size, cached and thread-safe:
// the SM count, the resident CTAs per SM, and the >48 KB opt-in (raised to the largest size the
// kernel has been launched with on that device).
struct LaunchFacts {
    int nsm = 1, per_sm = 1;
};
static LaunchFacts launch_facts(const void *fn, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, size_t>, LaunchFacts> cache;
    static std::map<std::pair<int, const void *>, size_t> optin;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, fn, smem);
    const auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    size_t &cur = optin[{dev, fn}];
    if (smem > cur) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cur = smem;
    }
    LaunchFacts f;
    cudaDeviceGetAttribute(&f.nsm, cudaDevAttrMultiProcessorCount, dev);
    int ps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, fn, threads, smem);
    f.per_sm = std::max(ps, 1);
    cache[key] = f;
    return f;
}

// ------------------------------------------------------------------------------------------
// partitioned banded sweeps (v3)
//
// Solves A_d x = r along every line of direction d: for each
// line, forward y_i = r_i - sum_k l_{i,k} y_{i-k}, then backward
// x_i = y_i dinv_i - sum_k us_{i,k} x_{i+k}, with the LU factors of the
// constant A_d computed once on the host.
//
// CTA = 8 warps on a tile of SW_LW = 8 adjacent lines.  Thread (lane, warp):
//   q = lane & 7          line of the tile
//   c = 4 warp + lane/8   chunk: rows [c L, c L + L) of the (identity-padded) line
// so the 32 chunks of a line are spread over the CTA and each thread keeps its
// L values in registers.  Per tile:
//   1. forward recurrence from a zero incoming state -> y0 (kept), tail h_c
//   2. h_c -> shared memory; barrier; incoming state of chunk c:
//      in_c = sum_{c'<c} Tf_{c-1} ... Tf_{c'+1} h_{c'}, folded over the last Kf
//      chunks (the host certifies older chunks contribute < 2^-64 of the state,
//      host_setup.h); then y = y0 + (response to in_c)
//   3. the same backward (head states, Rb maps, Kb chunks)
// = exact partitioned (SPIKE-style) elimination of the banded system.
// Uniform chunks (inside the frozen Toeplitz interior, all bitwise identical)
// take every coefficient -- LU rows, the chunk responses G and the transfer
// maps -- from the kernel's constant bank; the response to in_c is then a
// dependency-free G-multiply instead of a recurrence.  Edge chunks read their
// rows from a shared-memory table.
// y/z lines: each row access is 8 consecutive doubles of adjacent lines; the
// next tile streams HBM -> shared memory (cp.async) while the current one is
// solved.  x lines (contiguous): coalesced cooperative copies through shared
// memory; tile pitch np = 2 (mod 16) keeps the per-thread chunk reads
// conflict-free.  The z sweep fuses the kick V += tau a into its store.
// ------------------------------------------------------------------------------------------
// LW lines per tile (x: 8, y/z: 16); 32/LW chunks per warp; C (chunks per line) x LW threads
template <int LW, int C = kSweepChunks>
struct SW {
    static constexpr int G = 32 / LW, WARPS = C / G, THREADS = 32 * WARPS;
    static_assert(WARPS * G == C, "one chunk per (warp, lane group)");
};

__host__ __device__ constexpr int ring(int i, int P) { return ((i % P) + P) % P; }
template <int P> struct Rec {
    static constexpr int FW = (P + 1) & ~1;  // forward record: l_1..l_P (even length)
    static constexpr int BW = (P + 2) & ~1;  // backward record: dinv, us_1..us_P
};

// Coefficient sources.  UNI: constant bank.  EDGE: shared-memory records, row j of
// the chunk at rec + j * FW (bwd: + j * BW) -- compile-time offsets.
template <int P, bool UNI>
struct Coef {
    const double *f, *b;  // EDGE: records of the chunk's first row
    const SolveTab &t;
    __device__ __forceinline__ double l(int j, int k) const { return UNI ? t.lc[k - 1] : f[j * Rec<P>::FW + k - 1]; }
    __device__ __forceinline__ double d(int j) const { return UNI ? t.dic : b[j * Rec<P>::BW]; }
    __device__ __forceinline__ double u(int j, int k) const { return UNI ? t.usc[k - 1] : b[j * Rec<P>::BW + k]; }
};

// forward recurrence; ZERO: incoming 0, v <- y0, h <- tail (y_{L-1-m});
// !ZERO: homogeneous response to incoming y_{-1-m} = h[m], added to v
template <int P, int L, bool UNI, bool ZERO>
__device__ __forceinline__ void fwd_pass(double (&v)[L], double (&h)[P], const Coef<P, UNI> &cf) {
    double R[P];
#pragma unroll
    for (int m = 0; m < P; ++m) R[ring(-1 - m, P)] = ZERO ? 0.0 : h[m];
#pragma unroll
    for (int j = 0; j < L; ++j) {
        double acc = ZERO ? v[j] : 0.0;
#pragma unroll
        for (int k = P; k >= 1; --k)
            if (!ZERO || j - k >= 0) acc = fma(-cf.l(j, k), R[ring(j - k, P)], acc);
        R[ring(j, P)] = acc;
        if (ZERO) v[j] = acc;
        else v[j] += acc;
    }
    if (ZERO) {
#pragma unroll
        for (int m = 0; m < P; ++m) h[m] = R[ring(L - 1 - m, P)];
    }
}

// backward recurrence; ZERO: incoming 0, v <- x0, h <- head (x_m);
// !ZERO: homogeneous response to incoming x_{L+m} = h[m], added to v
template <int P, int L, bool UNI, bool ZERO>
__device__ __forceinline__ void bwd_pass(double (&v)[L], double (&h)[P], const Coef<P, UNI> &cf) {
    double R[P];
#pragma unroll
    for (int m = 0; m < P; ++m) R[ring(L + m, P)] = ZERO ? 0.0 : h[m];
#pragma unroll
    for (int q = 0; q < L; ++q) {
        const int j = L - 1 - q;
        double acc = ZERO ? v[j] * cf.d(j) : 0.0;
#pragma unroll
        for (int k = P; k >= 1; --k)
            if (!ZERO || j + k < L) acc = fma(-cf.u(j, k), R[ring(j + k, P)], acc);
        R[ring(j, P)] = acc;
        if (ZERO) v[j] = acc;
        else v[j] += acc;
    }
    if (ZERO) {
#pragma unroll
        for (int m = 0; m < P; ++m) h[m] = R[m];
    }
}

// incoming state of chunk c: Horner over chunks c-K .. c-1 (FWD) or c+K .. c+1
// (backward).  UNIW: every chunk of the window is uniform -> maps from the
// constant bank (Tf(a,b) = Gf[L-1-a][b], Rb(a,b) = Gb[a][b]).
template <int P, int L, int LW, bool FWD, bool UNIW>
__device__ __forceinline__ void chunk_walk(double (&in)[P], const SolveTab &t, const double *shT, const double *shh,
                                           int c, int K, int q) {
#pragma unroll
    for (int m = 0; m < P; ++m) in[m] = 0.0;
    const int c0 = FWD ? max(c - K, 0) : min(c + K, t.C - 1);
    for (int cc = c0; FWD ? cc < c : cc > c; cc += FWD ? 1 : -1) {
        double nin[P];
#pragma unroll
        for (int a = 0; a < P; ++a) {
            double acc = shh[(cc * P + a) * LW + q];
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double T = UNIW ? (FWD ? t.Gf[L - 1 - a][b] : t.Gb[a][b]) : shT[(cc * P + a) * P + b];
                acc = fma(T, in[b], acc);
            }
            nin[a] = acc;
        }
#pragma unroll
        for (int a = 0; a < P; ++a) in[a] = nin[a];
    }
}

struct SweepSmem {
    const double *shTf, *shRb, *ef, *eb;
    double *shf, *shb;
};

// The whole per-tile solve of one thread's chunk.  after_sync runs right after the
// first barrier (every thread has consumed its tile input by then).
template <int P, int L, int LW, bool UNI, class AfterSync>
__device__ __forceinline__ void solve_chunk(double (&v)[L], const SolveTab &t, const SweepSmem &sm, int c, int q,
                                            bool walk_uf, bool walk_ub, const double *recf, const double *recb,
                                            AfterSync after_sync) {
    const Coef<P, UNI> cf{recf, recb, t};
    double h[P], in[P];
    fwd_pass<P, L, UNI, true>(v, h, cf);
#pragma unroll
    for (int m = 0; m < P; ++m) sm.shf[(c * P + m) * LW + q] = h[m];
    __syncthreads();
    after_sync();
    if (walk_uf) chunk_walk<P, L, LW, true, true>(in, t, sm.shTf, sm.shf, c, t.Kf, q);
    else chunk_walk<P, L, LW, true, false>(in, t, sm.shTf, sm.shf, c, t.Kf, q);
    if (UNI) {
#pragma unroll
        for (int j = 0; j < L; ++j)
#pragma unroll
            for (int m = 0; m < P; ++m) v[j] = fma(t.Gf[j][m], in[m], v[j]);
    } else {
        fwd_pass<P, L, UNI, false>(v, in, cf);
    }
    bwd_pass<P, L, UNI, true>(v, h, cf);
#pragma unroll
    for (int m = 0; m < P; ++m) sm.shb[(c * P + m) * LW + q] = h[m];
    __syncthreads();
    if (walk_ub) chunk_walk<P, L, LW, false, true>(in, t, sm.shRb, sm.shb, c, t.Kb, q);
    else chunk_walk<P, L, LW, false, false>(in, t, sm.shRb, sm.shb, c, t.Kb, q);
    if (UNI) {
#pragma unroll
        for (int j = 0; j < L; ++j)
#pragma unroll
            for (int m = 0; m < P; ++m) v[j] = fma(t.Gb[j][m], in[m], v[j]);
    } else {
        bwd_pass<P, L, UNI, false>(v, in, cf);
    }
}

// Ampere-style asynchronous global -> shared copies (LDGSTS): the next tile streams in
// while the current one is solved, without holding registers.
__device__ __forceinline__ void cp_async8(double *sdst, const double *gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(double *sdst, const double *gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
// shared address + zero fill: copies nbytes (0 or 8) and fills the rest of the 8 bytes with 0
__device__ __forceinline__ void cp_async8_zfill(unsigned sdst, const double *gsrc, unsigned nbytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sdst), "l"(gsrc), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// x tiles: nbox TMA boxes of rb columns, rb = 2 (mod 16) and <= 256, nbox rb >= n
__host__ __device__ inline int xbox_count(int n) { return (n + 241) / 242; }
__host__ __device__ inline int xbox_cols(int n) {
    const int c = (n + xbox_count(n) - 1) / xbox_count(n);
    return c + ((2 - c) % 16 + 16) % 16;
}

// edge rows: [0, c_lo L) and [c_hi L, C L), plus one block of L uniform rows
__host__ __device__ inline int sweep_edge_rows(const SolveTab &t) {
    return t.c_lo * t.L + (t.C - t.c_hi) * t.L + t.L;
}
template <int P, int LW>
__host__ __device__ inline long sweep_smem_doubles(const SolveTab &t, bool xdir, long sy, bool kick, int vbufs = 1) {
    const long fixed = 2L * t.C * P * P + 2L * t.C * P * LW +
                       (long)sweep_edge_rows(t) * (Rec<P>::FW + Rec<P>::BW);
    if (xdir) {
        const int nb = xbox_count(t.n), rb = xbox_cols(t.n);
        return fixed + 2L * ((nb * LW * rb + 15) & ~15) + 16 + 4;
    }
    (void)kick;
    return fixed + (1L + vbufs) * t.C * t.L * LW + 16 + 4;
}

// dynamic shared memory of a sweep launch (the tile width and buffers sweep_launch picks, one
// output buffer): lets the host reject chunkings whose tables do not fit before a launch fails
long sweep_smem_bytes(int p, const SolveTab &t, int dir) {
    const bool X = dir == 0;
    const bool narrow = X || t.L > 17 || t.C > 32;
    long d = 0;
#define ADS_SSB(PP)                                                                                   \
    case PP:                                                                                         \
        d = narrow ? sweep_smem_doubles<PP, 8>(t, X, 0, false, 1) : sweep_smem_doubles<PP, 16>(t, X, 0, false, 1); \
        break;
    switch (p) { ADS_SSB(1) ADS_SSB(2) ADS_SSB(3) ADS_SSB(4) ADS_SSB(5) default: return -1; }
#undef ADS_SSB
    return d * (long)sizeof(double);
}

template <int P, int L, bool XDIR, int LW, int C>
__global__ void __launch_bounds__(SW<LW, C>::THREADS, 512 / SW<LW, C>::THREADS)
    sweep_kernel(const __grid_constant__ SweepArgs a) {
    constexpr int SW_LW = LW, SW_G = SW<LW, C>::G, SW_THREADS = SW<LW, C>::THREADS;
    extern __shared__ __align__(16) double smem[];
    constexpr int FW = Rec<P>::FW, BW = Rec<P>::BW;
    pdl_launch_dependents();
    const SolveTab &t = a.t;
    const int nedge = sweep_edge_rows(t);
    double *shTf = smem, *shRb = shTf + C * P * P;
    double *shf = shRb + C * P * P, *shb = shf + C * P * SW_LW;
    double *ef = shb + C * P * SW_LW, *eb = ef + nedge * FW;
    double *buf = eb + nedge * BW;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int q = lane & (SW_LW - 1), c = w * SW_G + lane / SW_LW, s = c * L;
    const int n = t.n;
    const int ulo = t.c_lo * L, uhi = t.c_hi * L;  // uniform rows [ulo, uhi)
    for (int e = tid; e < C * P * P; e += SW_THREADS) {
        shTf[e] = __ldg(t.Tf + e);
        shRb[e] = __ldg(t.Rb + e);
    }
    for (int e = tid; e < nedge; e += SW_THREADS) {
        // edge table row e -> matrix row r; the last L rows hold the uniform row
        const bool un = e >= nedge - L;
        const int r = e < ulo ? e : e - ulo + uhi;
#pragma unroll
        for (int k = 0; k < FW; ++k) ef[e * FW + k] = k < P ? (un ? t.lc[k] : __ldg(t.l + (long)r * P + k)) : 0.0;
        eb[e * BW] = un ? t.dic : __ldg(t.dinv + r);
#pragma unroll
        for (int k = 1; k < BW; ++k) eb[e * BW + k] = k <= P ? (un ? t.usc[k - 1] : __ldg(t.us + (long)r * P + k - 1)) : 0.0;
    }
    const bool cu = s >= ulo && s + L <= uhi;                           // my chunk uniform
    const bool uni = w * SW_G * L >= ulo && (w + 1) * SW_G * L <= uhi;  // whole warp uniform
    const int erow = cu ? nedge - L : (s < ulo ? s : s - uhi + ulo);
    const double *recf = ef + erow * FW, *recb = eb + erow * BW;
    // walk windows entirely uniform (warp-wide): forward chunks [4w - Kf, 4w + 2], backward [4w + 1, 4w + 3 + Kb]
    const bool walk_uf = uni && w * SW_G - t.Kf >= t.c_lo;
    const bool walk_ub = uni && (w + 1) * SW_G - 1 + t.Kb < t.c_hi;
    const SweepSmem sm{shTf, shRb, ef, eb, shf, shb};
    const Geom &g = a.geo;
    pdl_wait();  // fields (and the step counter) from here on
    auto solve = [&](double (&v)[L], auto after) {
        if (uni) solve_chunk<P, L, LW, true>(v, t, sm, c, q, walk_uf, walk_ub, recf, recb, after);
        else solve_chunk<P, L, LW, false>(v, t, sm, c, q, false, false, recf, recb, after);
    };

    if (XDIR) {
        // x lines: the field viewed as a 2D tensor (n0 columns x n1 n2 lines, pitch sy).  A tile
        // of SW_LW consecutive lines moves HBM -> shared memory as a.nbox TMA boxes of a.rb
        // columns (region b holds columns [b rb, (b+1) rb) as [line][rb]; rb = 2 mod 16 keeps the
        // per-thread chunk reads conflict-free), results go back with TMA stores from a second
        // buffer (out-of-bounds columns and lines are neither read nor written).
        const int XB = a.rb, NB = a.nbox, RS = SW_LW * XB;  // region size (doubles)
        double *xin = buf + ((128 - (reinterpret_cast<uintptr_t>(buf) & 127)) & 127) / sizeof(double);
        double *xout = xin + ((NB * RS + 15) & ~15);
        unsigned long long *mbar = reinterpret_cast<unsigned long long *>(xout + ((NB * RS + 15) & ~15));
        const unsigned mb = (unsigned)__cvta_generic_to_shared(mbar);
        const long nlines = (long)g.n1 * g.n2;
        const long ntiles = (nlines + SW_LW - 1) / SW_LW;
        // my chunk [s, s + L): region b0 up to column (b0 + 1) XB, then region b0 + 1
        const int b0 = s / XB, jb = min(L, (b0 + 1) * XB - s);
        const int o0 = b0 * RS + q * XB + (s - b0 * XB), o1 = (b0 + 1) * RS + q * XB - jb;
        auto tload = [&](long tile) {  // thread 0
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                         "r"((unsigned)(NB * RS * sizeof(double)))
                         : "memory");
            for (int bb = 0; bb < NB; ++bb) {
                const unsigned d = (unsigned)__cvta_generic_to_shared(xin + bb * RS);
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, 0}], [%4];\n" ::"r"(d),
                    "l"(reinterpret_cast<unsigned long long>(&a.tm_in)), "r"(bb * XB), "r"((int)(tile * SW_LW)),
                    "r"(mb)
                    : "memory");
            }
        };
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0 && (long)blockIdx.x < ntiles) tload(blockIdx.x);
        unsigned ph = 0;
        for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ph ^= 1u) {
            asm volatile(
                "{\n .reg .pred P1;\n WAITX_%=:\n"
                " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                " @!P1 bra WAITX_%=;\n}\n" ::"r"(mb), "r"(ph) : "memory");
            double v[L];
#pragma unroll
            for (int j = 0; j < L; ++j) v[j] = (s + j < n) ? xin[j < jb ? o0 + j : o1 + j] : 0.0;
            solve(v, [&] {
                if (tid == 0 && tile + gridDim.x < ntiles) {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    tload(tile + gridDim.x);
                }
            });
            if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // xout free
            __syncthreads();
#pragma unroll
            for (int j = 0; j < L; ++j)
                if (s + j < n) xout[j < jb ? o0 + j : o1 + j] = v[j];
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                for (int bb = 0; bb < NB; ++bb) {
                    const unsigned d = (unsigned)__cvta_generic_to_shared(xout + bb * RS);
                    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, 0}], [%3];\n" ::"l"(
                                     reinterpret_cast<unsigned long long>(&a.tm_out)),
                                 "r"(bb * XB), "r"((int)(tile * SW_LW)), "r"(d)
                                 : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            }
        }
        if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    } else {
        // y: lines (i, k), element stride sy; z: lines (i, j), element stride sz.
        // Tile = SW_LW adjacent i.  One thread moves the whole tile with TMA: `nbox` 3D boxes
        // (16 lines x rb rows) into the [row][q] buffer, rows beyond the line and lines beyond
        // n0 zero-filled by the TMA unit (out-of-bounds fill); mbarrier completion.  The next
        // tile's load is issued after the first in-solve barrier (everyone has read the buffer);
        // the kick's V tile is loaded at the tile start and consumed after the solve.
        const int nb = a.dir == 1 ? g.n2 : g.n1;
        const int nib = (g.n0 + SW_LW - 1) / SW_LW;
        const long ntiles = (long)nib * nb;
        const bool kick = a.mode == 1;
        const long sl = a.dir == 1 ? g.sy : g.sz;
        const long sb = a.dir == 1 ? g.sz : g.sy;
        const int nv = max(0, min(L, n - s));  // rows of my chunk inside the line
        // buffers (128-byte aligned) and two mbarriers after them
        double *ibase = buf + ((128 - (reinterpret_cast<uintptr_t>(buf) & 127)) & 127) / sizeof(double);
        double *vbase0 = ibase + C * L * SW_LW;  // a.vbufs tile buffers of C L SW_LW doubles
        unsigned long long *mbar = reinterpret_cast<unsigned long long *>(vbase0 + a.vbufs * C * L * SW_LW);
        const unsigned mb_in = (unsigned)__cvta_generic_to_shared(mbar), mb_v = mb_in + 8;
        const unsigned bytes = (unsigned)(C * L * SW_LW * sizeof(double));
        double *ib = ibase + s * SW_LW + q;
        auto tma = [&](const CUtensorMap *tm, double *dst, unsigned mb, long tile) {
            // thread 0 only
            const int i0 = (int)(tile % nib) * SW_LW, lb = (int)(tile / nib);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(bytes) : "memory");
            for (int b = 0; b < a.nbox; ++b) {
                const unsigned d = (unsigned)__cvta_generic_to_shared(dst + (long)b * a.rb * SW_LW);
                const int r0 = b * a.rb;
                const int c1 = a.dir == 1 ? r0 : lb, c2 = a.dir == 1 ? lb : r0;
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d),
                    "l"(reinterpret_cast<unsigned long long>(tm)), "r"(i0), "r"(c1), "r"(c2), "r"(mb)
                    : "memory");
            }
        };
        auto wait = [&](unsigned mb, unsigned parity) {
            asm volatile(
                "{\n .reg .pred P1;\n WAIT_%=:\n"
                " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                " @!P1 bra WAIT_%=;\n}\n" ::"r"(mb), "r"(parity) : "memory");
        };
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb_in) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb_v) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0 && (long)blockIdx.x < ntiles) tma(&a.tm_in, ibase, mb_in, blockIdx.x);
        if (a.dstep_inc && tid == 0 && blockIdx.x == 0) *a.dstep_inc += 1;  // read by the next step's kop
        // wait until at most vbufs - 1 TMA stores are still reading their buffer (thread 0)
        auto wait_store_read = [&] {
            if (a.vbufs > 1) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        };
        unsigned ph = 0;
        for (long tile = blockIdx.x, it = 0; tile < ntiles; tile += gridDim.x, ph ^= 1u, ++it) {
            double *vbase = vbase0 + (a.vbufs > 1 ? (it & 1) : 0) * (C * L * SW_LW);
            double *vb = vbase + s * SW_LW + q;
            const int i = (int)(tile % nib) * SW_LW + q;
            const long base = (tile / nib) * sb + i + (long)s * sl;
            const int nvl = i < g.n0 ? nv : 0;
            if (kick && tid == 0) {
                // vbuf: the TMA store of V that last used it must have read it before it is reloaded
                wait_store_read();
                tma(&a.tm_v, vbase, mb_v, tile);
            }
            wait(mb_in, ph);
            double v[L];
#pragma unroll
            for (int j = 0; j < L; ++j) v[j] = ib[j * SW_LW];
            solve(v, [&] {
                if (tid == 0 && tile + gridDim.x < ntiles) {
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    tma(&a.tm_in, ibase, mb_in, tile + gridDim.x);
                }
            });
            // results leave through vbuf with TMA stores (rows >= n and lines >= n0 clipped):
            // no kick: out = x;  kick: V += kick x in place (a is written directly when requested)
            if (!kick) {
                if (tid == 0) wait_store_read();
                __syncthreads();  // the store that last used this vbuf has read it
#pragma unroll
                for (int j = 0; j < L; ++j) vb[j * SW_LW] = v[j];
            } else {
                // a (the last step of a batch) is stored straight from registers: staging it by TMA
                // needs the input tile, and serialising the next tile's load behind that store
                // measured no faster (1.02 vs ~1.0 ms at c4)
                wait(mb_v, ph);
                double *po = a.out ? a.out + base : nullptr;
#pragma unroll
                for (int j = 0; j < L; ++j) {
                    vb[j * SW_LW] = fma(a.kick, v[j], vb[j * SW_LW]);
                    if (po && j < nvl) po[(long)j * sl] = v[j];
                }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                const CUtensorMap *tm = kick ? &a.tm_v : &a.tm_out;
                const int i0 = (int)(tile % nib) * SW_LW, lb = (int)(tile / nib);
                for (int bb = 0; bb < a.nbox; ++bb) {
                    const unsigned d = (unsigned)__cvta_generic_to_shared(vbase + (long)bb * a.rb * SW_LW);
                    const int r0 = bb * a.rb;
                    const int c1 = a.dir == 1 ? r0 : lb, c2 = a.dir == 1 ? lb : r0;
                    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                                     reinterpret_cast<unsigned long long>(tm)),
                                 "r"(i0), "r"(c1), "r"(c2), "r"(d)
                                 : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            }
        }
        if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
}

// first tile origin: ilo - T when the Toeplitz interior exists (ilo <= ihi), else 0
__host__ __device__ inline int kop_origin(int ilo, int ihi, int T) { return ilo <= ihi ? ilo - T : 0; }

// ------------------------------------------------------------------------------------------
// fused drift + source + K-apply (v4, "K first")
//
//   P = U + tau V (written to Pout),  r = g (bx (x) by (x) bz) + sign K P,
//   K P = Mz [My (Kx P) + Mx (Ky P)] + Kz (Mx My P)   (Eq. 14, 3D)
//
// K_d annihilates constants, so K_d applied to a ROUNDED mass product amplifies its last-ulp
// noise by ~ (sigma/h)^2 on smooth data and D^-1 passes it on (T1: the v3 kernel, which
// formed Kx (My P) and Kz (Mx My P), missed the extended-precision step by 1e-11 at 512^3).  Here
//   - Kx and Ky act on P itself (K first), then My / Mx;
//   - Kz acts on T = Mx My P through plane differences: Kz T_k = sum_m wz[k][m] dT_{k-p+m} with
//     dT_j = T_{j+1} - T_j = Mx My (P_{j+1} - P_j); the in-plane mass products of the small
//     differences round at the differences' scale, not T's.  The 2p weights per row are built on
//     the host from the band row with the row sum the exact matrix has (0 in the interior; the
//     removed boundary column on Dirichlet rows, with T = 0 on the boundary plane).
//
// CTA = 256 threads on a K4_X x K4_Y = 32 x 16 output tile, marching along z over [z0, z1).
// Per input plane c (TMA box of U and V over the haloed tile, K4_NPF - 1 planes ahead):
//   A. P = U + tau V over the staged box, a column pair per thread step (16-byte shared loads and
//      stores), into a ring of three P tiles whose columns are the staging columns; zero on planes
//      outside memory and on zero-Dirichlet z faces (their Mz / Mx / My columns are zero, and they
//      count as zero in the plane differences); the owned P to HBM;
//   B. column items (column, 4 rows): Ky P_c and My D with D = P_c - P_{c-1} formed from two P
//      tiles of the ring; row items (row, 4 columns): Kx P_c;
//   C. lane = x, 2 rows per thread: G_c = My (Kx P) + Mx (Ky P) and dT_{c-1} = Mx (My D) on the
//      FP64 tensor cores (band fragments in registers), scattered with (Mz, wz) into a register ring
//      of 2p + 1 pending output planes; output plane c - p is complete: r = g src + sign ring.
// The three stages run skewed (A of plane ii, B of ii - 1, C of ii - 2) with one barrier per
// plane.  Interior tiles/planes use the Toeplitz rows (kernel parameters) in pair form; boundary
// tiles read staged rows, boundary planes read global rows.
// HBM traffic: U, V read once (halos from L2), P and r written once: 32 B/DOF.
// ------------------------------------------------------------------------------------------
constexpr int K4_X = 32, K4_Y = 16, K4_THREADS = 256, K4_NPF = 3, K4_XP = 36, K4_YQP = 44;
template <int P>
struct K4Geo {
    static constexpr int W = 2 * P + 1;
    static constexpr int PA = (P + 1) & ~1;             // even x halo of the TMA box
    static constexpr int SFT = PA - P;                  // staged column of haloed column 0 (0 or 1)
    static constexpr int HXE = K4_X + 2 * PA;           // staged columns
    static constexpr int HY = K4_Y + 2 * P;             // rows of the haloed tile
    static constexpr int NC = K4_X + 2 * P;             // columns of the haloed tile
    // P tile pitch: the staging row plus 2, so pitch/2 is odd (HXE/2 = 16 + PA is even) and the row
    // items' 16-byte loads (a quarter-warp = 2 rows x 4 column quads) hit 8 distinct bank groups
    static constexpr int PP = HXE + 2;
    static constexpr int NPR = HXE / 2;                 // column pairs per staged row
    static constexpr int NA = NPR * HY;                 // stage-A pairs
    static constexpr int SA = (NA + K4_THREADS - 1) / K4_THREADS;
    static constexpr int NCOL = NC * (K4_Y / 4);        // column items (4 output rows each)
    static constexpr int CW = (NCOL + 31) / 32;         // warps running column items
    static constexpr int RW = K4_THREADS / 32 - CW;     // warps running row items
    static constexpr int RG = (HY + 3) / 4;             // row-item groups of 4 rows x 8 column quads
    static constexpr int RWIN = 4 + 2 * P + 2 * SFT;    // row-item window from the aligned staged column
    static_assert(RW >= 1, "row-item warps");
    static constexpr int al16(int v) { return (v + 15) & ~15; }
    static constexpr int STG = al16(HXE * HY);          // one staged field plane (128-byte multiple)
    // stage C runs on the FP64 tensor cores: KS k-steps of 4 cover the 8 + 2p band columns of an 8-wide
    // output block; the (Ky P, My D) tile rows are padded to K4_YQP double2 and the Kx P tile to HX1
    // rows (zero: the fragments of the last block read past the haloed tile)
    static constexpr int KS = (8 + 2 * P + 3) / 4, HX1 = 8 + 4 * KS;
    static_assert(24 + 4 * KS <= K4_YQP && HX1 >= HY, "stage-C fragment windows");
    static constexpr int PT = al16(HY * PP), YQ = al16(K4_Y * K4_YQP * 2);
    static constexpr int X1 = al16(HX1 * K4_XP), XB = al16(K4_X * 2 * W), YB = al16(K4_Y * 2 * W);
    static constexpr int OFF_PT = K4_NPF * 2 * STG, OFF_YQ = OFF_PT + 3 * PT;
    static constexpr int OFF_X1 = OFF_YQ + 2 * YQ, OFF_XB = OFF_X1 + 2 * X1, OFF_YB = OFF_XB + XB;
    static constexpr int OFF_MB = OFF_YB + YB;
    static constexpr int SMEM = OFF_MB + 16 + 16;       // mbarriers + 128-byte alignment slack
};

extern __shared__ __align__(128) double k4_smem[];

__device__ __forceinline__ void k4_dmma(double (&d)[2], double a, double b) {
#ifdef ADS_ABL_NODMMA  // experiment builds only (scripts/ablate_kop.sh)
    d[0] += a; d[1] += b; return;
#endif
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void k4_wait(unsigned mb, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n K4W_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra K4W_%=;\n}\n" ::"r"(mb), "r"(parity) : "memory");
}

// stage A of one input plane: column pairs m of this thread (so_: staging offset, -1 none; po_: P
// tile offset; go_: global offset of the pair's first column; om_: bit 0/1 owned columns, bit 2 the
// pair store is 16-byte aligned).  KIND 0: no plane in memory (P = 0); 1: slab halo plane (P staged
// from Ph in the U half); 2: zero-Dirichlet z face (P = U + tau V to HBM, zero in the tile);
// 3: P = U + tau V
template <int P, int KIND>
__device__ __forceinline__ void k4_stage_a(double tau, const int (&so_)[K4Geo<P>::SA], const int (&po_)[K4Geo<P>::SA],
                                           const int (&go_)[K4Geo<P>::SA], const int (&om_)[K4Geo<P>::SA], int sbase,
                                           int pbase, double *pout) {
    using G = K4Geo<P>;
#pragma unroll
    for (int m = 0; m < G::SA; ++m) {
        if (G::NA % K4_THREADS != 0 && m == G::SA - 1 && so_[m] < 0) break;
        double2 p = make_double2(0.0, 0.0);
        if (KIND != 0) {
            const double2 u = *reinterpret_cast<const double2 *>(k4_smem + sbase + so_[m]);
            if (KIND == 1) p = u;
            else {
                const double2 v = *reinterpret_cast<const double2 *>(k4_smem + sbase + G::STG + so_[m]);
                p = make_double2(fma(tau, v.x, u.x), fma(tau, v.y, u.y));
            }
        }
        *reinterpret_cast<double2 *>(k4_smem + pbase + po_[m]) = KIND == 2 ? make_double2(0.0, 0.0) : p;
        if (KIND != 0 && pout) {
            const int om = om_[m];
            if (om == 7) *reinterpret_cast<double2 *>(pout + go_[m]) = p;
            else {
                if (om & 1) pout[go_[m]] = p.x;
                if (om & 2) pout[go_[m] + 1] = p.y;
            }
        }
    }
}

// z scatter of plane kk (ring slot U): G_kk with Mz(k, kk) into outputs k = kk-P .. kk+P and
// dT_{kk-1} with wz[k][kk-1-k+P] into outputs kk-P .. kk+P-1; returns the completed output kk - P
template <int P, int U>
__device__ __forceinline__ void k4_zscatter(const KopArgs &a, double (&A0)[2 * P + 1], double (&A1)[2 * P + 1],
                                            double g0, double g1, double d0, double d1, int kk, bool zint, double &o0,
                                            double &o1) {
    constexpr int W = 2 * P + 1;
    if (zint) {
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const int sl = ((U - P + c) % W + W) % W, d = c < P ? P - c : c - P;
            A0[sl] = fma(a.mc[2][P + d], g0, A0[sl]);
            A1[sl] = fma(a.mc[2][P + d], g1, A1[sl]);
            if (c < 2 * P) {  // output k = kk - P + c: dT_{kk-1} is its tap m = 2P - 1 - c
                A0[sl] = fma(a.wzc[2 * P - 1 - c], d0, A0[sl]);
                A1[sl] = fma(a.wzc[2 * P - 1 - c], d1, A1[sl]);
            }
        }
    } else {
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const int sl = ((U - P + c) % W + W) % W, k = kk - P + c;
            double mz_ = 0.0, wz_ = 0.0;
            if (k >= 0 && k < a.geo.n2) {
                mz_ = __ldg(a.mz + (long)(k + a.zoff) * W + 2 * P - c);
                if (c < 2 * P) wz_ = a.kw[2] * __ldg(a.wz + (long)(k + a.zoff) * (2 * P) + 2 * P - 1 - c);
            }
            A0[sl] = fma(mz_, g0, A0[sl]);
            A1[sl] = fma(mz_, g1, A1[sl]);
            A0[sl] = fma(wz_, d0, A0[sl]);
            A1[sl] = fma(wz_, d1, A1[sl]);
        }
    }
    constexpr int so = ((U - P) % W + W) % W;
    o0 = A0[so];
    o1 = A1[so];
    A0[so] = 0.0;
    A1[so] = 0.0;
}

template <int P, bool XI, bool YI>
__device__ __forceinline__ void kop4_tile(const KopArgs &a, const CUtensorMap *tmu, const CUtensorMap *tmv,
                                          const CUtensorMap *tmp, int sh, int x0, int y0, int z0, int z1) {
    using G = K4Geo<P>;
    constexpr int W = G::W, NC = G::NC, HY = G::HY, PP = G::PP, SFT = G::SFT;
    // shared memory: k4_smem[sh + offset]; sh aligns the TMA staging to 128 bytes
    double *const xb = k4_smem + sh + G::OFF_XB;  // [W][2][K4_X]: (Mx, kw0 Kx) rows of x0 + xr
    double *const yb = k4_smem + sh + G::OFF_YB;  // [K4_Y][2][W]: (My, kw1 Ky) rows of y0 + yr
    const unsigned mb0 = (unsigned)__cvta_generic_to_shared(k4_smem + sh + G::OFF_MB);
    const unsigned stg_s = (unsigned)__cvta_generic_to_shared(k4_smem + sh);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n0 = a.geo.n0, n1 = a.geo.n1;
    const long sy = a.geo.sy, sz = a.geo.sz;
    if (!XI)
        for (int e = tid; e < K4_X * 2 * W; e += K4_THREADS) {
            const int xr = e % K4_X, m = (e / K4_X) & 1, c = e / (2 * K4_X), X = x0 + xr;
            xb[e] = (X >= 0 && X < n0) ? (m ? a.kw[0] : 1.0) * __ldg((m ? a.kx : a.mx) + (long)X * W + c) : 0.0;
        }
    if (!YI)
        for (int e = tid; e < K4_Y * 2 * W; e += K4_THREADS) {
            const int yr = e / (2 * W), m = (e / W) & 1, c = e % W, Y = y0 + yr;
            yb[e] = (Y >= 0 && Y < n1) ? (m ? a.kw[1] : 1.0) * __ldg((m ? a.ky : a.my) + (long)Y * W + c) : 0.0;
        }
    // zero the stage-C fragment padding (never written by stage B) and the P tile of plane -1
    for (int e = tid; e < 2 * K4_Y * (K4_YQP - NC); e += K4_THREADS) {
        const int b = e / (K4_Y * (K4_YQP - NC)), q = e % (K4_Y * (K4_YQP - NC));
        reinterpret_cast<double2 *>(k4_smem + sh + G::OFF_YQ + b * G::YQ)[(q / (K4_YQP - NC)) * K4_YQP + NC + q % (K4_YQP - NC)] =
            make_double2(0.0, 0.0);
    }
    if constexpr (G::HX1 > HY)
        for (int e = tid; e < 2 * (G::HX1 - HY) * K4_XP; e += K4_THREADS) {
            const int b = e / ((G::HX1 - HY) * K4_XP), q = e % ((G::HX1 - HY) * K4_XP);
            k4_smem[sh + G::OFF_X1 + b * G::X1 + HY * K4_XP + q] = 0.0;
        }
    for (int e = tid; e < G::PT; e += K4_THREADS) k4_smem[sh + G::OFF_PT + 2 * G::PT + e] = 0.0;
    const int kk0 = z0 - P, npl = z1 - z0 + 2 * P;  // input planes z0 - P .. z1 + P - 1
    if (tid == 0) {
        for (int i = 0; i < K4_NPF; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mb0 + 8u * i) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // thread 0: stage input plane ii into slot ii % K4_NPF (planes outside [zv0, zv1) are zero:
    // nothing is loaded, the barrier phase completes by a plain arrival)
    auto issue = [&](int ii) {
        if (ii >= npl) return;
        const int kk = kk0 + ii, slot = ii % K4_NPF;
        const unsigned mb = mb0 + 8u * slot;
        if (a.Ph && kk >= a.zv0 && kk < a.zv1 && (kk < 0 || kk >= a.geo.n2)) {  // slab halo plane: P itself
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                         "r"((unsigned)(G::HXE * HY * sizeof(double)))
                         : "memory");
            const unsigned d = (unsigned)__cvta_generic_to_shared(k4_smem + sh + slot * 2 * G::STG);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d),
                "l"(reinterpret_cast<unsigned long long>(tmp)), "r"(x0 - G::PA), "r"(y0 - P), "r"(kk - a.zv0), "r"(mb)
                : "memory");
        } else if (kk >= a.zv0 && kk < a.zv1) {
#ifdef ADS_ABL_NOTMA  // experiment builds only: no plane loads
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mb) : "memory");
            return;
#endif
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb),
                         "r"((unsigned)(2 * G::HXE * HY * sizeof(double)))
                         : "memory");
            const unsigned d = stg_s + slot * 2 * G::STG * 8u;
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d),
                "l"(reinterpret_cast<unsigned long long>(tmu)), "r"(x0 - G::PA), "r"(y0 - P), "r"(kk - a.zv0), "r"(mb)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d + G::STG * 8u),
                "l"(reinterpret_cast<unsigned long long>(tmv)), "r"(x0 - G::PA), "r"(y0 - P), "r"(kk - a.zv0), "r"(mb)
                : "memory");
        } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(mb) : "memory");
        }
    };
    pdl_wait();  // fields (U, V, dstep) from here on
    if (tid == 0)
        for (int i = 0; i < K4_NPF - 1; ++i) issue(i);

    // stage-A pairs of this thread: staging / P tile / global offsets and ownership
    int so_[G::SA], po_[G::SA], go_[G::SA], om_[G::SA];
#pragma unroll
    for (int m = 0; m < G::SA; ++m) {
        const int e = tid + K4_THREADS * m, hy = e / G::NPR, cp = e - hy * G::NPR;
        const int X = x0 - G::PA + 2 * cp, Y = y0 - P + hy;  // global column of the pair's first element
        so_[m] = e < G::NA ? hy * G::HXE + 2 * cp : -1;
        po_[m] = e < G::NA ? hy * PP + 2 * cp : 0;
        const bool yo = e < G::NA && hy >= P && hy < P + K4_Y && Y >= 0 && Y < n1;
        const bool o0 = yo && X >= x0 && X < x0 + K4_X && X >= 0 && X < n0;
        const bool o1 = yo && X + 1 >= x0 && X + 1 < x0 + K4_X && X + 1 >= 0 && X + 1 < n0;
        go_[m] = Y * (int)sy + X;
        om_[m] = (o0 ? 1 : 0) | (o1 ? 2 : 0) | ((X & 1) == 0 ? 4 : 0);
    }
    double A0[W], A1[W];
#pragma unroll
    for (int c = 0; c < W; ++c) A0[c] = A1[c] = 0.0;

    // stage-C constants: warp w owns the 8 x 8 output block (rows 8 mi.., columns 8 nj..), lane l the
    // outputs (row y0 + 8 mi + l/4, columns x0 + 8 nj + 2 (l%4) + {0, 1}); tiles start at ilo - 32 /
    // ilo - 16 (interior alignment): rows and columns can be negative
    const int mi = w >> 2, nj = w & 3;
    const int Yo = y0 + 8 * mi + (lane >> 2), X = x0 + 8 * nj + 2 * (lane & 3);
    const bool yin = Yo >= 0 && Yo < n1;
    const bool own0 = yin && X >= 0 && X < n0, own1 = yin && X + 1 >= 0 && X + 1 < n0;
    const bool has_src = a.bx != nullptr;
    const double sxy0 = (has_src && own0) ? __ldg(a.bx + X) * __ldg(a.by + Yo) : 0.0;
    const double sxy1 = (has_src && own1) ? __ldg(a.bx + X + 1) * __ldg(a.by + Yo) : 0.0;
    // band fragments (constant over the planes), per k step s4 (k = 4 s4 + l%4):
    // B[k][n] = Mx(x0 + 8 nj + n, band c = k - n), n = l/4;  A[m][k] = My(y0 + 8 mi + m, band c = k - m)
    double frx[G::KS], fry[G::KS];
#pragma unroll
    for (int s4 = 0; s4 < G::KS; ++s4) {
        const int cb = 4 * s4 + (lane & 3) - (lane >> 2);
        const int xr = x0 + 8 * nj + (lane >> 2), yr = y0 + 8 * mi + (lane >> 2);
        double vx = 0.0, vy = 0.0;
        if (cb >= 0 && cb <= 2 * P) {
            vx = XI ? a.mc[0][cb] : (xr >= 0 && xr < n0 ? __ldg(a.mx + (long)xr * W + cb) : 0.0);
            vy = YI ? a.mc[1][cb] : (yr >= 0 && yr < n1 ? __ldg(a.my + (long)yr * W + cb) : 0.0);
        }
        frx[s4] = vx;
        fry[s4] = vy;
    }
    double gsrc = a.g;
    if (has_src && a.dstep) {  // source time from the device step counter (CUDA graph replays)
        const double x = 3.141592653589793238462643383 * a.f0 * ((double)(*a.dstep + 1) * a.tau_g - a.t0);
        gsrc = a.amp * (a.wav ? (1.0 - 2.0 * x * x) * exp(-x * x) : 1.0);
    }
    double *rq = a.r + (long)Yo * sy + X + (long)z0 * sz;
    const bool pair = own0 && own1 && (reinterpret_cast<unsigned long long>(rq) & 15) == 0;  // sz keeps it
    // stage-B column item (threads [0, NCOL)) and row item (warps [CW, 8)) constants
    const int nc = tid % NC, g4 = tid / NC;
    const int rq4 = (lane & 3) + 4 * (lane >> 4), rsub = (lane >> 2) & 3;

    // one plane step; ST: a steady-state plane (every stage active, a plain interior input plane,
    // Toeplitz z rows, an owned output plane), which skips the per-plane case analysis
    auto plane = [&](const int ii, auto st_tag) {
        constexpr bool ST = decltype(st_tag)::value;
#ifndef ADS_ABL_NOSYNC
        __syncthreads();  // C(ii-3), B(ii-2), A(ii-1) done: tiles, staging slot (ii-1) % K4_NPF free
#endif
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(ii + K4_NPF - 1);
        }
        // program order C, B, A: no stage reads what another writes in this interval, and C's
        // shared loads, then B's, go first (the compiler cannot hoist a shared load above a
        // shared store it cannot disambiguate); only A waits for the TMA of plane ii
        // ---- C: plane c = kk0 + ic: G = My (Kx P) + Mx (Ky P), dT_{c-1} = Mx (My D) into the z ring.
        // DMMA m8n8k4: warp w owns the 8 x 8 block (rows 8 mi.., columns 8 nj..); lane l its outputs
        // (row 8 mi + l/4, columns 8 nj + 2 (l%4) + {0, 1}).  Mx acts as the B operand (band, in
        // registers) on the (Ky P, My D) rows, My as the A operand on the Kx P columns.
        const int ic = ii - 2;
        if (ST || ic >= 0) {
            const int b = ic & 1, kc_ = kk0 + ic, kout = kc_ - P;
            const double2 *Yq = reinterpret_cast<const double2 *>(k4_smem + sh + G::OFF_YQ + b * G::YQ) +
                                (8 * mi + (lane >> 2)) * K4_YQP + 8 * nj + (lane & 3);
            const double *Xq = k4_smem + sh + G::OFF_X1 + b * G::X1 + (8 * mi + (lane & 3)) * K4_XP + 8 * nj + (lane >> 2);
            double gacc[2] = {0.0, 0.0}, hacc[2] = {0.0, 0.0}, tacc[2] = {0.0, 0.0};
#pragma unroll
            for (int s4 = 0; s4 < G::KS; ++s4) {
                const double2 av = Yq[4 * s4];
                const double bv = Xq[4 * s4 * K4_XP];
                k4_dmma(gacc, av.x, frx[s4]);
                k4_dmma(tacc, av.y, frx[s4]);
                k4_dmma(hacc, fry[s4], bv);
            }
            // (two accumulators per product, even / odd k steps, measured no faster and change the
            // rounding of a by ~1e-11 at p = 5: single chains)
            const double g0 = gacc[0] + hacc[0], g1 = gacc[1] + hacc[1], t0 = tacc[0], t1 = tacc[1];
            const bool zint = ST || (kc_ + a.zoff - P >= a.ilo[2] && kc_ + a.zoff + P <= a.ihi[2]);
            double o0 = 0.0, o1 = 0.0;  // t0, t1: dT_{c-1} = Mx My D of the lane's two outputs
#ifdef ADS_ABL_NOZ
            o0 = g0 + t0; o1 = g1 + t1;
            if (false)
#endif
            switch (ic % W) {
#define ADS_K4C(U)                                                                      \
    case U:                                                                             \
        if constexpr (U < W) k4_zscatter<P, U>(a, A0, A1, g0, g1, t0, t1, kc_, zint, o0, o1); \
        break;
                ADS_K4C(0) ADS_K4C(1) ADS_K4C(2) ADS_K4C(3) ADS_K4C(4) ADS_K4C(5)
                ADS_K4C(6) ADS_K4C(7) ADS_K4C(8) ADS_K4C(9) ADS_K4C(10)
#undef ADS_K4C
            }
            if (ST || kout >= z0) {  // output plane kout = c - P: r = g src + sign K P
                const double gz = has_src ? gsrc * __ldg(a.bz + kout + a.zoff) : 0.0;
                const double r0 = fma(a.sign, o0, gz * sxy0), r1 = fma(a.sign, o1, gz * sxy1);
                if (pair) *reinterpret_cast<double2 *>(rq) = make_double2(r0, r1);
                else if (own0) rq[0] = r0;
                else if (own1) rq[1] = r1;
                rq += sz;
            }
        }
        // ---- B: plane c = kk0 + ib (Ky P, Kx P) and D = P_c - P_{c-1} (My D)
        const int ib = ii - 1;
        if (ST || (ib >= 0 && ib < npl)) {
            const int b = ib & 1;
            const double *pt = k4_smem + sh + G::OFF_PT + (ib % 3) * G::PT;
            if (w < G::CW) {
                if (tid < G::NCOL) {
                    const int off = (4 * g4) * PP + nc + SFT;
                    double pw[4 + 2 * P], dw[4 + 2 * P];
#pragma unroll
                    for (int r = 0; r < 4 + 2 * P; ++r) {
                        pw[r] = pt[off + r * PP];
                        // plane c - 1 from its tile (keeping the item's previous window in registers
                        // measured the same time at c4 and spills at p = 3)
                        dw[r] = pw[r] - k4_smem[sh + G::OFF_PT + ((ib + 2) % 3) * G::PT + off + r * PP];
                    }
                    double ky[4], mq[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
#ifdef ADS_ABL_NOCOL
                        ky[r] = pw[r] + pw[r + 2 * P]; mq[r] = dw[r] + dw[r + 2 * P]; continue;
#endif
                        if (YI) {
                            double s = a.kc[1][P] * pw[r + P], t = a.mc[1][P] * dw[r + P];
#pragma unroll
                            for (int d = 1; d <= P; ++d) {
                                s = fma(a.kc[1][P + d], pw[r + P - d] + pw[r + P + d], s);
                                t = fma(a.mc[1][P + d], dw[r + P - d] + dw[r + P + d], t);
                            }
                            ky[r] = s;
                            mq[r] = t;
                        } else {
                            const double *rk = yb + ((4 * g4 + r) * 2 + 1) * W, *rm = yb + ((4 * g4 + r) * 2) * W;
                            double s = 0.0, t = 0.0;
#pragma unroll
                            for (int c = 0; c < W; ++c) {
                                s = fma(rk[c], pw[r + c], s);
                                t = fma(rm[c], dw[r + c], t);
                            }
                            ky[r] = s;
                            mq[r] = t;
                        }
                    }
                    double2 *o = reinterpret_cast<double2 *>(k4_smem + sh + G::OFF_YQ + b * G::YQ) + (4 * g4) * K4_YQP + nc;
#pragma unroll
                    for (int r = 0; r < 4; ++r) o[r * K4_YQP] = make_double2(ky[r], mq[r]);
                }
            } else {
                // row items: a warp covers 4 rows x 8 column quads (16-byte window loads from the
                // aligned staged column 4 q; haloed column 4 q + j is window element j + SFT)
#pragma unroll 1
                for (int t = 0; t < (G::RG + G::RW - 1) / G::RW; ++t) {
                    const int hy = 4 * (w - G::CW + t * G::RW) + rsub;
                    if (hy < HY) {
                        const double2 *src = reinterpret_cast<const double2 *>(pt + hy * PP + 4 * rq4);
                        double pw[G::RWIN];
#pragma unroll
                        for (int j = 0; j < G::RWIN / 2; ++j) {
                            const double2 v = src[j];
                            pw[2 * j] = v.x;
                            pw[2 * j + 1] = v.y;
                        }
                        double kx[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
#ifdef ADS_ABL_NOROW
                            kx[j] = pw[j] + pw[j + 2 * P]; continue;
#endif
                            if (XI) {
                                double s = a.kc[0][P] * pw[j + P + SFT];
#pragma unroll
                                for (int d = 1; d <= P; ++d)
                                    s = fma(a.kc[0][P + d], pw[j + P + SFT - d] + pw[j + P + SFT + d], s);
                                kx[j] = s;
                            } else {
                                double s = 0.0;
#pragma unroll
                                for (int c = 0; c < W; ++c) s = fma(xb[(c * 2 + 1) * K4_X + 4 * rq4 + j], pw[j + c + SFT], s);
                                kx[j] = s;
                            }
                        }
                        // odd quads store their second half first: each quarter-warp store then hits 8
                        // distinct bank groups (row pitch 18 x 16 bytes)
                        double2 *o = reinterpret_cast<double2 *>(k4_smem + sh + G::OFF_X1 + b * G::X1 + hy * K4_XP + 4 * rq4);
                        const int sw = lane & 1;
                        o[sw] = sw ? make_double2(kx[2], kx[3]) : make_double2(kx[0], kx[1]);
                        o[sw ^ 1] = sw ? make_double2(kx[0], kx[1]) : make_double2(kx[2], kx[3]);
                    }
                }
            }
        }
        // ---- A: input plane kk = kk0 + ii into P tile ii % 3
        if (ST || ii < npl) {
#ifndef ADS_ABL_NOWAIT  // experiment builds only: data races, timing of the rest
            k4_wait(mb0 + 8u * (ii % K4_NPF), (unsigned)((ii / K4_NPF) & 1));
#endif
            const int kk = kk0 + ii;
            const int sb = sh + (ii % K4_NPF) * 2 * G::STG, pb = sh + G::OFF_PT + (ii % 3) * G::PT;
            double *const po = (a.Pout && kk >= z0 && kk < z1) ? a.Pout + (long)kk * sz : nullptr;
            if (ST) k4_stage_a<P, 3>(a.tau, so_, po_, go_, om_, sb, pb, po);
            else if (!(kk >= a.zv0 && kk < a.zv1)) k4_stage_a<P, 0>(a.tau, so_, po_, go_, om_, sb, pb, po);
            else if (a.Ph && (kk < 0 || kk >= a.geo.n2)) k4_stage_a<P, 1>(a.tau, so_, po_, go_, om_, sb, pb, po);
            else if (kk + a.zoff == a.zd0 || kk + a.zoff == a.zd1) k4_stage_a<P, 2>(a.tau, so_, po_, go_, om_, sb, pb, po);
            else k4_stage_a<P, 3>(a.tau, so_, po_, go_, om_, sb, pb, po);
        }
    };
    // steady range [ss0, ss1): ii >= 2 + 2p (stages B, C active, output owned), input plane plain
    // (in memory, not a slab halo, not a zero-Dirichlet face), zint for the stage-C plane ii - 2
    int klo = a.zv0, khi = a.zv1;
    if (a.Ph) {
        klo = max(klo, 0);
        khi = min(khi, a.geo.n2);
    }
    if (a.zd0 >= 0) klo = max(klo, a.zd0 - a.zoff + 1);
    if (a.zd1 >= 0) khi = min(khi, a.zd1 - a.zoff);
    const int ss0 = max(max(2 + 2 * P, klo - kk0), a.ilo[2] - a.zoff + P - kk0 + 2);
    const int ss1 = max(ss0, min(min(npl, khi - kk0), a.ihi[2] - a.zoff - P - kk0 + 3));
    using SF = std::integral_constant<bool, false>;
    using STT = std::integral_constant<bool, true>;
    for (int ii = 0; ii < ss0; ++ii) plane(ii, SF{});
    for (int ii = ss0; ii < ss1; ++ii) plane(ii, STT{});
    for (int ii = ss1; ii < npl + 2; ++ii) plane(ii, SF{});
}

template <int P>
__global__ void __launch_bounds__(K4_THREADS, P <= 3 ? 2 : 1)
    kop4_kernel(const KopArgs a, const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmv,
                const __grid_constant__ CUtensorMap tmp) {
    pdl_launch_dependents();
    // TMA staging needs 128-byte alignment of the dynamic shared memory window
    const int sh = (int)(((128 - (__cvta_generic_to_shared(k4_smem) & 127)) & 127) / sizeof(double));
    const int x0 = kop_origin(a.ilo[0], a.ihi[0], K4_X) + (int)blockIdx.x * K4_X;
    const int y0 = kop_origin(a.ilo[1], a.ihi[1], K4_Y) + (int)blockIdx.y * K4_Y;
    const int z0 = blockIdx.z * a.zlen, z1 = min(a.geo.n2, z0 + a.zlen);
    const bool xi = x0 >= a.ilo[0] && x0 + K4_X - 1 <= a.ihi[0];
    const bool yi = y0 >= a.ilo[1] && y0 + K4_Y - 1 <= a.ihi[1];
    if (xi && yi) kop4_tile<P, true, true>(a, &tmu, &tmv, &tmp, sh, x0, y0, z0, z1);
    else if (xi) kop4_tile<P, true, false>(a, &tmu, &tmv, &tmp, sh, x0, y0, z0, z1);
    else if (yi) kop4_tile<P, false, true>(a, &tmu, &tmv, &tmp, sh, x0, y0, z0, z1);
    else kop4_tile<P, false, false>(a, &tmu, &tmv, &tmp, sh, x0, y0, z0, z1);
}

// ------------------------------------------------------------------------------------------
// distributed z-solve fix-up + kick (see kernels.cuh ZfixArgs).  Thread per z-line and z piece
// of 32 planes (coalesced across x; each piece recomputes the line's interface values from the
// tips), streaming the nl owned planes once: 24 B/DOF (+8 when a is kept).
// ------------------------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void zload(const double *f, long base, long sz, int k0, double (&t)[P]) {
#pragma unroll
    for (int m = 0; m < P; ++m) t[m] = f ? f[base + (long)(k0 + m) * sz] : 0.0;
}

// stage 1: the two interface systems of this slab without their outer couplings
template <int P>
__global__ void __launch_bounds__(128) zint_kernel(const ZfixArgs a) {
    const Geom &g = a.geo;
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
    if (i >= g.n0 || j >= g.n1) return;
    const int nl = g.n2;
    const long base = (long)j * g.sy + i;
    double tp[P], xf[P], xl[P], tn[P];
    zload<P>(a.tip_prev, base, g.sz, 0, tp);
    zload<P>(a.X, base, g.sz, 0, xf);
    zload<P>(a.X, base, g.sz, nl - P, xl);
    zload<P>(a.tip_next, base, g.sz, 0, tn);
#pragma unroll
    for (int r = 0; r < P; ++r) {
        double b = 0.0, u = 0.0;
#pragma unroll
        for (int c = 0; c < P; ++c) {
            b = fma(a.qt[r][c], tp[c], fma(a.qt[r][P + c], xf[c], b));
            u = fma(a.qb[P + r][c], xl[c], fma(a.qb[P + r][P + c], tn[c], u));
        }
        if (a.tip_prev) a.b0buf[base + (long)r * g.sz] = b;
        if (a.tip_next) a.u0buf[base + (long)r * g.sz] = u;
    }
}

// stage 2 + correction + kick: thread per z-line of the slab (coalesced across x), streaming
// the nl owned planes once: 24 B/DOF (+8 when a is kept)
constexpr int ZF_X = 32, ZF_Y = 4, ZF_Z = 32;  // thread block 32 x 4 lines, z pieces of 32 planes
template <int P>
__global__ void __launch_bounds__(ZF_X * ZF_Y) zfix_kernel(const ZfixArgs a) {
    const Geom &g = a.geo;
    const int i = blockIdx.x * ZF_X + threadIdx.x, j = blockIdx.y * ZF_Y + threadIdx.y;
    if (i >= g.n0 || j >= g.n1) return;
    const int nl = g.n2;
    const long base = (long)j * g.sy + i;
    double bp[P], un[P];
#pragma unroll
    for (int m = 0; m < P; ++m) bp[m] = un[m] = 0.0;
    if (a.tip_prev) {  // top interface (j-1|j): rhs corrected by b_{j-2}^0 and u_{j+1}^0
        double tp[P], xf[P], b2[P], u1[P];
        zload<P>(a.tip_prev, base, g.sz, 0, tp);
        zload<P>(a.X, base, g.sz, 0, xf);
        zload<P>(a.b0_prev2, base, g.sz, 0, b2);
        zload<P>(a.tip_next ? a.u0buf : nullptr, base, g.sz, 0, u1);
#pragma unroll
        for (int r = 0; r < P; ++r)
#pragma unroll
            for (int c = 0; c < P; ++c) {
                tp[r] = fma(-a.wbp[r][c], b2[c], tp[r]);
                xf[r] = fma(-a.vtm[r][c], u1[c], xf[r]);
            }
#pragma unroll
        for (int r = 0; r < P; ++r)
#pragma unroll
            for (int c = 0; c < P; ++c) bp[r] = fma(a.qt[r][c], tp[c], fma(a.qt[r][P + c], xf[c], bp[r]));
    }
    if (a.tip_next) {  // bottom interface (j|j+1): rhs corrected by b_{j-1}^0 and u_{j+2}^0
        double xl[P], tn[P], b1[P], u2[P];
        zload<P>(a.X, base, g.sz, nl - P, xl);
        zload<P>(a.tip_next, base, g.sz, 0, tn);
        zload<P>(a.tip_prev ? a.b0buf : nullptr, base, g.sz, 0, b1);
        zload<P>(a.u0_next2, base, g.sz, 0, u2);
#pragma unroll
        for (int r = 0; r < P; ++r)
#pragma unroll
            for (int c = 0; c < P; ++c) {
                xl[r] = fma(-a.wbm[r][c], b1[c], xl[r]);
                tn[r] = fma(-a.vtn[r][c], u2[c], tn[r]);
            }
#pragma unroll
        for (int r = 0; r < P; ++r)
#pragma unroll
            for (int c = 0; c < P; ++c) un[r] = fma(a.qb[P + r][c], xl[c], fma(a.qb[P + r][P + c], tn[c], un[r]));
    }
    // the planes of this z piece (the fix-up of each plane is independent given the tips);
    // restrict-qualified copies let the loads of later planes move ahead of the stores
    const double *__restrict__ X = a.X;
    double *__restrict__ Vf = a.Vf;
    double *__restrict__ A = a.A;
    const int k0 = blockIdx.z * ZF_Z, k1 = min(nl, k0 + ZF_Z);
#pragma unroll 4
    for (int k = k0; k < k1; ++k) {
        const long idx = base + (long)k * g.sz;
        double x = X[idx];
        const double v = Vf[idx];
#pragma unroll
        for (int m = 0; m < P; ++m) {
            x = fma(-__ldg(a.Wsp + (long)k * P + m), bp[m], x);
            x = fma(-__ldg(a.Vsp + (long)k * P + m), un[m], x);
        }
        Vf[idx] = fma(a.kick, x, v);
        if (A) A[idx] = x;
    }
}

int launch_zint(int p, const ZfixArgs &a, cudaStream_t s) {
    dim3 blk(128), grd((a.geo.n0 + 127) / 128, a.geo.n1);
    switch (p) {
        case 1: zint_kernel<1><<<grd, blk, 0, s>>>(a); break;
        case 2: zint_kernel<2><<<grd, blk, 0, s>>>(a); break;
        case 3: zint_kernel<3><<<grd, blk, 0, s>>>(a); break;
        case 4: zint_kernel<4><<<grd, blk, 0, s>>>(a); break;
        case 5: zint_kernel<5><<<grd, blk, 0, s>>>(a); break;
        default: return -1;
    }
    return 0;
}

int launch_zfix(int p, const ZfixArgs &a, cudaStream_t s) {
    dim3 blk(ZF_X, ZF_Y), grd((a.geo.n0 + ZF_X - 1) / ZF_X, (a.geo.n1 + ZF_Y - 1) / ZF_Y, (a.geo.n2 + ZF_Z - 1) / ZF_Z);
    switch (p) {
        case 1: zfix_kernel<1><<<grd, blk, 0, s>>>(a); break;
        case 2: zfix_kernel<2><<<grd, blk, 0, s>>>(a); break;
        case 3: zfix_kernel<3><<<grd, blk, 0, s>>>(a); break;
        case 4: zfix_kernel<4><<<grd, blk, 0, s>>>(a); break;
        case 5: zfix_kernel<5><<<grd, blk, 0, s>>>(a); break;
        default: return -1;
    }
    return 0;
}

// Kronecker triples out = beta out + sum_t alpha_t (Fx_t (x) Fy_t (x) Fz_t) in, t < T <= 2, sharing
// input and output (elasticity couplings: the two triples of an off-diagonal
// block Upsilon_ik go in one pass; general bands, no Toeplitz assumption).
// 32 x 16 output tile marching z over a piece [z0, z1) of at most KR_ZMAX planes; per input plane
// (one barrier):
//   - all threads stream the haloed plane HBM -> shared memory in 16-byte zero-filling cp.async
//     pieces, KR_NPF - 1 planes ahead;
//   - y-pass items (column, 4 rows): Y = Fy in from a register window of 4 + 2p rows into a
//     double-buffered Y tile;
//   - x-pass of the previous plane (lane = x, 2 rows per thread, the lane's Fx rows in registers):
//     X = Fx Y;
//   - z: a register ring of the last 2p + 1 X planes, indexed statically (the march is dispatched
//     on the plane index mod 2p + 1, so no ring shifts); output plane kk - 2p ... gathered with the
//     piece's alpha_t Fz_t rows, staged once in shared memory.
// HBM traffic: in read once (halos from L2), out written once (read once when beta != 0).
#ifndef ADS_KR_RY
#define ADS_KR_RY 4
#endif
constexpr int KR_X = 32, KR_Y = 16, KR_THREADS = 256, KR_NPF = 4, KR_RY = ADS_KR_RY, KR_ZMAX = 160;
template <int P, int T>
struct KronGeo {
    static constexpr int W = 2 * P + 1;
    static constexpr int PA = (P + 1) & ~1;  // even x halo of the copied tile (16-byte pieces)
    static constexpr int HX = KR_X + 2 * PA, HY = KR_Y + 2 * P, HN = HX * HY;
    static constexpr int NC = KR_X + 2 * P;  // columns the x-pass needs
    static constexpr int NITEM = NC * (KR_Y / KR_RY);
    static constexpr int NPAIR = HN / 2, NSLOT = (NPAIR + KR_THREADS - 1) / KR_THREADS;
    // shared memory (doubles): ring [NPF][HY][HX] | Y tiles [2][KR_Y][NC][T] | Fy [T][KR_Y][W] |
    // alpha Fz [KR_ZMAX][W][T]
    static constexpr int RING = KR_NPF * HN, YT = 2 * KR_Y * NC * T, YB = T * KR_Y * W, ZB = KR_ZMAX * W * T;
    static_assert(RING % 2 == 0 && YT % 2 == 0 && (T == 1 || YB % 2 == 0), "16-byte aligned Fy / Fz tables");
    static constexpr int SMEM = RING + YT + YB + ZB;
    static_assert(NITEM <= 2 * KR_THREADS, "at most two y-pass items per thread");
};

// T terms sharing the input and the output: out = beta out + sum_t alpha_t (Fx_t (x) Fy_t (x) Fz_t) in
// SH (pairs): a factor both terms share, detected on the host by band identity: 1 = F_y (one y
// product Y, both x products from it), 2 = F_z (alpha_t folded into F_x: one ring X = sum_t alpha_t
// F_x,t Y_t and one gather); 0 = none.  TY / TZ: y products / z rings per point.
template <int P, int T, bool YT, int SH>
__device__ __forceinline__ void kron3_tile(const double *__restrict__ in, double *__restrict__ out, const KronTerms &k3,
                                           double beta, const Geom &g, int zlen) {
    using G = KronGeo<P, T>;
    constexpr int W = G::W, HX = G::HX, HN = G::HN, NC = G::NC, PA = G::PA;
    constexpr int TY = SH == 1 ? 1 : T, TZ = SH == 2 ? 1 : T;
    extern __shared__ __align__(16) double smem[];
    double *ring = smem;
    double *Ys = smem + G::RING;  // [2][KR_Y][NC][TY]
    double *cy = Ys + G::YT;      // [KR_Y][W][T]: Fy_t rows of y0 + row (both terms of a tap adjacent)
    double *fzs = cy + G::YB;     // [z1 - z0][W][TZ]: alpha_t Fz_t rows of the piece's output planes (SH 2: Fz)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int n0 = g.n0, n1 = g.n1, n2 = g.n2;
    const long sy = g.sy, sz = g.sz;
    const int x0 = blockIdx.x * KR_X, y0 = blockIdx.y * KR_Y;
    const int z0 = blockIdx.z * zlen, z1 = min(n2, z0 + zlen);
    for (int e = tid; e < KR_Y * W; e += KR_THREADS) {
        const int yr = e / W, c = e % W, Y = y0 + yr;
#pragma unroll
        for (int t = 0; t < T; ++t) cy[e * T + t] = Y < n1 ? __ldg(k3.fy[t] + (long)Y * W + c) : 0.0;
    }
    for (int e = tid; e < (z1 - z0) * W; e += KR_THREADS) {
        const int c = e % W, k = z0 + e / W;
#pragma unroll
        for (int t = 0; t < TZ; ++t)
            fzs[e * TZ + t] = (SH == 2 ? 1.0 : k3.alpha[t]) * __ldg(k3.fz[t] + (long)k * W + c);
    }
    const int X = x0 + lane, Yo = y0 + 2 * w;
    double fxr[T][W];  // Fx_t row of this lane's column
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
        for (int c = 0; c < W; ++c) fxr[t][c] = X < n0 ? (SH == 2 ? k3.alpha[t] : 1.0) * __ldg(k3.fx[t] + (long)X * W + c) : 0.0;
    // copies: 16-byte pieces e = tid + 256 m of the [HY][HX/2] plane
    int goff[G::NSLOT];
    unsigned inr = 0;
#pragma unroll
    for (int m = 0; m < G::NSLOT; ++m) {
        const int e = tid + m * KR_THREADS, hy = e / (HX / 2), hx = 2 * (e - hy * (HX / 2));
        const int Xg = x0 - PA + hx, Yg = y0 - P + hy;
        const bool ok = e < G::NPAIR && Xg >= 0 && Xg < n0 && Yg >= 0 && Yg < n1;
        goff[m] = ok ? (Yg * (int)sy + Xg) : 0;
        if (ok) inr |= 1u << m;
    }
    const int kk0 = z0 - P, npl = z1 - z0 + 2 * P;  // input planes z0 - p .. z1 + p - 1
    const unsigned ring_s = (unsigned)__cvta_generic_to_shared(ring) + 16u * tid;
    auto issue = [&](int ii) {
        if (ii < npl) {
            const int kk = kk0 + ii;
            const bool kv = kk >= 0 && kk < n2;
            const double *pin = in + (kv ? (long)kk * sz : 0);
            const unsigned su = ring_s + 8u * (unsigned)((ii & (KR_NPF - 1)) * HN);
#pragma unroll
            for (int m = 0; m < G::NSLOT; ++m) {
                if (tid + m * KR_THREADS >= G::NPAIR) break;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(su + 16u * m * KR_THREADS),
                             "l"(pin + goff[m]), "r"((kv && (inr >> m & 1)) ? 16u : 0u)
                             : "memory");
            }
        }
        cp_async_commit();
    };
    const int hcol0 = PA - P;
    const bool own0 = X < n0 && Yo < n1, own1 = X < n0 && Yo + 1 < n1;
    double r0[TZ][W], r1[TZ][W];  // X_t planes by slot: plane q in slot q mod W
#pragma unroll
    for (int t = 0; t < TZ; ++t)
#pragma unroll
        for (int c = 0; c < W; ++c) r0[t][c] = r1[t][c] = 0.0;
    // the old out / addend of output plane k (beta != 0) is loaded one plane ahead: a synchronous
    // read-modify-write would stall every plane on DRAM latency
    double ob0 = 0.0, ob1 = 0.0;
    const long oxy = (long)Yo * sy + X;
    const double *ad = k3.addend ? k3.addend : out;
    auto prefetch = [&](int k) {
        if (beta != 0.0 && k >= z0 && k < z1) {
            ob0 = own0 ? ad[(long)k * sz + oxy] : 0.0;
            ob1 = own1 ? ad[(long)k * sz + oxy + sy] : 0.0;
        }
    };
    pdl_wait();  // fields from here on
    prefetch(z0);
#pragma unroll
    for (int i = 0; i < KR_NPF - 1; ++i) issue(i);
    __syncthreads();  // band rows staged
    // one plane step; U = slot of the x-pass plane kx = kk0 + ii - 1 (kx mod W)
    auto plane = [&](const int ii, auto u_tag) {
        constexpr int U = decltype(u_tag)::value;
        if (ii < npl) cp_async_wait<KR_NPF - 2>();
        __syncthreads();  // plane ii landed; Y tile (ii - 1) & 1 complete; ring slot (ii - 1) free
        issue(ii + KR_NPF - 1);
        // y-pass of input plane kk0 + ii, every term from one window: item = (column, KR_RY rows)
        auto ypass = [&](const int item) {
            const int nc = item % NC, grp = item / NC, hcol = hcol0 + nc;
            const double *b = ring + (ii & (KR_NPF - 1)) * HN + KR_RY * grp * HX + hcol;
            double pr[KR_RY + 2 * P];
#pragma unroll
            for (int r = 0; r < KR_RY + 2 * P; ++r) pr[r] = b[r * HX];
            double *yb = Ys + ((ii & 1) * KR_Y * NC + KR_RY * grp * NC + nc) * TY;
#pragma unroll
            for (int r = 0; r < KR_RY; ++r) {
                double acc[TY];
                [[maybe_unused]] const double *c = cy + (KR_RY * grp + r) * W * T;
#pragma unroll
                for (int t = 0; t < TY; ++t) acc[t] = 0.0;
#pragma unroll
                for (int q = 0; q < W; ++q) {
                    if constexpr (YT) {  // Toeplitz rows: the coefficients are kernel parameters
#pragma unroll
                        for (int t = 0; t < TY; ++t) acc[t] = fma(k3.fyrow[t][q], pr[r + q], acc[t]);
                    } else if constexpr (TY == 2) {  // both terms' tap q in one 16-byte load
                        const double2 cq = reinterpret_cast<const double2 *>(c)[q];
                        acc[0] = fma(cq.x, pr[r + q], acc[0]);
                        acc[1] = fma(cq.y, pr[r + q], acc[1]);
                    } else {
                        acc[0] = fma(c[q * T], pr[r + q], acc[0]);
                    }
                }
                if constexpr (TY == 2) reinterpret_cast<double2 *>(yb)[r * NC] = make_double2(acc[0], acc[1]);
                else yb[r * NC] = acc[0];
            }
        };
        if (ii < npl) {
            if (tid < G::NITEM) ypass(tid);
            if constexpr (G::NITEM > KR_THREADS)
                if (tid + KR_THREADS < G::NITEM) ypass(tid + KR_THREADS);
        }
        if (ii == 0) return;
        // x-pass of input plane kx = kk0 + ii - 1, then the z gather for output kx - p
        const int kx = kk0 + ii - 1;
        const double *yr0 = Ys + (((ii - 1) & 1) * KR_Y * NC + (2 * w) * NC + lane) * TY, *yr1 = yr0 + NC * TY;
#pragma unroll
        for (int t = 0; t < TZ; ++t) r0[t][U] = r1[t][U] = 0.0;
#pragma unroll
        for (int c = 0; c < W; ++c) {
            if constexpr (SH == 1) {  // one Y, both x products
                const double q0 = yr0[c], q1 = yr1[c];
                r0[0][U] = fma(fxr[0][c], q0, r0[0][U]);
                r1[0][U] = fma(fxr[0][c], q1, r1[0][U]);
                r0[1][U] = fma(fxr[1][c], q0, r0[1][U]);
                r1[1][U] = fma(fxr[1][c], q1, r1[1][U]);
            } else if constexpr (SH == 2) {  // both terms into one ring (alpha_t in F_x,t)
                const double2 q0 = reinterpret_cast<const double2 *>(yr0)[c];
                const double2 q1 = reinterpret_cast<const double2 *>(yr1)[c];
                r0[0][U] = fma(fxr[0][c], q0.x, r0[0][U]);
                r1[0][U] = fma(fxr[0][c], q1.x, r1[0][U]);
                r0[0][U] = fma(fxr[1][c], q0.y, r0[0][U]);
                r1[0][U] = fma(fxr[1][c], q1.y, r1[0][U]);
            } else if constexpr (T == 2) {
                const double2 q0 = reinterpret_cast<const double2 *>(yr0)[c];
                const double2 q1 = reinterpret_cast<const double2 *>(yr1)[c];
                r0[0][U] = fma(fxr[0][c], q0.x, r0[0][U]);
                r1[0][U] = fma(fxr[0][c], q1.x, r1[0][U]);
                r0[T - 1][U] = fma(fxr[T - 1][c], q0.y, r0[T - 1][U]);
                r1[T - 1][U] = fma(fxr[T - 1][c], q1.y, r1[T - 1][U]);
            } else {
                r0[0][U] = fma(fxr[0][c], yr0[c], r0[0][U]);
                r1[0][U] = fma(fxr[0][c], yr1[c], r1[0][U]);
            }
        }
        const int k = kx - P;  // slots hold planes k - p .. k + p: plane k - p + c in slot (U + 1 + c) mod W
        if (k >= z0 && k < z1) {
            const double *fz = fzs + (k - z0) * W * TZ;
            double fzr[TZ][W];
#pragma unroll
            for (int c = 0; c < W; ++c) {
                if constexpr (TZ == 2) {
                    const double2 f = reinterpret_cast<const double2 *>(fz)[c];
                    fzr[0][c] = f.x;
                    fzr[1][c] = f.y;
                } else {
                    fzr[0][c] = fz[c];
                }
            }
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int t = 0; t < TZ; ++t)
#pragma unroll
                for (int c = 0; c < W; ++c) {
                    a0 = fma(fzr[t][c], r0[t][(U + 1 + c) % W], a0);
                    a1 = fma(fzr[t][c], r1[t][(U + 1 + c) % W], a1);
                }
            double *o = out + (long)k * sz + oxy;
            const double w0 = beta == 0.0 ? a0 : fma(beta, ob0, a0);
            const double w1 = beta == 0.0 ? a1 : fma(beta, ob1, a1);
            prefetch(k + 1);
            if (own0) o[0] = w0;
            if (own1) o[sy] = w1;
        }
    };
    int u = ((kk0 - 1) % W + W) % W;  // slot of plane kk0 + ii - 1
    for (int ii = 0; ii <= npl; ++ii, u = u + 1 == W ? 0 : u + 1) {
        switch (u) {
#define ADS_KRC(V)                                                                     \
    case V:                                                                            \
        if constexpr (V < W) plane(ii, std::integral_constant<int, V>{});              \
        break;
            ADS_KRC(0) ADS_KRC(1) ADS_KRC(2) ADS_KRC(3) ADS_KRC(4) ADS_KRC(5)
            ADS_KRC(6) ADS_KRC(7) ADS_KRC(8) ADS_KRC(9) ADS_KRC(10)
#undef ADS_KRC
        }
    }
}

// single triples fit 3 CTAs per SM without spills up to p = 3 (measured 8 % faster at c5@512);
// pairs spill at 80 registers and keep 2
template <int P, int T, int SH>
__global__ void __launch_bounds__(KR_THREADS, (T == 1 && P <= 3) ? 3 : 2) kron3_kernel(const double *__restrict__ in, double *__restrict__ out,
                                                               const KronTerms k3, double beta, Geom g, int zlen) {
    pdl_launch_dependents();
    const int y0 = blockIdx.y * KR_Y;
    bool yt = true;
#pragma unroll
    for (int t = 0; t < T; ++t) yt = yt && y0 >= k3.fylo[t] && y0 + KR_Y - 1 <= k3.fyhi[t];
    if (yt) kron3_tile<P, T, true, SH>(in, out, k3, beta, g, zlen);
    else kron3_tile<P, T, false, SH>(in, out, k3, beta, g, zlen);
}

// launch with programmatic stream serialisation when `pdl` (the kernel calls pdl_wait before
// touching the fields); ADS_PDL=0 launches plainly (experiment switch).  Used for the elastic step
// (c5: 793 -> 771 us/step); the P-wave steps measured 1-5 % slower with it and launch plainly.
static bool pdl_on() {
    static const bool on = [] {
        const char *e = std::getenv("ADS_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
template <class... KArgs, class... Args>
static void launch_pdl(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl && pdl_on() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

template <int P, int T, int SH = 0>
static int kron3_launch(const double *in, double *out, const KronTerms &k3, double beta, const Geom &g,
                        cudaStream_t s) {
    using G = KronGeo<P, T>;
    const size_t sm = sizeof(double) * G::SMEM;
    const LaunchFacts lf = launch_facts((const void *)kron3_kernel<P, T, SH>, KR_THREADS, sm);
    const int gx = (g.n0 + KR_X - 1) / KR_X, gy = (g.n1 + KR_Y - 1) / KR_Y;
    // z pieces by the fluid wave model of kop_launch (each piece reads 2p halo planes)
    const long resident = (long)lf.per_sm * lf.nsm, tiles = (long)gx * gy;
    int best = 1;
    double best_cost = 1e300;
    for (int nz = 1; nz <= 64; ++nz) {
        const int zl = (g.n2 + nz - 1) / nz;
        if (zl > KR_ZMAX) continue;  // the piece's Fz rows are staged in shared memory
        if (zl < 2 * P + 1 && nz > 1) break;
        const long ctas = tiles * ((g.n2 + zl - 1) / zl);
        const double cost = (ctas <= resident ? 1.0 : (double)ctas / resident + 0.5) * (zl + 2.0 * P);
        if (cost < best_cost * 0.999) { best_cost = cost; best = nz; }
    }
    static const int nz_env = [] {  // experiment override of the split
        const char *e = std::getenv("ADS_KRON_NZ");
        return e ? std::atoi(e) : 0;
    }();
    if (nz_env > 0) best = nz_env;
    const int zlen = (g.n2 + best - 1) / best;
    if (zlen > KR_ZMAX) return -1;
    dim3 grd(gx, gy, (g.n2 + zlen - 1) / zlen);
    launch_pdl(true, kron3_kernel<P, T, SH>, grd, dim3(KR_THREADS), sm, s, in, out, k3, beta, g, zlen);
    return 0;
}

template <int P>
static int kron3_dispatch(const double *in, double *out, const KronTerms &k3, double beta, const Geom &g,
                          cudaStream_t s) {
    if (k3.nterms == 1) return kron3_launch<P, 1>(in, out, k3, beta, g, s);
    if constexpr (P <= 3) {  // two terms in one pass (registers: two gather rings)
        static const bool share = [] {  // experiment switch (scripts/): ADS_KRON_SHARE=0 off
            const char *e = std::getenv("ADS_KRON_SHARE");
            return !(e && e[0] == '0');
        }();
        if (share && k3.fz[0] == k3.fz[1]) return kron3_launch<P, 2, 2>(in, out, k3, beta, g, s);
        if (share && k3.fy[0] == k3.fy[1]) return kron3_launch<P, 2, 1>(in, out, k3, beta, g, s);
        return kron3_launch<P, 2, 0>(in, out, k3, beta, g, s);
    } else {  // two passes, the second accumulating
        KronTerms a = k3, b = k3;
        a.nterms = b.nterms = 1;
        b.addend = nullptr;  // the second pass accumulates onto the first
        b.fx[0] = k3.fx[1], b.fy[0] = k3.fy[1], b.fz[0] = k3.fz[1], b.alpha[0] = k3.alpha[1];
        if (kron3_launch<P, 1>(in, out, a, beta, g, s)) return -1;
        return kron3_launch<P, 1>(in, out, b, 1.0, g, s);
    }
}

int launch_kron3(int p, const double *in, double *out, const KronTerms &k3, double beta, const Geom &g,
                 cudaStream_t s) {
    if (k3.nterms < 1 || k3.nterms > 2) return -1;
    switch (p) {
        case 1: return kron3_dispatch<1>(in, out, k3, beta, g, s);
        case 2: return kron3_dispatch<2>(in, out, k3, beta, g, s);
        case 3: return kron3_dispatch<3>(in, out, k3, beta, g, s);
        case 4: return kron3_dispatch<4>(in, out, k3, beta, g, s);
        case 5: return kron3_dispatch<5>(in, out, k3, beta, g, s);
        default: return -1;
    }
}

// ------------------------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------------------------
// out = alpha (A along axis d) in + beta out  (beta == 0: out is not read).  One thread per
// output: x from the block's x range, j = blockIdx.y, k = blockIdx.z (no index division).  Along
// z the band row of local plane k is global row k + zoff and input planes [zv0, zv1) exist (slab
// halos).  Interior outputs (all 2P+1 taps inside) skip the per-tap bounds checks.
template <int P, int D>
__global__ void __launch_bounds__(128) axis_apply_kernel(const double *__restrict__ band, const double *__restrict__ in,
                                                         double *__restrict__ out, Geom g, double alpha, double beta,
                                                         int zoff, int zv0, int zv1) {
    constexpr int W = 2 * P + 1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
    if (i >= g.n0) return;
    const int r = D == 0 ? i : D == 1 ? j : k;
    const int lo = D == 2 ? zv0 : 0, hi = D == 0 ? g.n0 : D == 1 ? g.n1 : zv1;
    const long st = D == 0 ? 1 : D == 1 ? g.sy : g.sz;
    const long idx = (long)k * g.sz + (long)j * g.sy + i;
    const double *brow = band + (long)(r + (D == 2 ? zoff : 0)) * W;
    const double *src = in + idx - (long)P * st;
    double acc = 0.0;
    if (r - P >= lo && r + P < hi) {
#pragma unroll
        for (int c = 0; c < W; ++c) acc = fma(__ldg(brow + c), src[(long)c * st], acc);
    } else {
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const int col = r - P + c;
            if (col >= lo && col < hi) acc = fma(__ldg(brow + c), src[(long)c * st], acc);
        }
    }
    out[idx] = beta == 0.0 ? alpha * acc : fma(alpha, acc, beta * out[idx]);
}

__global__ void axpby_kernel(long N, double alpha, const double *__restrict__ x, double beta, double *__restrict__ y) {
    pdl_launch_dependents();
    pdl_wait();
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x)
        y[q] = alpha * x[q] + beta * y[q];
}

// u_c = sum over the terms t of component c of amp_t sx_t[i] sy_t[j] sz_t[k + zoff], zero on the
// Dirichlet faces (mx, my: x / y faces; ngz > 0: the global z faces 0 and ngz - 1): one write pass
// for all terms and components.  f: per term [amp, comp, sx (n0), sy (n1), sz (nzf)]
// sum of separable terms amp_m fx_m(i) fy_m(j) fz_m(k) into component c_m (zero on the masked
// faces): block per (j, k) line, the term weights amp fy fz of the line staged in shared memory in
// chunks of 256 terms, threads along x
constexpr int SEP_THREADS = 128, SEP_CHUNK = 256;
__global__ void __launch_bounds__(SEP_THREADS) set_separable_kernel(double *u, long cstride, int nterms,
                                                                    const double *__restrict__ f, int n0f, int n1f,
                                                                    int nzf, Geom g, int zoff, int mx, int my, int ngz,
                                                                    int ncomp) {
    __shared__ double wt[SEP_CHUNK];
    __shared__ int cm[SEP_CHUNK];
    const int j = blockIdx.y, k = blockIdx.z, kg = k + zoff;
    const long tl = 2 + n0f + n1f + nzf;
    const bool line0 = (my && (j == 0 || j == g.n1 - 1)) || (ngz > 0 && (kg == 0 || kg == ngz - 1));
    for (int i0 = blockIdx.x * SEP_THREADS; i0 < g.n0; i0 += gridDim.x * SEP_THREADS) {
        const int i = i0 + threadIdx.x;
        double acc[3] = {0.0, 0.0, 0.0};
        for (int m0 = 0; m0 < nterms && !line0; m0 += SEP_CHUNK) {
            const int nm = min(SEP_CHUNK, nterms - m0);
            __syncthreads();
            for (int t = threadIdx.x; t < nm; t += SEP_THREADS) {
                const double *ft = f + (m0 + t) * tl;
                wt[t] = ft[0] * ft[2 + n0f + j] * ft[2 + n0f + n1f + kg];
                cm[t] = (int)ft[1];
            }
            __syncthreads();
            if (i < g.n0)
                for (int t = 0; t < nm; ++t) {
                    const double fx = __ldg(f + (m0 + t) * tl + 2 + i);
                    const int c = cm[t];
                    if (c == 0) acc[0] = fma(wt[t], fx, acc[0]);
                    else if (c == 1) acc[1] = fma(wt[t], fx, acc[1]);
                    else acc[2] = fma(wt[t], fx, acc[2]);
                }
        }
        if (i < g.n0) {
            const bool z0 = mx && (i == 0 || i == g.n0 - 1);
            const long o = (long)k * g.sz + (long)j * g.sy + i;
            for (int c = 0; c < ncomp; ++c) u[c * cstride + o] = z0 ? 0.0 : acc[c];
        }
    }
}

__global__ void drift_kernel(const double *__restrict__ U, const double *__restrict__ V, double tau,
                             double *__restrict__ P, long N) {
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x)
        P[q] = fma(tau, V[q], U[q]);
}

__global__ void mask_boundary_kernel(double *u, Geom g, int zoff, int ngz) {
    long N = (long)g.n0 * g.n1 * g.n2;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x) {
        int i = q % g.n0;
        long t = q / g.n0;
        int j = t % g.n1;
        int k = t / g.n1;
        const int kg = k + zoff;  // global plane
        if (i == 0 || j == 0 || i == g.n0 - 1 || j == g.n1 - 1 || (ngz > 0 && (kg == 0 || kg == ngz - 1)))
            u[(long)k * g.sz + (long)j * g.sy + i] = 0.0;
    }
}

// deterministic two-stage dot product (fixed grid, fixed tree)
constexpr int DOT_BLOCKS = 1024, DOT_THREADS = 256;
__global__ void dot_partial_kernel(long N, const double *__restrict__ x, const double *__restrict__ y,
                                   double *partial) {
    __shared__ double sh[DOT_THREADS];
    double s = 0.0;
    for (long q = blockIdx.x * (long)DOT_THREADS + threadIdx.x; q < N; q += (long)DOT_BLOCKS * DOT_THREADS)
        s = fma(x[q], y[q], s);
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = DOT_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}
__global__ void dot_final_kernel(const double *partial, double *res) {
    __shared__ double sh[DOT_BLOCKS];
    for (int q = threadIdx.x; q < DOT_BLOCKS; q += blockDim.x) sh[q] = partial[q];
    __syncthreads();
    for (int w = DOT_BLOCKS / 2; w > 0; w >>= 1) {
        for (int q = threadIdx.x; q < w; q += blockDim.x) sh[q] += sh[q + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *res = sh[0];
}

// ------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------

static int grid_for(long N) {
    long b = (N + 255) / 256;
    return (int)(b < 148 * 32 ? (b < 1 ? 1 : b) : 148 * 32);
}

static int encode_field_map(CUtensorMap *m, const double *base, const Geom &g, unsigned b0, unsigned b1,
                            unsigned b2);

// z split: CTAs are scheduled dynamically, so the time is about (CTAs per resident slot + 1/2 for
// the tail) x (planes per CTA incl. 2p halo planes); this fit the measured v3 kop times at 515^3
// for 1..12 pieces within 3 % (1.69 ms unsplit, 1.49 ms at 4 pieces).  A split that fits one wave
// has no tail (c5, 130^3: 6 pieces in one wave beat 10 in 1.5 waves, 1.22 -> 1.04 ms per step)
static int kop_pieces(int n2, int P, long tiles, long resident, double halo) {
    int best = 1;
    double best_cost = 1e300;
    for (int nz = 1; nz <= 32; ++nz) {
        const int zl = (n2 + nz - 1) / nz;
        if (zl < 2 * P + 1 && nz > 1) break;
        const long ctas = tiles * ((n2 + zl - 1) / zl);
        // one wave: no tail; several: the fluid model's mean tail of half a piece
        const double cost = (ctas <= resident ? 1.0 : (double)ctas / resident + 0.5) * (zl + halo);
        if (cost < best_cost * 0.999) {
            best_cost = cost;
            best = nz;
        }
    }
    static const int nz_env = [] {  // experiment override of the split (scripts/kop_nz.py)
        const char *e = std::getenv("ADS_KOP_NZ");
        return e ? std::atoi(e) : 0;
    }();
    return nz_env > 0 ? nz_env : best;
}

template <int P>
static int kop_launch(const KopArgs &a, cudaStream_t s) {
    KopArgs b = a;
    if (b.zv1 < b.zv0) {  // no halo planes: exactly the output planes exist
        b.zv0 = 0;
        b.zv1 = a.geo.n2;
    }
    using G = K4Geo<P>;
    const size_t sm = sizeof(double) * G::SMEM;
    const LaunchFacts lf = launch_facts((const void *)kop4_kernel<P>, K4_THREADS, sm);
    const int ox = kop_origin(a.ilo[0], a.ihi[0], K4_X), oy = kop_origin(a.ilo[1], a.ihi[1], K4_Y);
    const int gx = (a.geo.n0 - ox + K4_X - 1) / K4_X, gy = (a.geo.n1 - oy + K4_Y - 1) / K4_Y;
    const int nz = kop_pieces(a.geo.n2, P, (long)gx * gy, (long)lf.per_sm * lf.nsm, 2.0 * P);
    b.zlen = a.zlen > 0 ? a.zlen : (a.geo.n2 + nz - 1) / nz;
    // U and V over the planes that exist in memory, [zv0, zv1) (slabs: halo planes included)
    Geom gm = a.geo;
    gm.n2 = b.zv1 - b.zv0;
    const double *ub = a.U + (long)b.zv0 * a.geo.sz, *vb = (a.V ? a.V : a.U) + (long)b.zv0 * a.geo.sz;
    if (!a.V) b.tau = 0.0;
    CUtensorMap tmu, tmv, tmp;
    const double *pb = a.Ph ? a.Ph + (long)b.zv0 * a.geo.sz : ub;
    if (encode_field_map(&tmu, ub, gm, G::HXE, G::HY, 1) || encode_field_map(&tmv, vb, gm, G::HXE, G::HY, 1) ||
        encode_field_map(&tmp, pb, gm, G::HXE, G::HY, 1))
        return -2;
    dim3 grd(gx, gy, (a.geo.n2 + b.zlen - 1) / b.zlen);
    launch_pdl(a.pdl, kop4_kernel<P>, grd, dim3(K4_THREADS), sm, s, b, tmu, tmv, tmp);
    return 0;
}

int launch_kop(int p, const KopArgs &a, cudaStream_t s) {
    switch (p) {
        case 1: return kop_launch<1>(a, s);
        case 2: return kop_launch<2>(a, s);
        case 3: return kop_launch<3>(a, s);
        case 4: return kop_launch<4>(a, s);
        case 5: return kop_launch<5>(a, s);
        default: return -1;
    }
}

// ---- TMA descriptors (driver entry point through the runtime: no -lcuda) ----
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// general 3D fp64 map: dims (d0, d1, d2) elements, strides (s1, s2) in elements, box (b0, b1, b2);
// out-of-bounds boxes are zero-filled (modal_tc.cu)
int encode_map_3d(CUtensorMap *m, const double *base, long d0, long d1, long d2, long s1, long s2, unsigned b0,
                  unsigned b1, unsigned b2) {
    auto enc = tmap_encoder();
    if (!enc) return -1;
    const cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
    const cuuint64_t strides[2] = {(cuuint64_t)s1 * 8, (cuuint64_t)s2 * 8};
    const cuuint32_t box[3] = {b0, b1, b2}, es[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -1;
}

// 3D fp64 field (n0, n1, n2) with strides (sy, sz) elements, box (b0, b1, b2); OOB -> 0
static int encode_field_map(CUtensorMap *m, const double *base, const Geom &g, unsigned b0, unsigned b1,
                            unsigned b2) {
    auto enc = tmap_encoder();
    if (!enc) return -1;
    const cuuint64_t dims[3] = {(cuuint64_t)g.n0, (cuuint64_t)g.n1, (cuuint64_t)g.n2};
    const cuuint64_t strides[2] = {(cuuint64_t)g.sy * 8, (cuuint64_t)g.sz * 8};
    const cuuint32_t box[3] = {b0, b1, b2}, es[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -1;
}

template <int P, int L, bool X, int C>
static int sweep_launch(const SweepArgs &a, cudaStream_t s) {
    constexpr int LW = (X || L > 17 || C > 32) ? 8 : 16;  // y/z: 16-line tiles while the buffers fit
    constexpr int NT = SW<LW, C>::THREADS;
    const Geom &g = a.geo;
    // y/z: a second output / V buffer when it fits the 227 KB of shared memory per CTA
    const int vbufs = (!X && sizeof(double) * sweep_smem_doubles<P, LW>(a.t, X, a.geo.sy, a.mode != 0, 2) <= 227 * 1024)
                          ? 2 : 1;
    const size_t sm = sizeof(double) * (size_t)sweep_smem_doubles<P, LW>(a.t, X, a.geo.sy, a.mode != 0, vbufs);
    if (sm > (size_t)kMaxSmemPerCta) return -1;
    const LaunchFacts lf = launch_facts((const void *)sweep_kernel<P, L, X, LW, C>, NT, sm);
    long ntiles;
    if (X) ntiles = ((long)g.n1 * g.n2 + LW - 1) / LW;
    else ntiles = (long)((g.n0 + LW - 1) / LW) * (a.dir == 1 ? g.n2 : g.n1);
    const long cap = (long)lf.per_sm * lf.nsm;
    dim3 grd((unsigned)std::min(ntiles, cap));
    SweepArgs b = a;
    b.vbufs = vbufs;
    if (X) {
        // 2D view: n0 columns x (n1 n2) lines of pitch sy
        b.nbox = xbox_count(a.t.n);
        b.rb = xbox_cols(a.t.n);
        Geom g2 = g;
        g2.n1 = g.n1 * g.n2;
        g2.n2 = 1;
        if (encode_field_map(&b.tm_in, a.in, g2, (unsigned)b.rb, LW, 1) ||
            encode_field_map(&b.tm_out, a.out, g2, (unsigned)b.rb, LW, 1))
            return -2;
    } else {
        // boxes of LW lines x rb rows: the C L rows in nbox = 4 boxes, 8 when C L > 1024 (rb <= 256)
        b.nbox = (L > 32 || C * L > 1024) ? 8 : 4;
        b.rb = C * L / b.nbox;
        const unsigned rb = (unsigned)b.rb;
        const bool y = a.dir == 1;
        if (encode_field_map(&b.tm_in, a.in, g, LW, y ? rb : 1, y ? 1 : rb) ||
            (a.mode && encode_field_map(&b.tm_v, a.V, g, LW, y ? rb : 1, y ? 1 : rb)) ||
            (!a.mode && encode_field_map(&b.tm_out, a.out, g, LW, y ? rb : 1, y ? 1 : rb)))
            return -2;  // TMA descriptor could not be encoded
    }
    launch_pdl(a.pdl, sweep_kernel<P, L, X, LW, C>, grd, dim3(NT), sm, s, b);
    return 0;
}

template <int P, int LV>
static int sweep_launch_L(const SweepArgs &a, cudaStream_t s) {
    if constexpr (LV < P) {
        return -1;  // a chunk must hold a whole boundary state
    } else {
        if constexpr (LV <= 17) {  // 16 or 64 chunks of at most 17 rows (make_solve_tab)
            if (a.t.C == 16)
                return a.dir == 0 ? sweep_launch<P, LV, true, 16>(a, s) : sweep_launch<P, LV, false, 16>(a, s);
            if (a.t.C == 64)
                return a.dir == 0 ? sweep_launch<P, LV, true, 64>(a, s) : sweep_launch<P, LV, false, 64>(a, s);
        }
        if (a.t.C != kSweepChunks) return -1;
        return a.dir == 0 ? sweep_launch<P, LV, true, kSweepChunks>(a, s)
                          : sweep_launch<P, LV, false, kSweepChunks>(a, s);
    }
}

template <int P>
static int sweep_dispatch(const SweepArgs &a, cudaStream_t s) {
    if (a.dir == 0 && a.mode != 0) return -1;  // the kick is fused into y/z sweeps only
    if (a.dir == 0 && (a.geo.sy % 2 != 0 || a.geo.sz != a.geo.sy * a.geo.n1)) return -1;  // even pitch, packed planes
    switch (a.t.L) {
        case 1: return sweep_launch_L<P, 1>(a, s);
        case 3: return sweep_launch_L<P, 3>(a, s);
        case 5: return sweep_launch_L<P, 5>(a, s);
        case 9: return sweep_launch_L<P, 9>(a, s);
        case 17: return sweep_launch_L<P, 17>(a, s);
        case 33: return sweep_launch_L<P, 33>(a, s);
    }
    return -1;
}

// sequential banded LU along one line per thread (PAPER.md:533-618 as printed): forward
// y_i = r_i - sum_k l_{i,k} y_{i-k} (far terms first: y_{i-1} enters last), y kept in `out`;
// backward x_i = y_i dinv_i - sum_k us_{i,k} x_{i+k}, out = x, V += kick x.  Threads of a block
// take adjacent x-lines (coalesced rows).  (Staging each block of lines in shared memory with one
// bulk copy per row measured slower: a whole line per thread caps residency at ~7 warps/SM.)
template <int P>
__global__ void __launch_bounds__(128, 8) line_sweep_kernel(const SweepArgs a) {
    const int x = blockIdx.x * 128 + threadIdx.x, w = blockIdx.y;
    if (a.dstep_inc && x == 0 && w == 0) *a.dstep_inc += 1;
    const Geom &g = a.geo;
    if (x >= g.n0) return;
    const long ls = a.dir == 2 ? g.sz : g.sy, ws = a.dir == 2 ? g.sy : g.sz;
    const int n = a.t.n;
    const double *in = a.in + w * ws + x;  // may alias out (in-place solves)
    double *out = a.out + w * ws + x;       // holds y between the passes
    double *__restrict__ vv = a.V ? a.V + w * ws + x : nullptr;
    const double *__restrict__ L = a.t.l, *__restrict__ U = a.t.us, *__restrict__ D = a.t.dinv;
    double h[P];
#pragma unroll
    for (int k = 0; k < P; ++k) h[k] = 0.0;  // h[k] = y_{i-1-k}
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
        double s = in[i * ls];
#pragma unroll
        for (int k = P - 1; k >= 0; --k) s = fma(-__ldg(L + i * P + k), h[k], s);
#pragma unroll
        for (int k = P - 1; k > 0; --k) h[k] = h[k - 1];
        h[0] = s;
        out[i * ls] = s;
    }
#pragma unroll
    for (int k = 0; k < P; ++k) h[k] = 0.0;  // h[k] = x_{i+1+k}
#pragma unroll 4
    for (int i = n - 1; i >= 0; --i) {
        double v = out[i * ls] * __ldg(D + i);
#pragma unroll
        for (int k = P - 1; k >= 0; --k) v = fma(-__ldg(U + i * P + k), h[k], v);
#pragma unroll
        for (int k = P - 1; k > 0; --k) h[k] = h[k - 1];
        h[0] = v;
        out[i * ls] = v;
        if (vv) vv[i * ls] = fma(a.kick, v, vv[i * ls]);
    }
}

int launch_line_sweep(int p, const SweepArgs &a, cudaStream_t s) {
    if (a.dir == 0 || a.t.n > kLineSweepMax || !a.out) return -1;
    dim3 grd((a.geo.n0 + 127) / 128, a.dir == 2 ? a.geo.n1 : a.geo.n2);
    switch (p) {
        case 1: line_sweep_kernel<1><<<grd, 128, 0, s>>>(a); break;
        case 2: line_sweep_kernel<2><<<grd, 128, 0, s>>>(a); break;
        case 3: line_sweep_kernel<3><<<grd, 128, 0, s>>>(a); break;
        case 4: line_sweep_kernel<4><<<grd, 128, 0, s>>>(a); break;
        case 5: line_sweep_kernel<5><<<grd, 128, 0, s>>>(a); break;
        default: return -1;
    }
    return 0;
}

int launch_sweep(int p, const SweepArgs &a, cudaStream_t s) {
    switch (p) {
        case 1: return sweep_dispatch<1>(a, s);
        case 2: return sweep_dispatch<2>(a, s);
        case 3: return sweep_dispatch<3>(a, s);
        case 4: return sweep_dispatch<4>(a, s);
        case 5: return sweep_dispatch<5>(a, s);
    }
    return -1;
}

int launch_axis_apply(int p, int d, const double *band, const double *in, double *out, const Geom &g, double alpha,
                      double beta, cudaStream_t s, int zoff, int zv0, int zv1) {
    if (zv1 < zv0) {
        zv0 = 0;
        zv1 = g.n2;
    }
    dim3 blk(128), grd((g.n0 + 127) / 128, g.n1, g.n2);
#define ADS_AX(PP, DD) axis_apply_kernel<PP, DD><<<grd, blk, 0, s>>>(band, in, out, g, alpha, beta, zoff, zv0, zv1)
#define ADS_AXP(PP)                          \
    case PP:                                 \
        if (d == 0) ADS_AX(PP, 0);           \
        else if (d == 1) ADS_AX(PP, 1);      \
        else ADS_AX(PP, 2);                  \
        break;
    switch (p) {
        ADS_AXP(1) ADS_AXP(2) ADS_AXP(3) ADS_AXP(4) ADS_AXP(5)
        default: return -1;
    }
#undef ADS_AXP
#undef ADS_AX
    return 0;
}

int launch_axpby(long N, double alpha, const double *x, double beta, double *y, cudaStream_t s, bool pdl) {
    launch_pdl(pdl, axpby_kernel, dim3(grid_for(N)), dim3(256), 0, s, N, alpha, x, beta, y);
    return 0;
}

void launch_set_separable(double *u, long cstride, int ncomp, int nterms, const double *f, int n0f, int n1f, int nzf,
                          const Geom &g, int zoff, int mx, int my, int ngz, cudaStream_t s) {
    const dim3 grid((g.n0 + SEP_THREADS - 1) / SEP_THREADS, g.n1, g.n2);
    set_separable_kernel<<<grid, SEP_THREADS, 0, s>>>(u, cstride, nterms, f, n0f, n1f, nzf, g, zoff, mx, my, ngz, ncomp);
}

// thread per (x, row, plane); the row's y block found by a scan of the (few) block starts
__global__ void __launch_bounds__(256) kick_a2a_kernel(const KickA2AArgs a) {
    const int i = blockIdx.x * 64 + (threadIdx.x & 63), j = blockIdx.y * 4 + (threadIdx.x >> 6), k = blockIdx.z;
    const Geom &g = a.geo;
    if (i >= g.n0 || j >= g.n1) return;
    int q = 0;
    while (q + 1 < a.nq && j >= a.py0[q + 1]) ++q;
    const int r0 = a.py0[q], nr = a.py0[q + 1] - r0;
    const double v = a.arecv[(long)g.n2 * r0 * g.sy + ((long)k * nr + (j - r0)) * g.sy + i];
    const long o = (long)k * g.sz + (long)j * g.sy + i;
    a.V[o] = fma(a.kick, v, a.V[o]);
    if (a.A) a.A[o] = v;
}

int launch_kick_a2a(const KickA2AArgs &a, cudaStream_t s) {
    if (a.nq < 1 || a.nq > kMaxA2A) return -1;
    dim3 grd((a.geo.n0 + 63) / 64, (a.geo.n1 + 3) / 4, a.geo.n2);
    kick_a2a_kernel<<<grd, 256, 0, s>>>(a);
    return 0;
}

void launch_drift(const double *U, const double *V, double tau, double *P, long N, cudaStream_t s) {
    drift_kernel<<<grid_for(N), 256, 0, s>>>(U, V, tau, P, N);
}

int launch_mask_boundary(double *u, const Geom &g, cudaStream_t s, int zoff, int ngz) {
    mask_boundary_kernel<<<grid_for((long)g.n0 * g.n1 * g.n2), 256, 0, s>>>(u, g, zoff, ngz < 0 ? g.n2 : ngz);
    return 0;
}

int launch_dot(long N, const double *x, const double *y, double *partial, double *res, cudaStream_t s) {
    dot_partial_kernel<<<DOT_BLOCKS, DOT_THREADS, 0, s>>>(N, x, y, partial);
    dot_final_kernel<<<1, 256, 0, s>>>(partial, res);
    return 0;
}

// ------------------------------------------------------------------------------------------
// modal propagation (see kernels.cuh launch_modal): thread per mode, 8 + 8 B in / 24 B out
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128) modal_kernel(double *__restrict__ cU, double *__restrict__ cV,
                                                    double *__restrict__ ca, const double *__restrict__ lx,
                                                    const double *__restrict__ ly, const double *__restrict__ lz,
                                                    const double *__restrict__ fx, const double *__restrict__ fy,
                                                    const double *__restrict__ fz, const double *__restrict__ g,
                                                    long nsteps, double tau, Geom geo) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y, k = blockIdx.z;
    if (i >= geo.n0) return;
    const long o = (long)k * geo.sz + (long)j * geo.sy + i;
    const double eta = 0.25 * tau * tau;
    const double li = lx[i], lj = ly[j], lk = lz[k];
    const double L = li + lj + lk;
    const double delta = (1.0 + eta * li) * (1.0 + eta * lj) * (1.0 + eta * lk);
    double u = cU[o], v = cV[o], a;
    if (!g) {
        const double Ld = L / delta;
        double a11 = 1.0, a12 = tau, a21 = -tau * Ld, a22 = 1.0 - tau * tau * Ld;
        double r11 = 1.0, r12 = 0.0, r21 = 0.0, r22 = 1.0;
        for (long m = nsteps; m;) {
            if (m & 1) {
                const double t11 = r11 * a11 + r12 * a21, t12 = r11 * a12 + r12 * a22;
                const double t21 = r21 * a11 + r22 * a21, t22 = r21 * a12 + r22 * a22;
                r11 = t11, r12 = t12, r21 = t21, r22 = t22;
            }
            m >>= 1;
            if (m) {
                const double t11 = a11 * a11 + a12 * a21, t12 = a11 * a12 + a12 * a22;
                const double t21 = a21 * a11 + a22 * a21, t22 = a21 * a12 + a22 * a22;
                a11 = t11, a12 = t12, a21 = t21, a22 = t22;
            }
        }
        const double un = r11 * u + r12 * v, vn = r21 * u + r22 * v;
        u = un;
        v = vn;
        a = -Ld * u;
    } else {
        const double F = fx[i] * fy[j] * fz[k];
        a = ca[o];
        for (long s = 0; s < nsteps; ++s) {
            const double P = u + tau * v;
            a = (__ldg(g + s) * F - L * P) / delta;
            v = v + tau * a;
            u = P;
        }
    }
    cU[o] = u;
    cV[o] = v;
    ca[o] = a;
}

int launch_modal(double *cU, double *cV, double *ca, const double *lx, const double *ly, const double *lz,
                 const double *fx, const double *fy, const double *fz, const double *g, long nsteps, double tau,
                 const Geom &geo, cudaStream_t s) {
    if (geo.n1 > 65535 || geo.n2 > 65535) return -1;
    dim3 grd((geo.n0 + 127) / 128, geo.n1, geo.n2);
    modal_kernel<<<grd, 128, 0, s>>>(cU, cV, ca, lx, ly, lz, fx, fy, fz, g, nsteps, tau, geo);
    return 0;
}

__global__ void set_long_kernel(long *dst, long value) { *dst = value; }

void launch_set_long(long *dst, long value, cudaStream_t s) { set_long_kernel<<<1, 1, 0, s>>>(dst, value); }

__global__ void line1_kernel(const double *__restrict__ in, double *__restrict__ out, double *__restrict__ V,
                             double scale, double kick, long *inc, Geom g) {
    const long N = (long)g.n0 * g.n1 * g.n2;
    if (inc && blockIdx.x == 0 && threadIdx.x == 0) *inc += 1;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x) {
        const int i = (int)(q % g.n0);
        const long t = q / g.n0;
        const long o = (t / g.n1) * g.sz + (t % g.n1) * g.sy + i;
        const double x = scale * in[o];
        if (V) V[o] = fma(kick, x, V[o]);
        if (out) out[o] = x;
    }
}

void launch_line1(const double *in, double *out, double *V, double scale, double kick, long *inc, const Geom &g,
                  cudaStream_t s) {
    line1_kernel<<<grid_for((long)g.n0 * g.n1 * g.n2), 256, 0, s>>>(in, out, V, scale, kick, inc, g);
}

__global__ void repack_kernel(const double *__restrict__ src, double *__restrict__ dst, Geom g, int to_pitched) {
    const long N = (long)g.n0 * g.n1 * g.n2;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x) {
        const int i = (int)(q % g.n0);
        const long t = q / g.n0;
        const long o = (t / g.n1) * g.sz + (t % g.n1) * g.sy + i;
        if (to_pitched) dst[o] = src[q];
        else dst[q] = src[o];
    }
}

void launch_repack(const double *src, double *dst, const Geom &g, int to_pitched, cudaStream_t s) {
    repack_kernel<<<grid_for((long)g.n0 * g.n1 * g.n2), 256, 0, s>>>(src, dst, g, to_pitched);
}

}  // namespace ads

