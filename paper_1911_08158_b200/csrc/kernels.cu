// kernels.cu -- sm_100a fp64 kernels of the ADS wave step (arXiv:1911.08158).
//
//   kop_kernel   : drift P = U + tau V, source, and the sum-factorised
//                  Kronecker operator K P (Eq. 14, 3D) in ONE
//                  pass: a 32x8 (x,y) tile marches along z; per plane the x- and
//                  y-passes run from shared memory and the z-pass from a
//                  register ring of 2p+1 planes.  HBM: reads U, V; writes P, r.
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
#include <algorithm>
#include <cstdio>

#include "kernels.cuh"

namespace ads {

// ------------------------------------------------------------------------------------------
// fused drift + source + K-apply
//
// Tile: 32 (x) x 8 (y) outputs per CTA, marching along z.  Per input plane kk:
//   commit  P(kk) = U + tau V  -> shared tile (haloed by p in x and y) [+ HBM for owned points]
//   y-pass  Y1 = My P, Y2 = Ky P          on the 8 owned rows, 32+2p columns
//   x-pass  S  = Kx Y1 + Mx Y2, T = Mx Y1 on the 32x8 owned points -> register ring slot
//   z-pass  K P(k) = Mz S + Kz T over the ring (k = kk - p), + source -> r
// (K = Kx My Mz + Mx Ky Mz + Mx My Kz; 1D factors along different axes commute.)
// The ring of 2p+1 planes is rotated by unrolling the plane loop 2p+1 times.
// ------------------------------------------------------------------------------------------
template <int P>
struct KopSmem {
    static constexpr int TX = 32, TY = 8, W = 2 * P + 1, HX = TX + 2 * P, HY = TY + 2 * P;
    double Ps[HY][HX];
    double Y1[TY][HX], Y2[TY][HX];
    double zc[2][2][W];  // [parity][Mz|Kz][c] rows of the output plane
};

template <int P>
__global__ void __launch_bounds__(256, 2) kop_kernel(const KopArgs a) {
    using S_ = KopSmem<P>;
    constexpr int TX = S_::TX, TY = S_::TY, W = S_::W, HX = S_::HX, HY = S_::HY;
    __shared__ S_ sm;

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int n0 = a.geo.n0, n1 = a.geo.n1, n2 = a.geo.n2;
    const long sy = a.geo.sy, sz = a.geo.sz;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int z0 = blockIdx.z * a.zlen, z1 = min(n2, z0 + a.zlen);
    const int gx = x0 + tx, gy = y0 + ty;
    const bool own = gx < n0 && gy < n1;

    // band rows of this thread's x (Mx, Kx) and y (My, Ky)
    double mx[W], kx[W], my[W], ky[W];
#pragma unroll
    for (int c = 0; c < W; ++c) {
        mx[c] = gx < n0 ? __ldg(a.mx + (long)gx * W + c) : 0.0;
        kx[c] = gx < n0 ? __ldg(a.kx + (long)gx * W + c) : 0.0;
        my[c] = gy < n1 ? __ldg(a.my + (long)gy * W + c) : 0.0;
        ky[c] = gy < n1 ? __ldg(a.ky + (long)gy * W + c) : 0.0;
    }
    const double sxy = (a.bx && own) ? __ldg(a.bx + gx) * __ldg(a.by + gy) : 0.0;

    // load slots: haloed (ry, rx) = (ty + 8 sr, tx + 32 sc)
    constexpr int NSR = (HY + TY - 1) / TY, NS = 2 * NSR;
    bool sv[NS];
    long soff[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        const int ry = ty + TY * (q >> 1), rx = tx + TX * (q & 1);
        const int X = x0 - P + rx, Y = y0 - P + ry;
        sv[q] = ry < HY && rx < HX && X >= 0 && X < n0 && Y >= 0 && Y < n1;
        soff[q] = (long)Y * sy + X;
    }
    double pu[NS], pv[NS];
    auto load = [&](int kin) {
        const bool kv = kin >= 0 && kin < n2;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            pu[q] = 0.0;
            pv[q] = 0.0;
            if (sv[q] && kv) {
                pu[q] = __ldg(a.U + (long)kin * sz + soff[q]);
                pv[q] = __ldg(a.V + (long)kin * sz + soff[q]);
            }
        }
    };

    double Sr[W], Tr[W];
#pragma unroll
    for (int c = 0; c < W; ++c) Sr[c] = Tr[c] = 0.0;

    const int tid = ty * TX + tx;
    load(z0 - P);
    for (int kb = z0 - P; kb < z1 + P; kb += W) {
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const int kk = kb + u;
            if (kk < z1 + P) {
                const int k = kk - P;  // output plane
                // commit plane kk
#pragma unroll
                for (int q = 0; q < NS; ++q) {
                    const int ry = ty + TY * (q >> 1), rx = tx + TX * (q & 1);
                    if (ry < HY && rx < HX) {
                        const double pp = fma(a.tau, pv[q], pu[q]);
                        sm.Ps[ry][rx] = pp;
                        if (a.Pout && sv[q] && kk >= z0 && kk < z1 && ry >= P && rx >= P && rx < P + TX &&
                            ry < P + TY)
                            a.Pout[(long)kk * sz + soff[q]] = pp;
                    }
                }
                if (tid < 2 * W && k >= z0) {
                    const double *src = (tid < W ? a.mz : a.kz) + (long)k * W + (tid < W ? tid : tid - W);
                    sm.zc[kk & 1][tid < W ? 0 : 1][tid < W ? tid : tid - W] = __ldg(src);
                }
                __syncthreads();
                if (kk + 1 < z1 + P) load(kk + 1);  // in flight during the passes below

                // y-pass on owned rows, all haloed columns
#pragma unroll
                for (int cs = 0; cs < 2; ++cs) {
                    const int col = tx + TX * cs;
                    if (col < HX) {
                        double y1 = 0.0, y2 = 0.0;
#pragma unroll
                        for (int c = 0; c < W; ++c) {
                            const double v = sm.Ps[ty + c][col];
                            y1 = fma(my[c], v, y1);
                            y2 = fma(ky[c], v, y2);
                        }
                        sm.Y1[ty][col] = y1;
                        sm.Y2[ty][col] = y2;
                    }
                }
                __syncthreads();
                // x-pass on owned points
                double s = 0.0, t = 0.0;
#pragma unroll
                for (int c = 0; c < W; ++c) {
                    const double y1 = sm.Y1[ty][tx + c], y2 = sm.Y2[ty][tx + c];
                    s = fma(kx[c], y1, s);
                    s = fma(mx[c], y2, s);
                    t = fma(mx[c], y1, t);
                }
                Sr[u] = s;
                Tr[u] = t;
                // z-pass: plane k-p+c sits in ring slot (u + 1 + c) mod W
                if (k >= z0 && own) {
                    double acc = 0.0;
#pragma unroll
                    for (int c = 0; c < W; ++c) {
                        const int slot = (u + 1 + c) % W;
                        acc = fma(sm.zc[kk & 1][0][c], Sr[slot], acc);
                        acc = fma(sm.zc[kk & 1][1][c], Tr[slot], acc);
                    }
                    const double src = (a.bx) ? a.g * sxy * __ldg(a.bz + k) : 0.0;
                    a.r[(long)k * sz + (long)gy * sy + gx] = fma(a.sign, acc, src);
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// partitioned banded sweeps
//
// A CTA owns a tile of XW = 8 adjacent lines; warp w solves line w, lane c owns
// chunk c (rows [cL, cL+L), L odd, C <= 32 chunks; lines are padded to C*L rows
// with identity rows).  Per lane, four p-term recurrences over its chunk held in
// registers:
//   1. forward  y_i = r_i - sum_k l_{i,k} y_{i-k}                 zero incoming state -> tail
//   2. forward                                                    exact incoming state
//   3. backward x_i = y_i/u_ii - sum_k (u_{i,i+k}/u_ii) x_{i+k}    zero incoming state -> head
//   4. backward                                                   exact incoming state
// The exact incoming states come from a Kogge-Stone scan of the affine chunk
// maps across the lanes (shuffles; Phi = products of chunk transfer matrices,
// host-precomputed).  No block barrier inside the solve.
// The tile moves HBM <-> shared memory with coalesced cooperative loads/stores;
// y/z tiles are stored [row][XW+1] (odd pitch) and x tiles [line][n], so the
// lane-per-chunk reads (stride L, odd) are bank-conflict-free.
// Rows [i_lo, i_hi) of the factors are one constant row held in registers;
// the other ("edge") rows are read from a shared-memory table.
// ------------------------------------------------------------------------------------------
constexpr int XW = 8;        // lines per CTA
constexpr int YP = XW + 1;   // y/z tile row pitch (doubles)
constexpr int SWEEP_THREADS = 32 * XW;

template <int P, bool FWD>
__device__ __forceinline__ void warp_scan(double (&o)[P], double (&inc)[P], const double *phi, int C, int levels,
                                          int lane) {
    for (int lv = 0; lv < levels; ++lv) {
        const int d = 1 << lv;
        double u[P];
#pragma unroll
        for (int m = 0; m < P; ++m)
            u[m] = FWD ? __shfl_up_sync(0xffffffffu, o[m], d) : __shfl_down_sync(0xffffffffu, o[m], d);
        const bool has = FWD ? (lane >= d && lane < C) : (lane + d < C);
        if (has) {
            const double *ph = phi + (lv * C + lane) * P * P;
            double t[P];
#pragma unroll
            for (int i = 0; i < P; ++i) {
                double s = o[i];
#pragma unroll
                for (int j = 0; j < P; ++j) s = fma(ph[i * P + j], u[j], s);
                t[i] = s;
            }
#pragma unroll
            for (int i = 0; i < P; ++i) o[i] = t[i];
        }
    }
#pragma unroll
    for (int m = 0; m < P; ++m) {
        const double w = FWD ? __shfl_up_sync(0xffffffffu, o[m], 1) : __shfl_down_sync(0xffffffffu, o[m], 1);
        inc[m] = (FWD ? lane >= 1 : lane + 1 < C) ? w : 0.0;
    }
}

// Coefficient rows in shared memory, 16-byte aligned records of CW doubles:
//   forward  record: l_1 .. l_P            (padded to an even count)
//   backward record: dinv, us_1 .. us_P    (padded to an even count)
template <int P> struct CoefLayout {
    static constexpr int FW = (P + 1) & ~1;        // forward record doubles
    static constexpr int BW = (P + 2) & ~1;        // backward record doubles
};

// One recurrence pass over a chunk (all lanes run the same instructions).
// FWD: y_j = v_j - sum_k l_k y_{j-k};   BWD: x_j = v_j d_j - sum_k us_k x_{j+k}.
// h: incoming state on entry (h[0] = y_{s-1} / x_{e}), outgoing state on exit
// (tail y_{e-1-m} / head x_{s+m}).  Register ring R[pos mod P] (no moves).
// Row j of the chunk's coefficients is at rec + j*rstride (rstride = 0 for
// chunks inside the uniform interior: every read is the same broadcast row).
template <int P, int L, bool FWD, bool STORE>
__device__ __forceinline__ void rec_pass(double (&v)[L], double (&h)[P], const double *rec, int rstride) {
    constexpr int NC = FWD ? CoefLayout<P>::FW : CoefLayout<P>::BW;
    double R[P];
    if (FWD) {
#pragma unroll
        for (int m = 0; m < P; ++m) R[((-1 - m) % P + P) % P] = h[m];
    } else {
#pragma unroll
        for (int m = 0; m < P; ++m) R[(L + m) % P] = h[m];
    }
#pragma unroll
    for (int q = 0; q < L; ++q) {
        const int j = FWD ? q : L - 1 - q;
        const double2 *rp = reinterpret_cast<const double2 *>(rec + j * rstride);
        double cf[NC];
#pragma unroll
        for (int k = 0; k < NC / 2; ++k) {
            const double2 d2 = rp[k];
            cf[2 * k] = d2.x;
            cf[2 * k + 1] = d2.y;
        }
        double t;
        if (FWD) {
            t = v[j];
#pragma unroll
            for (int k = P; k >= 1; --k) t = fma(-cf[k - 1], R[((j - k) % P + P) % P], t);
        } else {
            t = v[j] * cf[0];
#pragma unroll
            for (int k = P; k >= 1; --k) t = fma(-cf[k], R[(j + k) % P], t);
        }
        R[j % P] = t;
        if (STORE) v[j] = t;
    }
    if (FWD) {
#pragma unroll
        for (int m = 0; m < P; ++m) h[m] = R[((L - 1 - m) % P + P) % P];
    } else {
#pragma unroll
        for (int m = 0; m < P; ++m) h[m] = R[m];
    }
}

// Lanes >= C (no chunk) skip the passes; the warp scans are reached by all lanes.
#ifdef ADS_PHASE_TIMING
__device__ long long g_sub[4][8];
#define SUB(k)                                                                                  \
    do {                                                                                        \
        if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 64 + 10))                    \
            g_sub[threadIdx.x == 0 ? 0 : 1][k] = clock64();                                     \
    } while (0)
#else
#define SUB(k) \
    do {       \
    } while (0)
#endif
template <int P, int L>
__device__ __forceinline__ void solve_chunk(double (&v)[L], bool active, const double *fr, const double *br,
                                            int rstride_f, int rstride_b, const double *phif, const double *phib,
                                            int C, int levels, int lane) {
    double h[P], inc[P];
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = 0.0;
    SUB(0);
    if (active) rec_pass<P, L, true, false>(v, h, fr, rstride_f);
    __syncwarp();
    SUB(1);
    warp_scan<P, true>(h, inc, phif, C, levels, lane);
    SUB(2);
    if (active) rec_pass<P, L, true, true>(v, inc, fr, rstride_f);
    SUB(3);
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = 0.0;
    if (active) rec_pass<P, L, false, false>(v, h, br, rstride_b);
    __syncwarp();
    SUB(4);
    warp_scan<P, false>(h, inc, phib, C, levels, lane);
    SUB(5);
    if (active) rec_pass<P, L, false, true>(v, inc, br, rstride_b);
    SUB(6);
}

#ifdef ADS_PHASE_TIMING
__device__ long long g_phase[64][16];
#define PHASE(k)                                                                  \
    do {                                                                          \
        if (blockIdx.x < 8 && t == (int)blockIdx.x && (tid == 0 || tid == 80))     \
            g_phase[blockIdx.x * 3 + (tid == 0 ? 0 : 1)][k] = clock64();          \
    } while (0)
#else
#define PHASE(k) \
    do {         \
    } while (0)
#endif

// Persistent CTAs; tiles (XW lines) round-robin.
template <int P, int L>
__global__ void __launch_bounds__(SWEEP_THREADS, 4) sweep_kernel(const SweepArgs a) {
    constexpr int FW = CoefLayout<P>::FW, BW = CoefLayout<P>::BW;
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int C = a.t.C, n = a.t.n, levels = a.t.levels;
    const int i_lo = a.t.i_lo, i_hi = a.t.i_hi, nedge = C * L - (i_hi - i_lo);
    const int nphi = max(levels, 1) * C * P * P;
    // edge rows (outside [i_lo, i_hi)) + one extra record: the constant interior row
    double *fwd = smem;                            // (nedge + 1) * FW
    double *bwd = fwd + (nedge + 1) * FW;          // (nedge + 1) * BW
    double *sphif = bwd + (nedge + 1) * BW;        // scan matrices (forward, backward)
    double *sphib = sphif + nphi;
    double *tile = sphib + nphi;                   // x: [XW][n]; y/z: [C*L][YP]
    for (int e = tid; e < nphi; e += SWEEP_THREADS) {
        sphif[e] = __ldg(a.t.phif + e);
        sphib[e] = __ldg(a.t.phib + e);
    }
    for (int e = tid; e <= nedge; e += SWEEP_THREADS) {
        const bool cst = e == nedge;
        const int i = e < i_lo ? e : e + (i_hi - i_lo);
#pragma unroll
        for (int k = 0; k < FW; ++k) fwd[e * FW + k] = k < P ? (cst ? a.t.lc[k] : __ldg(a.t.l + (long)i * P + k)) : 0.0;
        bwd[e * BW] = cst ? a.t.dic : __ldg(a.t.dinv + i);
#pragma unroll
        for (int k = 1; k < BW; ++k)
            bwd[e * BW + k] = k <= P ? (cst ? a.t.usc[k - 1] : __ldg(a.t.us + (long)i * P + k - 1)) : 0.0;
    }

    const Geom &g = a.geo;
    long sa, sb, sl;
    int na, nb;
    if (a.dir == 0) { sa = g.sy; sb = g.sz; sl = 1; na = g.n1; nb = g.n2; }
    else if (a.dir == 1) { sa = 1; sb = g.sz; sl = g.sy; na = g.n0; nb = g.n2; }
    else { sa = 1; sb = g.sy; sl = g.sz; na = g.n0; nb = g.n1; }
    const int nab = (na + XW - 1) / XW, ntiles = nab * nb;

    const int s = lane * L;  // chunk start (lanes >= C idle in the passes)
    const bool active = lane < C;
    const bool uni = s >= i_lo && s + L <= i_hi;
    const int erow = uni ? nedge : (s < i_lo ? s : s - (i_hi - i_lo));
    const double *fr = fwd + (active ? erow : nedge) * FW;
    const double *br = bwd + (active ? erow : nedge) * BW;
    const int rsf = (uni || !active) ? 0 : FW, rsb = (uni || !active) ? 0 : BW;
    constexpr int NLD = 20;  // cooperative transfer slots per thread (XW*n <= NLD*256 for n <= 640)

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int la0 = (t % nab) * XW, lb = t / nab, nl = min(XW, na - la0);
        const long base = (long)lb * sb + (long)la0 * sa;
        const int ntot = nl * n;
        __syncthreads();  // previous tile fully stored / tables staged
        PHASE(0);
        // ---- cooperative coalesced load: all requests in flight, then to shared memory
        if (a.dir == 0) {
            // nl consecutive x-lines are one contiguous block of nl*n doubles (sy == n0)
            for (int e0 = 0; e0 < ntot; e0 += NLD * SWEEP_THREADS) {
                double r[NLD];
#pragma unroll
                for (int k = 0; k < NLD; ++k) {
                    const int e = e0 + tid + k * SWEEP_THREADS;
                    r[k] = e < ntot ? __ldg(a.in + base + e) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < NLD; ++k) {
                    const int e = e0 + tid + k * SWEEP_THREADS;
                    if (e < ntot) tile[e] = r[k];
                }
            }
        } else {
            const int tot = n * XW;
            for (int e0 = 0; e0 < tot; e0 += NLD * SWEEP_THREADS) {
                double r[NLD];
#pragma unroll
                for (int k = 0; k < NLD; ++k) {
                    const int e = e0 + tid + k * SWEEP_THREADS, i = e >> 3, q = e & (XW - 1);
                    r[k] = (e < tot && q < nl) ? __ldg(a.in + base + (long)i * sl + q) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < NLD; ++k) {
                    const int e = e0 + tid + k * SWEEP_THREADS;
                    if (e < tot) tile[(e >> 3) * YP + (e & (XW - 1))] = r[k];
                }
            }
        }
        __syncthreads();
        PHASE(1);
        // ---- warp w solves line w (lane = chunk)
        if (w < nl) {
            double v[L];
#pragma unroll
            for (int j = 0; j < L; ++j) {
                const int i = s + j;
                v[j] = i < n ? (a.dir == 0 ? tile[w * n + i] : tile[i * YP + w]) : 0.0;
            }
            solve_chunk<P, L>(v, active, fr, br, rsf, rsb, sphif, sphib, C, levels, lane);
#pragma unroll
            for (int j = 0; j < L; ++j) {
                const int i = s + j;
                if (i < n) {
                    if (a.dir == 0) tile[w * n + i] = v[j];
                    else tile[i * YP + w] = v[j];
                }
            }
        }
        __syncthreads();
        PHASE(2);
        // ---- cooperative coalesced store (z: fused kick V += kick * a)
        if (a.dir == 0) {
            for (int e = tid; e < ntot; e += SWEEP_THREADS) a.out[base + e] = tile[e];
        } else {
            const int tot = n * XW;
            for (int e = tid; e < tot; e += SWEEP_THREADS) {
                const int i = e >> 3, q = e & (XW - 1);
                if (q < nl) {
                    const long idx = base + (long)i * sl + q;
                    const double x = tile[i * YP + q];
                    if (a.mode == 0) {
                        a.out[idx] = x;
                    } else {
                        a.V[idx] = fma(a.kick, x, a.V[idx]);
                        if (a.out) a.out[idx] = x;
                    }
                }
            }
        }
        PHASE(3);
    }
}

// ------------------------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------------------------
template <int P>
__global__ void axis_apply_kernel(int d, const double *__restrict__ band, const double *__restrict__ in,
                                  double *__restrict__ out, Geom g) {
    constexpr int W = 2 * P + 1;
    long N = (long)g.n0 * g.n1 * g.n2;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x) {
        int i = q % g.n0;
        long t = q / g.n0;
        int j = t % g.n1;
        int k = t / g.n1;
        int r = d == 0 ? i : d == 1 ? j : k;
        int nd = d == 0 ? g.n0 : d == 1 ? g.n1 : g.n2;
        long st = d == 0 ? 1 : d == 1 ? g.sy : g.sz;
        long idx = (long)k * g.sz + (long)j * g.sy + i;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < W; ++c) {
            int col = r - P + c;
            if (col >= 0 && col < nd) acc = fma(band[(long)r * W + c], in[idx + (long)(col - r) * st], acc);
        }
        out[idx] = acc;
    }
}

__global__ void axpby_kernel(long N, double alpha, const double *__restrict__ x, double beta, double *__restrict__ y) {
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x)
        y[q] = alpha * x[q] + beta * y[q];
}

__global__ void mask_boundary_kernel(double *u, Geom g) {
    long N = (long)g.n0 * g.n1 * g.n2;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x) {
        int i = q % g.n0;
        long t = q / g.n0;
        int j = t % g.n1;
        int k = t / g.n1;
        if (i == 0 || j == 0 || k == 0 || i == g.n0 - 1 || j == g.n1 - 1 || k == g.n2 - 1)
            u[(long)k * g.sz + (long)j * g.sy + i] = 0.0;
    }
}

__global__ void add_separable_kernel(double *u, double amp, const double *sx, const double *sy, const double *sz,
                                     Geom g) {
    long N = (long)g.n0 * g.n1 * g.n2;
    for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < N; q += (long)gridDim.x * blockDim.x) {
        int i = q % g.n0;
        long t = q / g.n0;
        int j = t % g.n1;
        int k = t / g.n1;
        u[(long)k * g.sz + (long)j * g.sy + i] += amp * sx[i] * sy[j] * sz[k];
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

template <int P>
static void kop_launch(const KopArgs &a, cudaStream_t s) {
    dim3 blk(32, 8);
    int zl = a.zlen > 0 ? a.zlen : a.geo.n2;
    dim3 grd((a.geo.n0 + 31) / 32, (a.geo.n1 + 7) / 8, (a.geo.n2 + zl - 1) / zl);
    KopArgs b = a;
    b.zlen = zl;
    kop_kernel<P><<<grd, blk, 0, s>>>(b);
}

int launch_kop(int p, const KopArgs &a, cudaStream_t s) {
    switch (p) {
        case 1: kop_launch<1>(a, s); break;
        case 2: kop_launch<2>(a, s); break;
        case 3: kop_launch<3>(a, s); break;
        case 4: kop_launch<4>(a, s); break;
        case 5: kop_launch<5>(a, s); break;
        default: return -1;
    }
    return 0;
}

template <int P, int L>
static void sweep_launch(const SweepArgs &a, cudaStream_t s) {
    const Geom &g = a.geo;
    const int na = a.dir == 0 ? g.n1 : g.n0, nb = a.dir == 2 ? g.n1 : g.n2;
    const int ntiles = ((na + XW - 1) / XW) * nb;
    const int nedge = a.t.C * L - (a.t.i_hi - a.t.i_lo);
    const size_t nphi = (size_t)std::max(a.t.levels, 1) * a.t.C * P * P;
    size_t tile = a.dir == 0 ? (size_t)XW * a.t.n : (size_t)a.t.n * YP;
    size_t sm = sizeof(double) * (2 * nphi + (size_t)(nedge + 1) * (CoefLayout<P>::FW + CoefLayout<P>::BW) + tile);
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(sweep_kernel<P, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<P, L>, SWEEP_THREADS, sm);
    dim3 grd(std::min(ntiles, std::max(per_sm, 1) * nsm));
    sweep_kernel<P, L><<<grd, SWEEP_THREADS, sm, s>>>(a);
}

template <int P>
static int sweep_dispatch(const SweepArgs &a, cudaStream_t s) {
    switch (a.t.L) {
#define ADS_L(LV) \
    case LV: sweep_launch<P, LV>(a, s); return 0;
        ADS_L(1) ADS_L(3) ADS_L(5) ADS_L(9) ADS_L(13) ADS_L(17) ADS_L(21) ADS_L(25) ADS_L(33)
#undef ADS_L
    }
    return -1;
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

int launch_axis_apply(int p, int d, const double *band, const double *in, double *out, const Geom &g,
                      cudaStream_t s) {
    long N = (long)g.n0 * g.n1 * g.n2;
    int grd = grid_for(N);
    switch (p) {
        case 1: axis_apply_kernel<1><<<grd, 256, 0, s>>>(d, band, in, out, g); break;
        case 2: axis_apply_kernel<2><<<grd, 256, 0, s>>>(d, band, in, out, g); break;
        case 3: axis_apply_kernel<3><<<grd, 256, 0, s>>>(d, band, in, out, g); break;
        case 4: axis_apply_kernel<4><<<grd, 256, 0, s>>>(d, band, in, out, g); break;
        case 5: axis_apply_kernel<5><<<grd, 256, 0, s>>>(d, band, in, out, g); break;
        default: return -1;
    }
    return 0;
}

int launch_axpby(long N, double alpha, const double *x, double beta, double *y, cudaStream_t s) {
    axpby_kernel<<<grid_for(N), 256, 0, s>>>(N, alpha, x, beta, y);
    return 0;
}

int launch_mask_boundary(double *u, const Geom &g, cudaStream_t s) {
    mask_boundary_kernel<<<grid_for((long)g.n0 * g.n1 * g.n2), 256, 0, s>>>(u, g);
    return 0;
}

int launch_add_separable(double *u, double amp, const double *sx, const double *sy, const double *sz, const Geom &g,
                         cudaStream_t s) {
    add_separable_kernel<<<grid_for((long)g.n0 * g.n1 * g.n2), 256, 0, s>>>(u, amp, sx, sy, sz, g);
    return 0;
}

int launch_dot(long N, const double *x, const double *y, double *partial, double *res, cudaStream_t s) {
    dot_partial_kernel<<<DOT_BLOCKS, DOT_THREADS, 0, s>>>(N, x, y, partial);
    dot_final_kernel<<<1, 256, 0, s>>>(partial, res);
    return 0;
}

}  // namespace ads
