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
// ------------------------------------------------------------------------------------------
constexpr int XW = 8;  // lines per CTA (adjacent lines; coalescing axis for y/z)

// Kogge-Stone scan of the chunk boundary states across the C chunks of each of
// the XW lines of the CTA.  forward: o_c += Phi_c^(lv) o_{c-2^lv};
// backward: o_c += Psi_c^(lv) o_{c+2^lv}.  Returns the neighbour's final state
// (the incoming state of this chunk) in inc[].
template <int P, bool FWD>
__device__ __forceinline__ void chunk_scan(double (&o)[P], double (&inc)[P], double *sbuf, const double *phi,
                                           int C, int levels, int c, int xl) {
    for (int lv = 0; lv < levels; ++lv) {
        const int d = 1 << lv;
        double *buf = sbuf + (lv & 1) * (C * XW * P);
#pragma unroll
        for (int m = 0; m < P; ++m) buf[(c * XW + xl) * P + m] = o[m];
        __syncthreads();
        const int src = FWD ? c - d : c + d;
        if (FWD ? (src >= 0) : (src < C)) {
            double u[P];
#pragma unroll
            for (int m = 0; m < P; ++m) u[m] = buf[(src * XW + xl) * P + m];
            const double *ph = phi + ((long)lv * C + c) * P * P;
            double t[P];
#pragma unroll
            for (int i = 0; i < P; ++i) {
                double s = o[i];
#pragma unroll
                for (int j = 0; j < P; ++j) s = fma(__ldg(ph + i * P + j), u[j], s);
                t[i] = s;
            }
#pragma unroll
            for (int i = 0; i < P; ++i) o[i] = t[i];
        }
    }
    double *buf = sbuf + 2 * (C * XW * P);
#pragma unroll
    for (int m = 0; m < P; ++m) buf[(c * XW + xl) * P + m] = o[m];
    __syncthreads();
    const int nb = FWD ? c - 1 : c + 1;
    const bool has = FWD ? (nb >= 0) : (nb < C);
#pragma unroll
    for (int m = 0; m < P; ++m) inc[m] = has ? buf[(nb * XW + xl) * P + m] : 0.0;
    __syncthreads();
}

// Forward recurrence y_i = r_i - sum_k l_{i,k} y_{i-k} over the chunk, from the
// incoming state h (h[0] = y_{s-1}, ...).  UNI: constant coefficients lc.
// STORE: overwrite v with y.  On return h holds the chunk's tail state.
template <int P, int L, bool UNI, bool STORE>
__device__ __forceinline__ void fwd_pass(double (&v)[L], double (&h)[P], int s, int len, const double *__restrict__ Lt,
                                         const double (&lc)[P]) {
#pragma unroll
    for (int j = 0; j < L; ++j) {
        if (UNI || j < len) {
            double t = v[j];
#pragma unroll
            for (int k = P - 1; k >= 0; --k) t = fma(-(UNI ? lc[k] : __ldg(Lt + (long)(s + j) * P + k)), h[k], t);
#pragma unroll
            for (int m = P - 1; m > 0; --m) h[m] = h[m - 1];
            h[0] = t;
            if (STORE) v[j] = t;
        }
    }
}

// Backward recurrence x_i = y_i / u_ii - sum_k (u_{i,i+k}/u_ii) x_{i+k} over the chunk,
// from the incoming state h (h[0] = x_e, ...).  On return h holds the head state.
template <int P, int L, bool UNI, bool STORE>
__device__ __forceinline__ void bwd_pass(double (&v)[L], double (&h)[P], int s, int len, const double *__restrict__ Ut,
                                         const double *__restrict__ Dt, const double (&uc)[P], double dc) {
#pragma unroll
    for (int j = L - 1; j >= 0; --j) {
        if (UNI || j < len) {
            double t = v[j] * (UNI ? dc : __ldg(Dt + s + j));
#pragma unroll
            for (int k = P - 1; k >= 0; --k) t = fma(-(UNI ? uc[k] : __ldg(Ut + (long)(s + j) * P + k)), h[k], t);
#pragma unroll
            for (int m = P - 1; m > 0; --m) h[m] = h[m - 1];
            h[0] = t;
            if (STORE) v[j] = t;
        }
    }
}

// Uniform chunks (len == L, constant coefficients): the last P values live in a
// register ring R indexed by position mod P (all indices compile-time).
template <int P, int L, bool STORE>
__device__ __forceinline__ void fwd_uni(double (&v)[L], double (&h)[P], const double (&lc)[P]) {
    double R[P];
#pragma unroll
    for (int m = 0; m < P; ++m) R[((-1 - m) % P + P) % P] = h[m];  // y_{-1-m}
#pragma unroll
    for (int j = 0; j < L; ++j) {
        double t = v[j];
#pragma unroll
        for (int k = P; k >= 1; --k) t = fma(-lc[k - 1], R[((j - k) % P + P) % P], t);
        R[j % P] = t;
        if (STORE) v[j] = t;
    }
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = R[((L - 1 - m) % P + P) % P];  // tail y_{L-1-m}
}

template <int P, int L, bool STORE>
__device__ __forceinline__ void bwd_uni(double (&v)[L], double (&h)[P], const double (&uc)[P], double dc) {
    double R[P];
#pragma unroll
    for (int m = 0; m < P; ++m) R[(L + m) % P] = h[m];  // x_{L+m}
#pragma unroll
    for (int j = L - 1; j >= 0; --j) {
        double t = v[j] * dc;
#pragma unroll
        for (int k = P; k >= 1; --k) t = fma(-uc[k - 1], R[(j + k) % P], t);
        R[j % P] = t;
        if (STORE) v[j] = t;
    }
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = R[m % P];  // head x_m
}

template <int P, int L>
__global__ void __launch_bounds__(256, 3) sweep_kernel(const SweepArgs a) {
    extern __shared__ double smem[];
    const int xl = threadIdx.x, c = threadIdx.y, C = a.t.C;
    const int nthr = XW * C, tid = c * XW + xl;
    const int n = a.t.n;
    double *sbuf = smem;                   // 3 * C * XW * P scan buffers
    double *tile = smem + 3 * C * XW * P;  // x-lines: XW x npad

    const Geom &g = a.geo;
    long sa, sb, sl;
    int na;
    if (a.dir == 0) { sa = g.sy; sb = g.sz; sl = 1; na = g.n1; }
    else if (a.dir == 1) { sa = 1; sb = g.sz; sl = g.sy; na = g.n0; }
    else { sa = 1; sb = g.sy; sl = g.sz; na = g.n0; }
    const int la0 = blockIdx.x * XW, lb = blockIdx.y;
    const long base = (long)lb * sb + (long)la0 * sa;
    const bool valid = la0 + xl < na;

    const int s = c * L, len = min(L, n - s);
    const bool uni = s >= a.t.i_lo && s + L <= a.t.i_hi;
    double lc[P], uc[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        lc[k] = a.t.lc[k];
        uc[k] = a.t.usc[k];
    }
    const double dc = a.t.dic;

    double v[L];
    const int npad = n | 1;  // odd row pitch: conflict-free transposed reads
    const int ntile = min(XW, na - la0) * n;  // x: nl consecutive lines, contiguous (sy == n0)
    const double inv_n = 1.0 / n;
    if (a.dir == 0) {
        // every thread issues its L loads before any store (loads in flight together)
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const int e = tid + j * nthr;
            v[j] = e < ntile ? __ldg(a.in + base + e) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const int e = tid + j * nthr;
            if (e < ntile) {
                const int q = __double2int_rz((e + 0.5) * inv_n);
                tile[q * npad + (e - q * n)] = v[j];
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < L; ++j) v[j] = (j < len && valid) ? tile[xl * npad + s + j] : 0.0;
    } else {
        const double *src = a.in + base + xl + (long)s * sl;
#pragma unroll
        for (int j = 0; j < L; ++j) v[j] = (j < len && valid) ? __ldg(src + (long)j * sl) : 0.0;
    }

    const double *Lt = a.t.l, *Ut = a.t.us, *Dt = a.t.dinv;
    double h[P], inc[P];

    // pass 1: forward from zero state -> tail; scan; pass 2: forward from the exact state
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = 0.0;
    if (uni) fwd_uni<P, L, false>(v, h, lc);
    else fwd_pass<P, L, false, false>(v, h, s, len, Lt, lc);
    if (C > 1) chunk_scan<P, true>(h, inc, sbuf, a.t.phif, C, a.t.levels, c, xl);
    else {
#pragma unroll
        for (int m = 0; m < P; ++m) inc[m] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = inc[m];
    if (uni) fwd_uni<P, L, true>(v, h, lc);
    else fwd_pass<P, L, false, true>(v, h, s, len, Lt, lc);

    // pass 3: backward from zero state -> head; scan; pass 4: backward from the exact state
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = 0.0;
    if (uni) bwd_uni<P, L, false>(v, h, uc, dc);
    else bwd_pass<P, L, false, false>(v, h, s, len, Ut, Dt, uc, dc);
    if (C > 1) chunk_scan<P, false>(h, inc, sbuf, a.t.phib, C, a.t.levels, c, xl);
    else {
#pragma unroll
        for (int m = 0; m < P; ++m) inc[m] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = inc[m];
    if (uni) bwd_uni<P, L, true>(v, h, uc, dc);
    else bwd_pass<P, L, false, true>(v, h, s, len, Ut, Dt, uc, dc);

    // store
    if (a.dir == 0) {
#pragma unroll
        for (int j = 0; j < L; ++j)
            if (j < len) tile[xl * npad + s + j] = v[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const int e = tid + j * nthr;
            if (e < ntile) {
                const int q = __double2int_rz((e + 0.5) * inv_n);
                a.out[base + e] = tile[q * npad + (e - q * n)];
            }
        }
    } else if (valid) {
        const long off = base + xl + (long)s * sl;
        if (a.mode == 0) {
#pragma unroll
            for (int j = 0; j < L; ++j)
                if (j < len) a.out[off + (long)j * sl] = v[j];
        } else {
#pragma unroll
            for (int j = 0; j < L; ++j)
                if (j < len) {
                    const long idx = off + (long)j * sl;
                    a.V[idx] = fma(a.kick, v[j], a.V[idx]);
                    if (a.out) a.out[idx] = v[j];
                }
        }
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
    int na = a.dir == 0 ? g.n1 : g.n0;
    int nb = a.dir == 2 ? g.n1 : g.n2;
    dim3 blk(XW, a.t.C);
    dim3 grd((na + XW - 1) / XW, nb);
    size_t sm = sizeof(double) * (3 * (size_t)a.t.C * XW * P);
    if (a.dir == 0) sm += sizeof(double) * (size_t)XW * (a.t.n | 1);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(sweep_kernel<P, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    sweep_kernel<P, L><<<grd, blk, sm, s>>>(a);
}

template <int P>
static int sweep_dispatch(const SweepArgs &a, cudaStream_t s) {
    switch (a.t.L) {
#define ADS_L(LV) \
    case LV: sweep_launch<P, LV>(a, s); return 0;
        ADS_L(1) ADS_L(2) ADS_L(3) ADS_L(4) ADS_L(5) ADS_L(8) ADS_L(9) ADS_L(12) ADS_L(13) ADS_L(16) ADS_L(17)
        ADS_L(24) ADS_L(25) ADS_L(32) ADS_L(33)
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
