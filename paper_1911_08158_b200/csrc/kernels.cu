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
// ------------------------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(256) kop_kernel(const KopArgs a) {
    constexpr int TX = 32, TY = 8, W = 2 * P + 1, HX = TX + 2 * P, HY = TY + 2 * P;
    constexpr int NE = HX * HY, NQ = (NE + TX * TY - 1) / (TX * TY);
    __shared__ double Ps[HY][HX];
    __shared__ double X1[HY][TX], X2[HY][TX];

    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int n0 = a.geo.n0, n1 = a.geo.n1, n2 = a.geo.n2;
    const long sy = a.geo.sy, sz = a.geo.sz;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int z0 = blockIdx.z * a.zlen, z1 = min(n2, z0 + a.zlen);
    const int gx = x0 + tx, gy = y0 + ty;
    const bool inx = gx < n0, iny = gy < n1;

    double mxr[W], kxr[W], myr[W], kyr[W];
#pragma unroll
    for (int c = 0; c < W; ++c) {
        mxr[c] = inx ? __ldg(a.mx + (long)gx * W + c) : 0.0;
        kxr[c] = inx ? __ldg(a.kx + (long)gx * W + c) : 0.0;
        myr[c] = iny ? __ldg(a.my + (long)gy * W + c) : 0.0;
        kyr[c] = iny ? __ldg(a.ky + (long)gy * W + c) : 0.0;
    }
    double Sr[W], Tr[W];
#pragma unroll
    for (int c = 0; c < W; ++c) Sr[c] = Tr[c] = 0.0;

    // prefetch registers for one haloed plane
    double pu[NQ], pv[NQ];
    long pidx[NQ];
    bool pval[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        int e = tid + q * TX * TY;
        int ry = e / HX, rx = e - ry * HX;
        int X = x0 - P + rx, Y = y0 - P + ry;
        pval[q] = (e < NE) && X >= 0 && X < n0 && Y >= 0 && Y < n1;
        pidx[q] = (long)Y * sy + X;
    }
    auto load = [&](int kin) {
        const bool kv = kin >= 0 && kin < n2;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (pval[q] && kv) {
                long idx = (long)kin * sz + pidx[q];
                pu[q] = __ldg(a.U + idx);
                pv[q] = __ldg(a.V + idx);
            } else {
                pu[q] = 0.0;
                pv[q] = 0.0;
            }
        }
    };

    load(z0 - P);
    for (int kin = z0 - P; kin < z1 + P; ++kin) {
        // commit plane kin: P = U + tau V into shared memory (and HBM for owned points)
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            int e = tid + q * TX * TY;
            if (e < NE) {
                int ry = e / HX, rx = e - ry * HX;
                double pp = fma(a.tau, pv[q], pu[q]);
                Ps[ry][rx] = pp;
                if (a.Pout && kin >= z0 && kin < z1 && pval[q] && rx >= P && rx < P + TX && ry >= P && ry < P + TY)
                    a.Pout[(long)kin * sz + pidx[q]] = pp;
            }
        }
        __syncthreads();
        if (kin + 1 < z1 + P) load(kin + 1);  // in flight during the passes below

        // x-pass: X1 = Mx P, X2 = Kx P on all haloed rows
        for (int ry = ty; ry < HY; ry += TY) {
            double s1 = 0.0, s2 = 0.0;
#pragma unroll
            for (int c = 0; c < W; ++c) {
                double v = Ps[ry][tx + c];
                s1 = fma(mxr[c], v, s1);
                s2 = fma(kxr[c], v, s2);
            }
            X1[ry][tx] = s1;
            X2[ry][tx] = s2;
        }
        __syncthreads();

        // y-pass: S = My Kx P + Ky Mx P,  T = My Mx P
        double S = 0.0, T = 0.0;
#pragma unroll
        for (int c = 0; c < W; ++c) {
            double x1 = X1[ty + c][tx], x2 = X2[ty + c][tx];
            S = fma(myr[c], x2, S);
            S = fma(kyr[c], x1, S);
            T = fma(myr[c], x1, T);
        }
#pragma unroll
        for (int c = 0; c < W - 1; ++c) {
            Sr[c] = Sr[c + 1];
            Tr[c] = Tr[c + 1];
        }
        Sr[W - 1] = S;
        Tr[W - 1] = T;

        // z-pass for output plane k = kin - P:  K P = Mz S + Kz T
        const int k = kin - P;
        if (k >= z0 && inx && iny) {
            const double *mzr = a.mz + (long)k * W;
            const double *kzr = a.kz + (long)k * W;
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < W; ++c) {
                acc = fma(__ldg(mzr + c), Sr[c], acc);
                acc = fma(__ldg(kzr + c), Tr[c], acc);
            }
            double src = 0.0;
            if (a.bx) src = a.g * __ldg(a.bx + gx) * __ldg(a.by + gy) * __ldg(a.bz + k);
            a.r[(long)k * sz + (long)gy * sy + gx] = fma(a.sign, acc, src);
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

template <int P, int LMAX>
__global__ void __launch_bounds__(256) sweep_kernel(const SweepArgs a) {
    extern __shared__ double smem[];
    const int xl = threadIdx.x, c = threadIdx.y, C = a.t.C;
    const int nthr = XW * C, tid = c * XW + xl;
    const int n = a.t.n;
    double *sbuf = smem;                        // 3 * C * XW * P scan buffers
    double *tile = smem + 3 * C * XW * P;       // x-lines: XW x npad

    // line set: lines indexed (la, lb); the XW lines of this CTA are la0 .. la0+XW-1
    const Geom &g = a.geo;
    long sa, sb, sl;
    int na;
    if (a.dir == 0) { sa = g.sy; sb = g.sz; sl = 1; na = g.n1; }
    else if (a.dir == 1) { sa = 1; sb = g.sz; sl = g.sy; na = g.n0; }
    else { sa = 1; sb = g.sy; sl = g.sz; na = g.n0; }
    const int la0 = blockIdx.x * XW, lb = blockIdx.y;
    const long base = (long)lb * sb + (long)la0 * sa;
    const int la = la0 + xl;
    const bool valid = la < na;

    const int s = __ldg(a.t.cs + c), len = __ldg(a.t.cs + c + 1) - s;
    double v[LMAX];

    int npad = n | 1;  // odd row pitch: conflict-free transposed reads
    if (a.dir == 0) {
        const int nl = min(XW, na - la0);
        for (int q = 0; q < nl; ++q) {
            const double *src = a.in + base + (long)q * sa;
            for (int i = tid; i < n; i += nthr) tile[q * npad + i] = __ldg(src + i);
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < LMAX; ++j) v[j] = (j < len && valid) ? tile[xl * npad + s + j] : 0.0;
    } else {
        const double *src = a.in + base + xl + (long)s * sl;
#pragma unroll
        for (int j = 0; j < LMAX; ++j) v[j] = (j < len && valid) ? __ldg(src + (long)j * sl) : 0.0;
    }

    const double *L = a.t.l, *US = a.t.us, *DI = a.t.dinv;
    double h[P], o[P], inc[P];

    // pass 1: forward recurrence y_i = r_i - sum_k l_{i,k} y_{i-k} from zero state -> tail
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = 0.0;
#pragma unroll
    for (int j = 0; j < LMAX; ++j) {
        if (j < len) {
            const double *lr = L + (long)(s + j) * P;
            double t = v[j];
#pragma unroll
            for (int k = P - 1; k >= 0; --k) t = fma(-__ldg(lr + k), h[k], t);
#pragma unroll
            for (int m = P - 1; m > 0; --m) h[m] = h[m - 1];
            h[0] = t;
        }
    }
#pragma unroll
    for (int m = 0; m < P; ++m) o[m] = h[m];
    if (a.t.C > 1) {
        chunk_scan<P, true>(o, inc, sbuf, a.t.phif, C, a.t.levels, c, xl);
    } else {
#pragma unroll
        for (int m = 0; m < P; ++m) inc[m] = 0.0;
    }
    // pass 2: forward recurrence from the exact incoming state
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = inc[m];
#pragma unroll
    for (int j = 0; j < LMAX; ++j) {
        if (j < len) {
            const double *lr = L + (long)(s + j) * P;
            double t = v[j];
#pragma unroll
            for (int k = P - 1; k >= 0; --k) t = fma(-__ldg(lr + k), h[k], t);
#pragma unroll
            for (int m = P - 1; m > 0; --m) h[m] = h[m - 1];
            h[0] = t;
            v[j] = t;
        }
    }
    // pass 3: backward recurrence x_i = y_i / u_ii - sum_k (u_{i,i+k}/u_ii) x_{i+k} from zero -> head
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = 0.0;
#pragma unroll
    for (int j = LMAX - 1; j >= 0; --j) {
        if (j < len) {
            const double *ur = US + (long)(s + j) * P;
            double t = v[j] * __ldg(DI + s + j);
#pragma unroll
            for (int k = P - 1; k >= 0; --k) t = fma(-__ldg(ur + k), h[k], t);
#pragma unroll
            for (int m = P - 1; m > 0; --m) h[m] = h[m - 1];
            h[0] = t;
        }
    }
#pragma unroll
    for (int m = 0; m < P; ++m) o[m] = h[m];
    if (a.t.C > 1) {
        chunk_scan<P, false>(o, inc, sbuf, a.t.phib, C, a.t.levels, c, xl);
    } else {
#pragma unroll
        for (int m = 0; m < P; ++m) inc[m] = 0.0;
    }
    // pass 4: backward recurrence from the exact incoming state
#pragma unroll
    for (int m = 0; m < P; ++m) h[m] = inc[m];
#pragma unroll
    for (int j = LMAX - 1; j >= 0; --j) {
        if (j < len) {
            const double *ur = US + (long)(s + j) * P;
            double t = v[j] * __ldg(DI + s + j);
#pragma unroll
            for (int k = P - 1; k >= 0; --k) t = fma(-__ldg(ur + k), h[k], t);
#pragma unroll
            for (int m = P - 1; m > 0; --m) h[m] = h[m - 1];
            h[0] = t;
            v[j] = t;
        }
    }

    // store
    if (a.dir == 0) {
#pragma unroll
        for (int j = 0; j < LMAX; ++j)
            if (j < len) tile[xl * npad + s + j] = v[j];
        __syncthreads();
        const int nl = min(XW, na - la0);
        for (int q = 0; q < nl; ++q) {
            double *dst = a.out + base + (long)q * sa;
            for (int i = tid; i < n; i += nthr) dst[i] = tile[q * npad + i];
        }
    } else if (valid) {
        const long off = base + xl + (long)s * sl;
        if (a.mode == 0) {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
                if (j < len) a.out[off + (long)j * sl] = v[j];
        } else {
#pragma unroll
            for (int j = 0; j < LMAX; ++j)
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

template <int P, int LMAX>
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
        cudaFuncSetAttribute(sweep_kernel<P, LMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    sweep_kernel<P, LMAX><<<grd, blk, sm, s>>>(a);
}

template <int P>
static int sweep_dispatch(const SweepArgs &a, cudaStream_t s) {
    int L = a.t.lmax;
    if (L <= 4) sweep_launch<P, 4>(a, s);
    else if (L <= 8) sweep_launch<P, 8>(a, s);
    else if (L <= 12) sweep_launch<P, 12>(a, s);
    else if (L <= 17) sweep_launch<P, 17>(a, s);
    else if (L <= 24) sweep_launch<P, 24>(a, s);
    else if (L <= 33) sweep_launch<P, 33>(a, s);
    else return -1;
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
