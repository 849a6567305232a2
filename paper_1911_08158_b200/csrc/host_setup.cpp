// host_setup.cpp -- see host_setup.h.  Runs once per ads_create on the host.
#include "host_setup.h"

#include <algorithm>
#include <cmath>
#include <limits>

namespace ads {

// The 1D Gram matrices and load vectors are accumulated in extended precision (x87 long double,
// 64-bit significand) and rounded to fp64 once: quadrature in fp64 leaves entries ~1e-13 off in
// relative terms, and the stiffness rows' rounding error is amplified by (sigma/h)^2 in K P on
// smooth data (T1).  Host work, once per handle.
using xreal = long double;

// Gauss-Legendre nodes/weights on [-1,1]: Newton iteration on P_m using the
// Bonnet recurrence (j+1) P_{j+1} = (2j+1) x P_j - j P_{j-1};
// w = 2 / ((1 - x^2) P_m'(x)^2).
template <class T>
static void gauss_legendre_t(int m, T *x, T *w) {
    const T kPi = 3.14159265358979323846264338327950288L;
    for (int i = 0; i < (m + 1) / 2; ++i) {
        T z = std::cos(kPi * (T)(i + 0.75) / (T)(m + 0.5));
        T pm = 0, dpm = 0;
        for (int it = 0; it < 64; ++it) {
            T pjm1 = 0.0, pj = 1.0;
            for (int j = 0; j < m; ++j) {
                T pjp1 = ((2 * j + 1) * z * pj - j * pjm1) / (T)(j + 1);
                pjm1 = pj;
                pj = pjp1;
            }
            pm = pj;
            dpm = m * (z * pj - pjm1) / (z * z - 1);
            T dz = pm / dpm;
            z -= dz;
            if (std::fabs(dz) <= std::numeric_limits<T>::epsilon() * 0.25) break;
        }
        {
            T pjm1 = 0.0, pj = 1.0;
            for (int j = 0; j < m; ++j) {
                T pjp1 = ((2 * j + 1) * z * pj - j * pjm1) / (T)(j + 1);
                pjm1 = pj;
                pj = pjp1;
            }
            dpm = m * (z * pj - pjm1) / (z * z - 1);
        }
        T wi = 2 / ((1 - z * z) * dpm * dpm);
        x[i] = -z;
        x[m - 1 - i] = z;
        w[i] = w[m - 1 - i] = wi;
    }
    if (m % 2 == 1) x[m / 2] = 0;
}

int gauss_legendre(int m, double *x, double *w) {
    xreal xl[64], wl[64];
    if (m < 1 || m > 64) return -1;
    gauss_legendre_t<xreal>(m, xl, wl);
    for (int i = 0; i < m; ++i) {
        x[i] = (double)xl[i];
        w[i] = (double)wl[i];
    }
    return 0;
}

// de Boor's triangular evaluation of the p+1 nonzero B-splines and their first
// derivatives in knot span `span` (t[span] <= x < t[span+1]).
template <class T>
static void basis_and_derivs_t(const T *t, int p, int span, T x, T *N, T *dN) {
    T ndu[8][8];
    T left[8], right[8];
    ndu[0][0] = 1;
    for (int j = 1; j <= p; ++j) {
        left[j] = x - t[span + 1 - j];
        right[j] = t[span + j] - x;
        T saved = 0;
        for (int r = 0; r < j; ++r) {
            ndu[j][r] = right[r + 1] + left[j - r];      // lower triangle: knot differences
            T tmp = ndu[r][j - 1] / ndu[j][r];
            ndu[r][j] = saved + right[r + 1] * tmp;      // upper triangle: basis values
            saved = left[j - r] * tmp;
        }
        ndu[j][j] = saved;
    }
    for (int r = 0; r <= p; ++r) N[r] = ndu[r][p];
    // first derivative: N'_{r} = p (N_{r,p-1}/(t_{r+p}-t_r) - N_{r+1,p-1}/(t_{r+p+1}-t_{r+1}))
    for (int r = 0; r <= p; ++r) {
        T d = 0;
        if (r >= 1) d += ndu[r - 1][p - 1] / ndu[p][r - 1];
        if (r <= p - 1) d -= ndu[r][p - 1] / ndu[p][r];
        dN[r] = p * d;
    }
}

void basis_and_derivs(const std::vector<double> &t, int p, int span, double x, double *N, double *dN) {
    basis_and_derivs_t<double>(t.data(), p, span, x, N, dN);
}

// open uniform knots in extended precision: t_i = e / nel
static std::vector<xreal> knots_x(int p, int nel) {
    std::vector<xreal> t(nel + 2 * p + 1);
    for (int i = 0; i < (int)t.size(); ++i) t[i] = (xreal)std::min(std::max(i - p, 0), nel) / (xreal)nel;
    return t;
}

int build_space(int p, int nel, int bc, Space1D &s) {
    if (p < 1 || p > 5 || nel < 1) return -1;
    s.p = p;
    s.nel = nel;
    s.n = nel + p;
    s.bc = bc;
    const std::vector<xreal> tx = knots_x(p, nel);
    s.knots.assign(tx.size(), 0.0);
    for (size_t i = 0; i < tx.size(); ++i) s.knots[i] = (double)tx[i];
    s.M = Band(s.n, p);
    s.K = Band(s.n, p);
    s.B = Band(s.n, p);
    const int W = 2 * p + 1;
    std::vector<xreal> Mx((size_t)s.n * W, 0), Kx((size_t)s.n * W, 0), Bx((size_t)s.n * W, 0);
    xreal xg[8], wg[8];
    gauss_legendre_t<xreal>(p + 1, xg, wg);
    xreal N[8], dN[8];
    for (int e = 0; e < nel; ++e) {
        int span = e + p;
        xreal a = tx[span], b = tx[span + 1];
        xreal half = (b - a) / 2, mid = (a + b) / 2;
        for (int q = 0; q <= p; ++q) {
            xreal x = mid + half * xg[q], w = half * wg[q];
            basis_and_derivs_t<xreal>(tx.data(), p, span, x, N, dN);
            for (int r = 0; r <= p; ++r)
                for (int c = 0; c <= p; ++c) {
                    const size_t ix = (size_t)(e + r) * W + (c - r + p);
                    Mx[ix] += w * N[r] * N[c];
                    Kx[ix] += w * dN[r] * dN[c];
                    Bx[ix] += w * dN[r] * N[c];
                }
        }
    }
    for (size_t q = 0; q < Mx.size(); ++q) {
        s.M.v[q] = (double)Mx[q];
        s.K.v[q] = (double)Kx[q];
        s.B.v[q] = (double)Bx[q];
    }
    // Uniform mesh: every row whose basis function and all p neighbours on each
    // side are interior cardinal B-splines (rows [2p, n-1-2p]) has the same band
    // in exact arithmetic (h-scaled cardinal B-spline autocorrelation); quadrature
    // rounding can still jitter them by an ulp.  Use the middle row for all of them so
    // the interior is bitwise Toeplitz ("Toeplitz interior").
    {
        const int lo = 2 * p, hi = s.n - 1 - 2 * p, mid = s.n / 2;
        if (hi - lo >= 2) {
            double rm[2 * 8 + 1], rk[2 * 8 + 1], rb[2 * 8 + 1];
            for (int k = -p; k <= p; ++k) {
                rm[k + p] = s.M.at(mid, mid + k);
                rk[k + p] = s.K.at(mid, mid + k);
                rb[k + p] = s.B.at(mid, mid + k);
            }
            // M and K are symmetric; make the Toeplitz row bitwise symmetric too (the
            // quadrature sums of row entries +k and -k can differ by rounding), so
            // kernels may use pair sums with p+1 distinct coefficients.
            for (int k = 1; k <= p; ++k) {
                rm[p + k] = rm[p - k] = 0.5 * (rm[p + k] + rm[p - k]);
                rk[p + k] = rk[p - k] = 0.5 * (rk[p + k] + rk[p - k]);
            }
            for (int i = lo; i <= hi; ++i)
                for (int k = -p; k <= p; ++k) {
                    s.M.at(i, i + k) = rm[k + p];
                    s.K.at(i, i + k) = rk[k + p];
                    s.B.at(i, i + k) = rb[k + p];
                }
        }
    }
    if (bc == 1) {
        // interior restriction (C3): the two end functions are removed
        for (int end : {0, s.n - 1})
            for (int j = end - p; j <= end + p; ++j) {
                if (j < 0 || j >= s.n) continue;
                s.M.at(end, j) = s.M.at(j, end) = 0.0;
                s.K.at(end, j) = s.K.at(j, end) = 0.0;
                s.B.at(end, j) = s.B.at(j, end) = 0.0;
            }
    }
    return 0;
}

void diff_weights(const Space1D &s, std::vector<double> &w) {
    const int n = s.n, p = s.p, W2 = 2 * p;
    w.assign((size_t)n * W2, 0.0);
    if (s.nel == 0) return;  // the 2D axis: K = 0
    for (int k = 0; k < n; ++k) {
        xreal wk[16] = {};
        xreal rs = 0;  // row sum of the band row
        for (int c = std::max(0, k - p); c <= std::min(n - 1, k + p); ++c) rs += (xreal)s.K.get(k, c);
        // sum_c K_kc (T_c - T_k): T_c - T_k = sum_{j=k}^{c-1} dT_j (c > k), -sum_{j=c}^{k-1} dT_j (c < k)
        for (int m = 0; m < W2; ++m) {
            const int j = k - p + m;
            xreal v = 0;
            if (j >= k)
                for (int c = j + 1; c <= k + p; ++c) v += (xreal)s.K.get(k, c);
            else
                for (int c = k - p; c <= j; ++c) v -= (xreal)s.K.get(k, c);
            wk[m] = v;
        }
        // + s_k T_k: zero except on Dirichlet rows that lost a column (|k - end| <= p), where T = 0
        // on the boundary function: T_k = sum_{j<k} dT_j (bottom) or -sum_{j>=k} dT_j (top)
        if (s.bc == 1 && k > 0 && k < n - 1 && (k <= p || k >= n - 1 - p)) {
            if (k <= p)
                for (int j = 0; j < k; ++j) wk[j - k + p] += rs;
            else
                for (int j = k; j <= n - 2; ++j) wk[j - k + p] -= rs;
        }
        for (int m = 0; m < W2; ++m) w[(size_t)k * W2 + m] = (double)wk[m];
    }
}

void trivial_space(int p, Space1D &s) {
    s.p = p;
    s.nel = 0;
    s.n = 1;
    s.bc = 0;
    s.knots.clear();
    s.M = Band(1, p);
    s.K = Band(1, p);
    s.B = Band(1, p);
    s.M.at(0, 0) = 1.0;
}

void load_vector(const Space1D &s, int func, double c, double sigma, double *out) {
    if (s.nel == 0) {  // the 2D axis: the load of any f(x, y) (x) 1 has the factor 1
        out[0] = 1.0;
        return;
    }
    const xreal kPi = 3.14159265358979323846264338327950288L;
    const std::vector<xreal> tx = knots_x(s.p, s.nel);
    xreal xg[8], wg[8], N[8], dN[8];
    gauss_legendre_t<xreal>(8, xg, wg);
    std::vector<xreal> acc(s.n, 0);
    const xreal cx = c, sx = sigma;
    for (int e = 0; e < s.nel; ++e) {
        int span = e + s.p;
        xreal a = tx[span], b = tx[span + 1];
        xreal half = (b - a) / 2, mid = (a + b) / 2;
        for (int q = 0; q < 8; ++q) {
            xreal x = mid + half * xg[q], w = half * wg[q];
            xreal f = (func == 0) ? std::sin(kPi * x) : std::exp(-(x - cx) * (x - cx) / (2 * sx * sx));
            basis_and_derivs_t<xreal>(tx.data(), s.p, span, x, N, dN);
            for (int r = 0; r <= s.p; ++r) acc[e + r] += w * f * N[r];
        }
    }
    for (int i = 0; i < s.n; ++i) out[i] = (double)acc[i];
    if (s.bc == 1) out[0] = out[s.n - 1] = 0.0;
}

// Row-wise Doolittle on band storage: row i of L and U from row i of A and the
// previous p rows of U (no pivoting).
static bool lu_row(const Band &A, std::vector<double> &Lw, std::vector<double> &Ur, int i, double amax) {
    const int n = A.n, p = A.p, W = 2 * p + 1;
    // L(i, j) for j in [i-p, i): stored Lw[i*p + (i-j-1)]
    for (int j = std::max(0, i - p); j < i; ++j) {
        double v = A.get(i, j);
        for (int m = std::max(0, i - p); m < j; ++m) v -= Lw[(size_t)i * p + (i - m - 1)] * Ur[(size_t)m * W + (j - m)];
        Lw[(size_t)i * p + (i - j - 1)] = v / Ur[(size_t)j * W + 0];
    }
    // U(i, j) for j in [i, i+p]: stored Ur[i*W + (j-i)]
    for (int j = i; j <= std::min(n - 1, i + p); ++j) {
        double v = A.get(i, j);
        for (int m = std::max(0, j - p); m < i; ++m) v -= Lw[(size_t)i * p + (i - m - 1)] * Ur[(size_t)m * W + (j - m)];
        Ur[(size_t)i * W + (j - i)] = v;
    }
    return std::fabs(Ur[(size_t)i * W]) >= 1e-14 * amax;
}

int banded_lu(const Band &A, LUFactors &f, bool freeze) {
    const int n = A.n, p = A.p, W = 2 * p + 1;
    f.n = n;
    f.p = p;
    f.i_lo = f.i_hi = 0;
    double amax = 0.0;
    for (double v : A.v) amax = std::max(amax, std::fabs(v));
    if (amax == 0.0) return -2;
    std::vector<double> Lw((size_t)n * p, 0.0), Ur((size_t)n * W, 0.0);
    for (int i = 0; i < n; ++i)
        if (!lu_row(A, Lw, Ur, i, amax)) return -2;

    auto row_close = [&](int a, int b) {
        for (int k = 0; k < p; ++k) {
            double x = Lw[(size_t)a * p + k], y = Lw[(size_t)b * p + k];
            if (std::fabs(x - y) > 4.5e-16 * std::max(std::fabs(x), std::fabs(y))) return false;
        }
        for (int k = 0; k <= p; ++k) {
            double x = Ur[(size_t)a * W + k], y = Ur[(size_t)b * W + k];
            if (std::fabs(x - y) > 4.5e-16 * std::max(std::fabs(x), std::fabs(y))) return false;
        }
        return true;
    };
    if (freeze && n > 4 * p + 8) {
        // A is Toeplitz on rows [2p, n-1-2p] (uniform mesh, host_setup build_space)
        const int a_hi = n - 1 - 2 * p;
        int i_lo = -1;
        for (int i = 2 * p + 1; i + p < a_hi; ++i) {
            bool ok = true;
            for (int q = i - p; q < i && ok; ++q) ok = row_close(q, i);
            if (ok) { i_lo = i; break; }
        }
        int i_hi = a_hi - p;  // rows >= i_hi are recomputed from the frozen rows
        if (i_lo > 0 && i_hi - i_lo > 2 * p) {
            std::vector<double> L2 = Lw, U2 = Ur;
            for (int i = i_lo + 1; i < i_hi; ++i) {
                for (int k = 0; k < p; ++k) L2[(size_t)i * p + k] = Lw[(size_t)i_lo * p + k];
                for (int k = 0; k < W; ++k) U2[(size_t)i * W + k] = Ur[(size_t)i_lo * W + k];
            }
            bool ok = true;
            for (int i = i_hi; i < n && ok; ++i) ok = lu_row(A, L2, U2, i, amax);
            // residual of the frozen factorisation over the band
            double res = 0.0;
            for (int i = 0; i < n && ok; ++i)
                for (int j = std::max(0, i - p); j <= std::min(n - 1, i + p); ++j) {
                    double s = 0.0;
                    for (int m = std::max(0, std::max(i, j) - p); m <= std::min(i, j); ++m) {
                        double lim = (m == i) ? 1.0 : L2[(size_t)i * p + (i - m - 1)];
                        s += lim * U2[(size_t)m * W + (j - m)];
                    }
                    res = std::max(res, std::fabs(s - A.get(i, j)));
                }
            if (ok && res <= 1e-14 * amax) {
                Lw.swap(L2);
                Ur.swap(U2);
                f.i_lo = i_lo;
                f.i_hi = i_hi;
                f.residual = res / amax;
            }
        }
    }
    f.l.assign((size_t)n * p, 0.0);
    f.us.assign((size_t)n * p, 0.0);
    f.dinv.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double d = Ur[(size_t)i * W];
        f.dinv[i] = 1.0 / d;
        for (int k = 1; k <= p; ++k) {
            if (i - k >= 0) f.l[(size_t)i * p + k - 1] = Lw[(size_t)i * p + (k - 1)];
            if (i + k < n) f.us[(size_t)i * p + k - 1] = Ur[(size_t)i * W + k] / d;
        }
    }
    if (f.i_hi > f.i_lo) {
        // the frozen rows of us/dinv must be bitwise uniform too
        for (int i = f.i_lo + 1; i < f.i_hi; ++i) {
            f.dinv[i] = f.dinv[f.i_lo];
            for (int k = 0; k < p; ++k) f.us[(size_t)i * p + k] = f.us[(size_t)f.i_lo * p + k];
        }
    }
    return 0;
}

void lu_solve_host(const LUFactors &f, double *x) {
    const int n = f.n, p = f.p;
    for (int i = 0; i < n; ++i)
        for (int k = 1; k <= p && i - k >= 0; ++k) x[i] -= f.l[(size_t)i * p + k - 1] * x[i - k];
    for (int i = n - 1; i >= 0; --i) {
        double v = x[i] * f.dinv[i];
        for (int k = 1; k <= p && i + k < n; ++k) v -= f.us[(size_t)i * p + k - 1] * x[i + k];
        x[i] = v;
    }
}

int choose_chunk_len(int n, int p, int C) {
    for (int L : kChunkLens)
        if ((long)L * C >= n && L >= p) return L;
    return 0;
}

static double inf_norm(const std::vector<double> &A, int p) {
    double m = 0.0;
    for (int a = 0; a < p; ++a) {
        double r = 0.0;
        for (int b = 0; b < p; ++b) r += std::fabs(A[a * p + b]);
        m = std::max(m, r);
    }
    return m;
}

// smallest k such that every product of k consecutive maps (in chain order) has
// inf-norm < 2^-64; C-1 if none.  fwd: Tf_{c-1}...Tf_{c-k}; bwd: Rb_{c+1}...Rb_{c+k}.
static int truncation_depth(const std::vector<double> &T, int C, int p, bool fwd) {
    const double thr = std::ldexp(1.0, -64);
    std::vector<double> acc(p * p), tmp(p * p);
    for (int k = 1; k < C; ++k) {
        bool ok = true;
        for (int c0 = 0; c0 + k <= C && ok; ++c0) {
            // chunks c0 .. c0+k-1, newest applied last (fwd) / first (bwd)
            for (int a = 0; a < p * p; ++a) acc[a] = (a % (p + 1) == 0) ? 1.0 : 0.0;
            for (int q = 0; q < k; ++q) {
                const int cc = fwd ? c0 + q : c0 + k - 1 - q;
                const double *M = &T[(size_t)cc * p * p];
                for (int a = 0; a < p; ++a)
                    for (int b = 0; b < p; ++b) {
                        double v = 0.0;
                        for (int m = 0; m < p; ++m) v += M[a * p + m] * acc[m * p + b];
                        tmp[a * p + b] = v;
                    }
                acc.swap(tmp);
            }
            ok = inf_norm(acc, p) < thr;
        }
        if (ok) return k;
    }
    return std::max(C - 1, 0);
}

void build_part_tables(const LUFactors &f, int C, int L, PartTables &t) {
    const int n = f.n, p = f.p;
    t.n = n;
    t.p = p;
    t.C = C;
    t.L = L;
    t.gf.assign((size_t)n * p, 0.0);
    t.gb.assign((size_t)n * p, 0.0);
    std::vector<double> y(n + 2 * p);
    for (int c = 0; c < C; ++c) {
        int s = c * L, e = std::min(n, s + L);
        for (int m = 0; m < p; ++m) {
            // forward homogeneous recurrence with incoming y_{s-1-m} = 1
            std::fill(y.begin(), y.end(), 0.0);
            double *Y = y.data() + p;  // Y[i] for i >= -p
            if (s - 1 - m >= -p) Y[s - 1 - m] = 1.0;
            for (int i = s; i < e; ++i) {
                double v = 0.0;
                for (int k = 1; k <= p; ++k)
                    if (i - k >= s - p) v -= f.l[(size_t)i * p + k - 1] * Y[i - k];
                Y[i] = v;
                t.gf[(size_t)i * p + m] = v;
            }
            // backward homogeneous recurrence with incoming x_{e+m} = 1
            std::fill(y.begin(), y.end(), 0.0);
            Y = y.data();
            if (e + m < n + p) Y[e + m] = 1.0;
            for (int i = e - 1; i >= s; --i) {
                double v = 0.0;
                for (int k = 1; k <= p; ++k)
                    if (i + k < n + p) v -= (i + k < n ? f.us[(size_t)i * p + k - 1] : 0.0) * Y[i + k];
                Y[i] = v;
                t.gb[(size_t)i * p + m] = v;
            }
        }
    }
    t.Tf.assign((size_t)C * p * p, 0.0);
    t.Rb.assign((size_t)C * p * p, 0.0);
    for (int c = 0; c < C; ++c) {
        int s = c * L, e = std::min(n, s + L);
        if (e - s < p) continue;  // only the padded tail can be short; its maps stay 0
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b) {
                t.Tf[((size_t)c * p + a) * p + b] = t.gf[(size_t)(e - 1 - a) * p + b];
                t.Rb[((size_t)c * p + a) * p + b] = t.gb[(size_t)(s + a) * p + b];
            }
    }
    t.Kf = truncation_depth(t.Tf, C, p, true);
    t.Kb = truncation_depth(t.Rb, C, p, false);
}

}  // namespace ads

namespace ads {

void slab_plan(int n, int G, std::vector<int> &z0, std::vector<int> &nl) {
    z0.assign(G, 0);
    nl.assign(G, 0);
    int at = 0;
    for (int j = 0; j < G; ++j) {
        nl[j] = n / G + (j < n % G ? 1 : 0);
        z0[j] = at;
        at += nl[j];
    }
}

int build_slab_spikes(const Band &A, int z0, int nl, SlabSpikes &s) {
    const int p = A.p, n = A.n, z1 = z0 + nl;
    s.block = Band(nl, p);
    for (int i = 0; i < nl; ++i)
        for (int j = i - p; j <= i + p; ++j)
            if (j >= 0 && j < nl) s.block.at(i, j) = A.get(z0 + i, z0 + j);
    if (banded_lu(s.block, s.lu)) return -2;
    s.V.assign((size_t)nl * p, 0.0);
    s.W.assign((size_t)nl * p, 0.0);
    std::vector<double> col(nl);
    for (int b = 0; b < p; ++b) {
        // V column b: rhs rows nl-p+a hold B(a, b) = A(z1 - p + a, z1 + b)
        std::fill(col.begin(), col.end(), 0.0);
        for (int a = 0; a < p; ++a)
            if (nl - p + a >= 0 && z1 + b < n) col[nl - p + a] = A.get(z1 - p + a, z1 + b);
        lu_solve_host(s.lu, col.data());
        for (int i = 0; i < nl; ++i) s.V[(size_t)i * p + b] = col[i];
        // W column b: rhs rows a hold C(a, b) = A(z0 + a, z0 - p + b)
        std::fill(col.begin(), col.end(), 0.0);
        for (int a = 0; a < p; ++a)
            if (a < nl && z0 - p + b >= 0) col[a] = A.get(z0 + a, z0 - p + b);
        lu_solve_host(s.lu, col.data());
        for (int i = 0; i < nl; ++i) s.W[(size_t)i * p + b] = col[i];
    }
    return 0;
}

double interface_inverse(const SlabSpikes &sj, const SlabSpikes &sj1, int p, std::vector<double> &Q) {
    const int nl = sj.block.n, m = 2 * p;
    std::vector<double> S((size_t)m * m, 0.0);
    for (int a = 0; a < p; ++a) {
        S[a * m + a] = 1.0;
        S[(p + a) * m + p + a] = 1.0;
        for (int b = 0; b < p; ++b) {
            S[a * m + p + b] = sj.V[(size_t)(nl - p + a) * p + b];  // Vbot_j
            S[(p + a) * m + b] = sj1.W[(size_t)a * p + b];          // Wtop_{j+1}
        }
    }
    // Gauss-Jordan with partial pivoting (2p <= 10)
    Q.assign((size_t)m * m, 0.0);
    for (int a = 0; a < m; ++a) Q[a * m + a] = 1.0;
    for (int c = 0; c < m; ++c) {
        int piv = c;
        for (int r = c + 1; r < m; ++r)
            if (std::fabs(S[r * m + c]) > std::fabs(S[piv * m + c])) piv = r;
        for (int k = 0; k < m; ++k) {
            std::swap(S[c * m + k], S[piv * m + k]);
            std::swap(Q[c * m + k], Q[piv * m + k]);
        }
        const double d = S[c * m + c];
        for (int k = 0; k < m; ++k) {
            S[c * m + k] /= d;
            Q[c * m + k] /= d;
        }
        for (int r = 0; r < m; ++r)
            if (r != c) {
                const double f = S[r * m + c];
                for (int k = 0; k < m; ++k) {
                    S[r * m + k] -= f * S[c * m + k];
                    Q[r * m + k] -= f * Q[c * m + k];
                }
            }
    }
    // dropped couplings: W_j bottom p rows (slab j's own W) and V_{j+1} top p rows
    double dropped = 0.0;
    const int nl1 = sj1.block.n;
    for (int a = 0; a < p; ++a)
        for (int b = 0; b < p; ++b) {
            dropped = std::max(dropped, std::fabs(sj.W[(size_t)(nl - p + a) * p + b]));
            if (a < nl1) dropped = std::max(dropped, std::fabs(sj1.V[(size_t)a * p + b]));
        }
    return dropped;
}

}  // namespace ads

namespace ads {

// ---- modal (fast-diagonalisation) basis of one direction ----
// Symmetric tridiagonal reduction by Householder reflections, accumulated into Zt (row r of Zt is
// column r of the orthogonal factor): C = Z T Z^T with T = tridiag(e, d, e).
static void householder_tridiag(std::vector<double> &C, int n, std::vector<double> &Zt, std::vector<double> &d,
                                std::vector<double> &e) {
    Zt.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) Zt[(size_t)i * n + i] = 1.0;
    std::vector<double> v(n), pv(n);
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;  // reflector acts on indices k+1 .. n-1
        double nx = 0.0;
        for (int i = 0; i < m; ++i) nx = std::hypot(nx, C[(size_t)(k + 1 + i) * n + k]);
        if (nx == 0.0) continue;
        const double x0 = C[(size_t)(k + 1) * n + k];
        const double alpha = x0 > 0 ? -nx : nx;  // reflected column becomes alpha e_1
        for (int i = 0; i < m; ++i) v[i] = C[(size_t)(k + 1 + i) * n + k];
        v[0] -= alpha;
        double nv = 0.0;
        for (int i = 0; i < m; ++i) nv = std::hypot(nv, v[i]);
        for (int i = 0; i < m; ++i) v[i] /= nv;
        // H = I - 2 v v^T on the trailing block: C <- H C H = C - 2 v w^T - 2 w v^T,
        // w = p - (v^T p) v, p = C v
        double vp = 0.0;
        for (int i = 0; i < m; ++i) {
            double s = 0.0;
            const double *row = &C[(size_t)(k + 1 + i) * n + k + 1];
            for (int j = 0; j < m; ++j) s += row[j] * v[j];
            pv[i] = s;
            vp += v[i] * s;
        }
        for (int i = 0; i < m; ++i) pv[i] -= vp * v[i];
        for (int i = 0; i < m; ++i) {
            double *row = &C[(size_t)(k + 1 + i) * n + k + 1];
            for (int j = 0; j < m; ++j) row[j] -= 2.0 * (v[i] * pv[j] + pv[i] * v[j]);
        }
        for (int i = 0; i < m; ++i) C[(size_t)(k + 1 + i) * n + k] = C[(size_t)k * n + k + 1 + i] = 0.0;
        C[(size_t)(k + 1) * n + k] = C[(size_t)k * n + k + 1] = alpha;
        // Z <- Z H: column j of Z (row j of Zt) for j in k+1..n-1 mixes by v
        for (int r = 0; r < n; ++r) {  // row r of Z: z_r <- z_r - 2 (z_r . v) v^T on those columns
            double s = 0.0;
            for (int i = 0; i < m; ++i) s += Zt[(size_t)(k + 1 + i) * n + r] * v[i];
            for (int i = 0; i < m; ++i) Zt[(size_t)(k + 1 + i) * n + r] -= 2.0 * s * v[i];
        }
    }
    d.resize(n);
    e.assign(n, 0.0);
    for (int i = 0; i < n; ++i) d[i] = C[(size_t)i * n + i];
    for (int i = 0; i + 1 < n; ++i) e[i] = C[(size_t)(i + 1) * n + i];
}

// Eigenvalues of tridiag(e, d, e) by implicit QL sweeps with Wilkinson-type shifts; the plane
// rotations are accumulated into the rows of Zt (the eigenvector basis).  Returns 0 or -1.
static int tridiag_ql(std::vector<double> &d, std::vector<double> &e, std::vector<double> &Zt, int n) {
    const double eps = std::numeric_limits<double>::epsilon();
    for (int l = 0; l < n; ++l) {
        for (int iter = 0;; ++iter) {
            int m = l;
            for (; m + 1 < n; ++m)  // first negligible coupling at or after l
                if (std::fabs(e[m]) <= eps * (std::fabs(d[m]) + std::fabs(d[m + 1]))) break;
            if (m == l) break;
            if (iter == 60) return -1;
            // shift from the leading 2x2 block at l
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = std::hypot(g, 1.0);
            g = d[m] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
            double s = 1.0, c = 1.0, pshift = 0.0;
            bool deflated = false;
            for (int i = m - 1; i >= l; --i) {
                const double f = s * e[i], b = c * e[i];
                r = std::hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {  // underflow: the block splits here
                    d[i + 1] -= pshift;
                    e[m] = 0.0;
                    deflated = true;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[i + 1] - pshift;
                r = (d[i] - g) * s + 2.0 * c * b;
                pshift = s * r;
                d[i + 1] = g + pshift;
                g = c * r - b;
                double *zi = &Zt[(size_t)i * n], *zj = &Zt[(size_t)(i + 1) * n];
                for (int k = 0; k < n; ++k) {
                    const double t = zj[k];
                    zj[k] = s * zi[k] + c * t;
                    zi[k] = c * zi[k] - s * t;
                }
            }
            if (deflated) continue;
            d[l] -= pshift;
            e[l] = g;
            e[m] = 0.0;
        }
    }
    return 0;
}

// K phi = lambda M phi for dense symmetric na x na matrices (M positive definite): Cholesky
// M = L L^T, C = L^-1 K L^-T, Householder tridiagonalisation, implicit QL, Phi = L^-T Z.
static int gen_eig_dense(int na, std::vector<double> L, std::vector<double> X, std::vector<double> &lam,
                         std::vector<double> &phi) {
    struct { int p; } s{na};  // no band structure assumed
    for (int j = 0; j < na; ++j) {
        double dj = L[(size_t)j * na + j];
        for (int k = std::max(0, j - s.p); k < j; ++k) dj -= L[(size_t)j * na + k] * L[(size_t)j * na + k];
        if (!(dj > 0.0)) return -1;
        dj = std::sqrt(dj);
        L[(size_t)j * na + j] = dj;
        for (int i = j + 1; i < std::min(na, j + s.p + 1); ++i) {  // the factor keeps M's band
            double v = L[(size_t)i * na + j];
            for (int k = std::max(0, i - s.p); k < j; ++k) v -= L[(size_t)i * na + k] * L[(size_t)j * na + k];
            L[(size_t)i * na + j] = v / dj;
        }
        for (int i = j + s.p + 1; i < na; ++i) L[(size_t)i * na + j] = 0.0;
    }
    for (int i = 0; i < na; ++i)
        for (int j = i + 1; j < na; ++j) L[(size_t)i * na + j] = 0.0;
    // C = L^-1 K L^-T: X <- L^-1 K (columns), then C = L^-1 X^T
    auto lower_solve_cols = [&](std::vector<double> &B) {  // B <- L^-1 B, column by column
        for (int c = 0; c < na; ++c)
            for (int i = 0; i < na; ++i) {
                double v = B[(size_t)i * na + c];
                for (int k = std::max(0, i - s.p); k < i; ++k) v -= L[(size_t)i * na + k] * B[(size_t)k * na + c];
                B[(size_t)i * na + c] = v / L[(size_t)i * na + i];
            }
    };
    lower_solve_cols(X);
    std::vector<double> C((size_t)na * na);
    for (int i = 0; i < na; ++i)
        for (int j = 0; j < na; ++j) C[(size_t)i * na + j] = X[(size_t)j * na + i];
    lower_solve_cols(C);
    for (int i = 0; i < na; ++i)
        for (int j = i + 1; j < na; ++j) {
            const double a = 0.5 * (C[(size_t)i * na + j] + C[(size_t)j * na + i]);
            C[(size_t)i * na + j] = C[(size_t)j * na + i] = a;
        }
    std::vector<double> Zt, d, e;
    householder_tridiag(C, na, Zt, d, e);
    if (tridiag_ql(d, e, Zt, na)) return -1;
    // Phi = L^-T Z (back substitution per eigenvector), eigenpairs in ascending order
    std::vector<int> ord(na);
    for (int i = 0; i < na; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](int a, int b) { return d[a] < d[b]; });
    lam.resize(na);
    phi.assign((size_t)na * na, 0.0);
    std::vector<double> z(na);
    for (int kk = 0; kk < na; ++kk) {
        const int k = ord[kk];
        lam[kk] = d[k];
        for (int i = 0; i < na; ++i) z[i] = Zt[(size_t)k * na + i];
        for (int i = na - 1; i >= 0; --i) {
            double v = z[i];
            for (int r = i + 1; r < std::min(na, i + s.p + 1); ++r) v -= L[(size_t)r * na + i] * z[r];
            z[i] = v / L[(size_t)i * na + i];
        }
        for (int i = 0; i < na; ++i) phi[(size_t)i * na + kk] = z[i];
    }
    return 0;
}


int modal_basis(const Space1D &s, std::vector<double> &lam, std::vector<double> &phi, std::vector<int> *parity) {
    const int o = s.bc == 1 ? 1 : 0, na = s.n - 2 * o;
    if (na <= 0) return -1;
    // the uniform open knot vector is mirror-symmetric, so M and K (active block) commute with the
    // reversal J: the pencil splits into an even block on (u + Ju) and an odd block on (u - Ju),
    // each solved on its own -- every eigenvector has an exact parity (needed by the folded
    // modal transforms) and each eigensolve is half the size
    const int hb = na / 2, Hb = hb + (na & 1);
    const double r2 = std::sqrt(0.5);
    std::vector<double> M((size_t)na * na), K((size_t)na * na);
    for (int i = 0; i < na; ++i)
        for (int j = 0; j < na; ++j) {
            M[(size_t)i * na + j] = s.M.get(i + o, j + o);
            K[(size_t)i * na + j] = s.K.get(i + o, j + o);
        }
    struct Part { std::vector<double> lam, phi; int m, sign; };
    Part parts[2] = {{{}, {}, Hb, 1}, {{}, {}, hb, -1}};
    for (Part &pt : parts) {
        const int m = pt.m;
        if (m == 0) continue;
        // basis columns: b_i = (e_i + sign e_{na-1-i}) / sqrt 2 (i < hb), the middle e_hb (even, odd na)
        auto B = [&](int r, int i) {  // entry r of basis vector i
            if (i == hb) return r == hb ? 1.0 : 0.0;
            return (r == i ? r2 : 0.0) + (r == na - 1 - i ? pt.sign * r2 : 0.0);
        };
        std::vector<double> Mp((size_t)m * m), Kp((size_t)m * m);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                const int ri[2] = {i, na - 1 - i}, rj[2] = {j, na - 1 - j};
                double vm = 0.0, vk = 0.0;
                for (int a = 0; a < (i == hb ? 1 : 2); ++a)
                    for (int b = 0; b < (j == hb ? 1 : 2); ++b) {
                        const double w = B(ri[a], i) * B(rj[b], j);
                        vm += w * M[(size_t)ri[a] * na + rj[b]];
                        vk += w * K[(size_t)ri[a] * na + rj[b]];
                    }
                Mp[(size_t)i * m + j] = vm;
                Kp[(size_t)i * m + j] = vk;
            }
        std::vector<double> ph;
        if (gen_eig_dense(m, Mp, Kp, pt.lam, ph)) return -1;
        pt.phi.assign((size_t)na * m, 0.0);  // full eigenvectors phi = B ph, [na][m]
        for (int k = 0; k < m; ++k)
            for (int i = 0; i < m; ++i) {
                const double c = ph[(size_t)i * m + k];
                if (i == hb) {
                    pt.phi[(size_t)hb * m + k] += c;
                } else {
                    pt.phi[(size_t)i * m + k] += r2 * c;
                    pt.phi[(size_t)(na - 1 - i) * m + k] += pt.sign * r2 * c;
                }
            }
    }
    // merge in ascending eigenvalue order
    std::vector<std::pair<double, std::pair<int, int>>> all;
    for (int q = 0; q < 2; ++q)
        for (int k = 0; k < parts[q].m; ++k) all.push_back({parts[q].lam[k], {q, k}});
    std::sort(all.begin(), all.end());
    lam.resize(na);
    phi.assign((size_t)na * na, 0.0);
    if (parity) parity->resize(na);
    for (int c = 0; c < na; ++c) {
        const int q = all[c].second.first, k = all[c].second.second;
        lam[c] = all[c].first;
        for (int i = 0; i < na; ++i) phi[(size_t)i * na + c] = parts[q].phi[(size_t)i * parts[q].m + k];
        if (parity) (*parity)[c] = parts[q].sign;
    }
    return 0;
}

}  // namespace ads
