/*
 * ads_oracle.c -- plain, slow, single-threaded fp64 CPU ORACLE for the
 * alternating-direction-split (ADS) isogeometric wave step of
 * Łoś, Behnoudfar, Paszyński, Calo, arXiv:1911.08158 ("the paper", PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this code.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_1911_08158_b200/), and never includes or links it.
 *
 * Style: every operation is written out as its definition, in the paper's
 * order and notation, with dense 1D matrices and band-limited loops
 * ("M_ij = 0 <=> |i-j| > p").  No blocking, no fusion, no
 * reordering beyond what the definitions state.  Compile with
 * -O2 -ffp-contract=off (no FMA contraction).
 *
 * Readings of the paper taken here (all listed in DESIGN.md §3):
 *   R1  time scheme: PAPER.md:143-147 (Eq. 16) with the velocity increment
 *       tau*Udd (not tau/2*Udd); equivalently the paper's own three-level form
 *       PAPER.md:426 with Upsilon -> K.  SURVEY.md §8(c) C1.
 *   R0  the literal Eq. 16 is kept behind scheme=0 to document the garble.
 *   C2  half-kick start a0 = D^-1 (F(0) - K u0), V0 = udot0 + tau/2 a0.
 *   C3  zero Dirichlet = interior restriction of each 1D space; arrays keep
 *       the boundary DOFs (always 0).
 *   C4  p+1 Gauss points per element for Gram matrices, 8 for load vectors.
 *   C5  3D: K = Kx(x)My(x)Mz + Mx(x)Ky(x)Mz + Mx(x)My(x)Kz, D = Ax(x)Ay(x)Az.
 *   C6  energies: kinetic 1/2 v'Mv (v = V - tau/2 a), potential 1/2 U'KU,
 *       invariant 1/2 V'DV + 1/2 U_n' K U_{n+1}.
 *   C10/C11/C12  3D elasticity blocks from the weak form PAPER.md:307-361,
 *       alternating-triangular split PAPER.md:388-405 applied to the
 *       increment (predictor/corrector PAPER.md:406-414 rewritten in delta
 *       form), per-component Kronecker split PAPER.md:415-422.
 *   C14 time levels: F evaluated at t_{n+1} = (n+1)*tau, Ricker wavelet.
 *
 * Pins (tests/test_oracle_pins.py): SPEC p=1 fixtures, cardinal B-spline
 * closed-form interior rows, scipy-BSpline brute-force assembly, dense
 * Kronecker solve/apply, brute-force 3D quadrature stiffness and elasticity,
 * modal closed form (oracle/modal.py), exact discrete
 * energy invariant, work identity, PDE eigenmode accuracy and order 2.
 *
 * Arithmetic type: `real` is double (the oracle proper, libads_oracle.so).  The same source
 * compiled with -DOR_LONG_DOUBLE (libads_oracle_ld.so) runs every step in x87 extended precision
 * (64-bit significand): the truth reference the GPU's one-step fp64 bound is measured against
 * (north_star "relative L2 <= 1e-12 after one step"; T1).  <tgmath.h> makes sin, cos,
 * exp, fabs follow the argument type; the double build is bitwise the oracle it always was.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <tgmath.h>

#ifdef OR_LONG_DOUBLE
typedef long double real;
#else
typedef double real;
#endif

#define OR_OK 0
#define OR_E_INVAL (-1)
#define OR_E_SINGULAR (-2)
#define OR_E_NOMEM (-5)

/* ------------------------------------------------------------------------ */
/* 1D open uniform B-spline space on [0,1] */
/* ------------------------------------------------------------------------ */

int or_nbasis(int p, int nel) { return nel + p; }

/* Open (clamped) uniform knot vector: p+1 zeros, interior e/nel, p+1 ones.
 * Length nel + 2p + 1. */
void or_knots(int p, int nel, real *t) {
    int m = nel + 2 * p + 1;
    for (int i = 0; i < m; ++i) {
        if (i <= p) t[i] = 0.0;
        else if (i >= nel + p) t[i] = 1.0;
        else t[i] = (real)(i - p) / (real)nel;
    }
}

/* Cox-de Boor recursion, written as the definition:
 *   N_{i,0}(x) = 1 if t_i <= x < t_{i+1} else 0
 *   N_{i,q}(x) = (x - t_i)/(t_{i+q} - t_i) N_{i,q-1}(x)
 *              + (t_{i+q+1} - x)/(t_{i+q+1} - t_{i+1}) N_{i+1,q-1}(x)
 * with 0/0 := 0.  Only evaluated at points strictly inside elements. */
real or_bspline(const real *t, int i, int q, real x) {
    if (q == 0) return (t[i] <= x && x < t[i + 1]) ? 1.0 : 0.0;
    real a = 0.0, b = 0.0;
    real d1 = t[i + q] - t[i];
    real d2 = t[i + q + 1] - t[i + 1];
    if (d1 > 0.0) a = (x - t[i]) / d1 * or_bspline(t, i, q - 1, x);
    if (d2 > 0.0) b = (t[i + q + 1] - x) / d2 * or_bspline(t, i + 1, q - 1, x);
    return a + b;
}

/* Derivative: N'_{i,q} = q/(t_{i+q}-t_i) N_{i,q-1} - q/(t_{i+q+1}-t_{i+1}) N_{i+1,q-1}. */
real or_bspline_d(const real *t, int i, int q, real x) {
    if (q == 0) return 0.0;
    real a = 0.0, b = 0.0;
    real d1 = t[i + q] - t[i];
    real d2 = t[i + q + 1] - t[i + 1];
    if (d1 > 0.0) a = (real)q / d1 * or_bspline(t, i, q - 1, x);
    if (d2 > 0.0) b = (real)q / d2 * or_bspline(t, i + 1, q - 1, x);
    return a - b;
}

/* Gauss-Legendre rule with m points on [-1,1]: Newton iteration on P_m. */
void or_gauss(int m, real *xi, real *w) {
    const real pi = (real)3.14159265358979323846264338327950288L;
    for (int k = 0; k < m; ++k) {
        real x = cos(pi * (k + 0.75) / (m + 0.5));
        real dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            real p0 = 1.0, p1 = x;
            for (int j = 2; j <= m; ++j) {
                real p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            if (m == 1) { p1 = x; p0 = 1.0; }
            dp = m * (x * p1 - p0) / (x * x - 1.0);
            real dx = p1 / dp;
            x -= dx;
            if (fabs(dx) < 1e-16) break;
        }
        {
            real p0 = 1.0, p1 = x;
            for (int j = 2; j <= m; ++j) {
                real p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j;
                p0 = p1;
                p1 = p2;
            }
            if (m == 1) { p1 = x; p0 = 1.0; }
            dp = m * (x * p1 - p0) / (x * x - 1.0);
        }
        xi[k] = x;
        w[k] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
}

/* ------------------------------------------------------------------------ */
/* 1D Gram matrices (Eq. 13; mixed B PAPER.md:381-387)      */
/*   M(a,c) = int N_a N_c,  K(a,c) = int N'_a N'_c,  B(a,c) = int N'_a N_c   */
/* dense row-major n x n; p+1 Gauss points per element (exact, C4).          */
/* bc = 1: zero Dirichlet -> rows/cols of the two end functions zeroed (C3). */
/* ------------------------------------------------------------------------ */
int or_matrices_1d(int p, int nel, int bc, real *M, real *K, real *B) {
    if (p < 1 || nel < 0) return OR_E_INVAL;
    if (nel == 0) {  /* the 2D scheme's third axis: one function, M = 1, K = B = 0 (see or_pw_create) */
        M[0] = 1.0; K[0] = 0.0;
        if (B) B[0] = 0.0;
        return OR_OK;
    }
    int n = nel + p;
    real *t = (real *)malloc(sizeof(real) * (nel + 2 * p + 1));
    real xi[16], wq[16];
    or_knots(p, nel, t);
    or_gauss(p + 1, xi, wq);
    memset(M, 0, sizeof(real) * n * n);
    memset(K, 0, sizeof(real) * n * n);
    if (B) memset(B, 0, sizeof(real) * n * n);
    for (int e = 0; e < nel; ++e) {
        real xa = t[p + e], xb = t[p + e + 1];
        real J = 0.5 * (xb - xa);
        for (int q = 0; q <= p; ++q) {
            real x = 0.5 * (xa + xb) + J * xi[q];
            real w = J * wq[q];
            for (int a = e; a <= e + p; ++a) {
                real Na = or_bspline(t, a, p, x), dNa = or_bspline_d(t, a, p, x);
                for (int c = e; c <= e + p; ++c) {
                    real Nc = or_bspline(t, c, p, x), dNc = or_bspline_d(t, c, p, x);
                    M[a * n + c] += w * Na * Nc;
                    K[a * n + c] += w * dNa * dNc;
                    if (B) B[a * n + c] += w * dNa * Nc;
                }
            }
        }
    }
    if (bc == 1) {
        for (int i = 0; i < n; ++i) {
            int ends[2] = {0, n - 1};
            for (int s = 0; s < 2; ++s) {
                int b = ends[s];
                M[b * n + i] = M[i * n + b] = 0.0;
                K[b * n + i] = K[i * n + b] = 0.0;
                if (B) B[b * n + i] = B[i * n + b] = 0.0;
            }
        }
    }
    free(t);
    return OR_OK;
}

/* 1D load vector b_a = int f(x) N_a(x) dx, 8 Gauss points per element (C4).
 * kind 0: f = sin(pi x); kind 1: f = exp(-(x-c)^2/(2 sigma^2)). */
int or_load_1d(int p, int nel, int bc, int kind, real c, real sigma, real *b) {
    const real pi = (real)3.14159265358979323846264338327950288L;
    int n = nel + p;
    real *t = (real *)malloc(sizeof(real) * (nel + 2 * p + 1));
    real xi[8], wq[8];
    or_knots(p, nel, t);
    or_gauss(8, xi, wq);
    memset(b, 0, sizeof(real) * n);
    for (int e = 0; e < nel; ++e) {
        real xa = t[p + e], xb = t[p + e + 1];
        real J = 0.5 * (xb - xa);
        for (int q = 0; q < 8; ++q) {
            real x = 0.5 * (xa + xb) + J * xi[q];
            real w = J * wq[q];
            real f;
            if (kind == 0) f = sin(pi * x);
            else f = exp(-(x - c) * (x - c) / (2.0 * sigma * sigma));
            for (int a = e; a <= e + p; ++a) b[a] += w * f * or_bspline(t, a, p, x);
        }
    }
    if (bc == 1) { b[0] = 0.0; b[n - 1] = 0.0; }
    free(t);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Banded LU without pivoting.               */
/* In place on a dense n x n matrix, loops restricted to |i-j| <= p.         */
/* L is unit lower (stored below the diagonal), U on and above.             */
/* Singular guard: pivot < 1e-14 * max|A| -> OR_E_SINGULAR.   */
/* ------------------------------------------------------------------------ */
int or_banded_lu(int n, int p, real *A) {
    real amax = 0.0;
    for (int i = 0; i < n * n; ++i) if (fabs(A[i]) > amax) amax = fabs(A[i]);
    for (int k = 0; k < n; ++k) {
        real piv = A[k * n + k];
        if (!(fabs(piv) >= 1e-14 * amax) || amax == 0.0) return OR_E_SINGULAR;
        int iend = (k + p < n - 1) ? k + p : n - 1;
        for (int i = k + 1; i <= iend; ++i) {
            real l = A[i * n + k] / piv;
            A[i * n + k] = l;
            for (int j = k + 1; j <= iend; ++j) A[i * n + j] -= l * A[k * n + j];
        }
    }
    return OR_OK;
}

/* Solve (LU) x = r in place for one vector with stride s. */
static void lu_solve_strided(int n, int p, const real *LU, real *x, long s) {
    for (int i = 0; i < n; ++i) {           /* forward: L y = r */
        real acc = x[i * s];
        int j0 = (i - p > 0) ? i - p : 0;
        for (int j = j0; j < i; ++j) acc -= LU[i * n + j] * x[j * s];
        x[i * s] = acc;
    }
    for (int i = n - 1; i >= 0; --i) {      /* backward: U x = y */
        real acc = x[i * s];
        int j1 = (i + p < n - 1) ? i + p : n - 1;
        for (int j = i + 1; j <= j1; ++j) acc -= LU[i * n + j] * x[j * s];
        x[i * s] = acc / LU[i * n + i];
    }
}

void or_lu_solve(int n, int p, const real *LU, real *x) { lu_solve_strided(n, p, LU, x, 1); }

/* ------------------------------------------------------------------------ */
/* 3D tensor algebra on x-fastest arrays u[(k*ny + j)*nx + i]                */
/* ------------------------------------------------------------------------ */

/* out = (A acting along `axis`) in, A dense na x na with band p.
 * This is the action of I(x)..(x)A(x)..(x)I on the vectorised tensor. */
static void mode_apply(const int n[3], int axis, const real *A, int p, const real *in, real *out) {
    int na = n[axis];
    long stride = (axis == 0) ? 1 : (axis == 1) ? (long)n[0] : (long)n[0] * n[1];
    for (int k = 0; k < n[2]; ++k)
        for (int j = 0; j < n[1]; ++j)
            for (int i = 0; i < n[0]; ++i) {
                long base = ((long)k * n[1] + j) * n[0] + i;
                int r = (axis == 0) ? i : (axis == 1) ? j : k;
                long line0 = base - (long)r * stride;
                int c0 = (r - p > 0) ? r - p : 0, c1 = (r + p < na - 1) ? r + p : na - 1;
                real acc = 0.0;
                for (int c = c0; c <= c1; ++c) acc += A[r * na + c] * in[line0 + (long)c * stride];
                out[base] = acc;
            }
}

/* out += coef * (Ax (x) Ay (x) Az) in      (three mode products) */
static void kron3_acc(const int n[3], int p, const real *Ax, const real *Ay, const real *Az,
                      real coef, const real *in, real *out, real *t1, real *t2) {
    long N = (long)n[0] * n[1] * n[2];
    mode_apply(n, 0, Ax, p, in, t1);
    mode_apply(n, 1, Ay, p, t1, t2);
    mode_apply(n, 2, Az, p, t2, t1);
    for (long q = 0; q < N; ++q) out[q] += coef * t1[q];
}

/* x <- (A_x (x) A_y (x) A_z)^{-1} x by the Appendix's three multi-RHS sweeps
 * (PAPER.md:533-618): solve along x for all (j,k), then y, then z. */
static void kron3_solve(const int n[3], int p, real *const LU[3], real *x) {
    for (int k = 0; k < n[2]; ++k)
        for (int j = 0; j < n[1]; ++j) lu_solve_strided(n[0], p, LU[0], x + ((long)k * n[1] + j) * n[0], 1);
    for (int k = 0; k < n[2]; ++k)
        for (int i = 0; i < n[0]; ++i) lu_solve_strided(n[1], p, LU[1], x + (long)k * n[1] * n[0] + i, n[0]);
    for (int j = 0; j < n[1]; ++j)
        for (int i = 0; i < n[0]; ++i) lu_solve_strided(n[2], p, LU[2], x + (long)j * n[0] + i, (long)n[0] * n[1]);
}

static real dot(long N, const real *a, const real *b) {
    real s = 0.0;
    for (long q = 0; q < N; ++q) s += a[q] * b[q];
    return s;
}

/* Ricker wavelet R(t) = (1 - 2 pi^2 f0^2 (t-t0)^2) exp(-pi^2 f0^2 (t-t0)^2)  (C14) */
real or_ricker(real t, real f0, real t0) {
    const real pi = (real)3.14159265358979323846264338327950288L;
    real a = pi * pi * f0 * f0 * (t - t0) * (t - t0);
    return (1.0 - 2.0 * a) * exp(-a);
}

/* ------------------------------------------------------------------------ */
/* Scalar P-wave solver (3D per C5)                         */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n[3], nel[3], p, bc, scheme;   /* scheme 1 = R1 (default), 0 = literal Eq. 16 */
    int bcd[3];                        /* zero Dirichlet on direction d (the 2D axis has none) */
    real tau, eta;
    long step;
    real *M[3], *K[3], *A[3], *LU[3], *MDLU[3];
    real *U, *V, *a;                 /* R1: V = V_{n+1/2}; R0: V = Udot_n; a = Udd_n */
    real *src[3];
    int has_src, wavelet;
    real f0, t0, amp;
    real *w1, *w2, *w3, *w4;
} or_pwave;

static void pw_free(or_pwave *h) {
    if (!h) return;
    for (int d = 0; d < 3; ++d) {
        free(h->M[d]); free(h->K[d]); free(h->A[d]); free(h->LU[d]); free(h->MDLU[d]); free(h->src[d]);
    }
    free(h->U); free(h->V); free(h->a); free(h->w1); free(h->w2); free(h->w3); free(h->w4);
    free(h);
}

long or_pw_size(const or_pwave *h) { return (long)h->n[0] * h->n[1] * h->n[2]; }

int or_pw_create(or_pwave **out, int nelx, int nely, int nelz, int p, real tau, int bc, int scheme) {
    *out = NULL;
    /* nelz = 0: the 2D scheme as the paper prints it (Eqs. 14-16): a third axis
     * with one function, M_z = 1, K_z = 0 and no boundary, so that K = Kx(x)My + Mx(x)Ky and
     * D = Ax(x)Ay exactly (Kronecker products with the 1 x 1 identity) */
    if (p < 1 || p > 5 || nelx < 1 || nely < 1 || nelz < 0 || !(tau > 0.0) || !isfinite(tau) || (bc != 0 && bc != 1))
        return OR_E_INVAL;
    or_pwave *h = (or_pwave *)calloc(1, sizeof(or_pwave));
    int nel[3] = {nelx, nely, nelz};
    h->p = p; h->bc = bc; h->tau = tau; h->eta = tau * tau / 4.0; h->scheme = scheme;  /* eta: PAPER.md:173 */
    for (int d = 0; d < 3; ++d) {
        int n = nel[d] == 0 ? 1 : nel[d] + p;
        h->nel[d] = nel[d]; h->n[d] = n;
        h->bcd[d] = nel[d] == 0 ? 0 : bc;
        if (h->bcd[d] == 1 && n < 3) { pw_free(h); return OR_E_INVAL; }
        h->M[d] = (real *)malloc(sizeof(real) * n * n);
        h->K[d] = (real *)malloc(sizeof(real) * n * n);
        h->A[d] = (real *)malloc(sizeof(real) * n * n);
        h->LU[d] = (real *)malloc(sizeof(real) * n * n);
        h->MDLU[d] = (real *)malloc(sizeof(real) * n * n);
        or_matrices_1d(p, nel[d], bc, h->M[d], h->K[d], NULL);
        /* A_d = M_d + tau^2/4 K_d   (Eq. 16) */
        for (int q = 0; q < n * n; ++q) h->A[d][q] = h->M[d][q] + h->eta * h->K[d][q];
        memcpy(h->MDLU[d], h->M[d], sizeof(real) * n * n);
        if (h->bcd[d] == 1) {
            h->A[d][0] = 1.0; h->A[d][n * n - 1] = 1.0;
            h->MDLU[d][0] = 1.0; h->MDLU[d][n * n - 1] = 1.0;
        }
        memcpy(h->LU[d], h->A[d], sizeof(real) * n * n);
        int rc = or_banded_lu(n, p, h->LU[d]);
        if (rc == OR_OK) rc = or_banded_lu(n, p, h->MDLU[d]);
        if (rc != OR_OK) { pw_free(h); return rc; }
    }
    long N = or_pw_size(h);
    h->U = (real *)calloc(N, sizeof(real));
    h->V = (real *)calloc(N, sizeof(real));
    h->a = (real *)calloc(N, sizeof(real));
    h->w1 = (real *)calloc(N, sizeof(real));
    h->w2 = (real *)calloc(N, sizeof(real));
    h->w3 = (real *)calloc(N, sizeof(real));
    h->w4 = (real *)calloc(N, sizeof(real));
    if (!h->U || !h->V || !h->a || !h->w1 || !h->w2 || !h->w3 || !h->w4) { pw_free(h); return OR_E_NOMEM; }
    *out = h;
    return OR_OK;
}

void or_pw_destroy(or_pwave *h) { pw_free(h); }

int or_pw_set_source(or_pwave *h, const real *bx, const real *by, const real *bz,
                     int wavelet, real f0, real t0, real amp) {
    for (int d = 0; d < 3; ++d) { free(h->src[d]); h->src[d] = NULL; }
    h->has_src = 0;
    if (!bx) return OR_OK;
    const real *b[3] = {bx, by, bz};
    for (int d = 0; d < 3; ++d) {
        h->src[d] = (real *)malloc(sizeof(real) * h->n[d]);
        memcpy(h->src[d], b[d], sizeof(real) * h->n[d]);
        if (h->bcd[d] == 1) { h->src[d][0] = 0.0; h->src[d][h->n[d] - 1] = 0.0; }
    }
    h->has_src = 1; h->wavelet = wavelet; h->f0 = f0; h->t0 = t0; h->amp = amp;
    return OR_OK;
}

/* g(t) of F(t) = g(t) b_x(x)b_y(x)b_z */
static real src_g(const or_pwave *h, real t) {
    if (!h->has_src) return 0.0;
    if (h->wavelet == 1) return h->amp * or_ricker(t, h->f0, h->t0);
    return h->amp;
}

/* out = F(t) - K P  (RHS of Eq. 14/16 with P = U + tau*Udot, 3D terms C5).
 * Dirichlet rows vanish because the 1D factors are interior-restricted. */
static void pw_rhs(or_pwave *h, real t, const real *P, real *out) {
    const int *n = h->n;
    long N = or_pw_size(h);
    int p = h->p;
    for (long q = 0; q < N; ++q) out[q] = 0.0;
    kron3_acc(n, p, h->K[0], h->M[1], h->M[2], -1.0, P, out, h->w3, h->w4);
    kron3_acc(n, p, h->M[0], h->K[1], h->M[2], -1.0, P, out, h->w3, h->w4);
    kron3_acc(n, p, h->M[0], h->M[1], h->K[2], -1.0, P, out, h->w3, h->w4);
    real g = src_g(h, t);
    if (h->has_src && g != 0.0) {
        for (int k = 0; k < n[2]; ++k)
            for (int j = 0; j < n[1]; ++j)
                for (int i = 0; i < n[0]; ++i)
                    out[((long)k * n[1] + j) * n[0] + i] += g * h->src[0][i] * h->src[1][j] * h->src[2][k];
    }
}

/* Unit operations exposed for kernel-level parity tests. */
int or_pw_kapply(or_pwave *h, const real *P, real *out) {   /* out = K P */
    long N = or_pw_size(h);
    for (long q = 0; q < N; ++q) out[q] = 0.0;
    kron3_acc(h->n, h->p, h->K[0], h->M[1], h->M[2], 1.0, P, out, h->w3, h->w4);
    kron3_acc(h->n, h->p, h->M[0], h->K[1], h->M[2], 1.0, P, out, h->w3, h->w4);
    kron3_acc(h->n, h->p, h->M[0], h->M[1], h->K[2], 1.0, P, out, h->w3, h->w4);
    return OR_OK;
}
int or_pw_dsolve(or_pwave *h, real *x) { kron3_solve(h->n, h->p, h->LU, x); return OR_OK; }  /* x <- D^-1 x */
int or_pw_dapply(or_pwave *h, const real *x, real *out) {                              /* out = D x */
    long N = or_pw_size(h);
    for (long q = 0; q < N; ++q) out[q] = 0.0;
    kron3_acc(h->n, h->p, h->A[0], h->A[1], h->A[2], 1.0, x, out, h->w3, h->w4);
    return OR_OK;
}
int or_pw_mapply(or_pwave *h, const real *x, real *out) {                              /* out = M x */
    long N = or_pw_size(h);
    for (long q = 0; q < N; ++q) out[q] = 0.0;
    kron3_acc(h->n, h->p, h->M[0], h->M[1], h->M[2], 1.0, x, out, h->w3, h->w4);
    return OR_OK;
}
/* x <- (M_x (x) M_y (x) M_z)^-1 x  (L2 projection solve) */
int or_pw_msolve(or_pwave *h, real *x) { kron3_solve(h->n, h->p, h->MDLU, x); return OR_OK; }

/* Mass solve of a 1D vector in direction d (for separable L2 projections). */
int or_pw_msolve_1d(or_pwave *h, int d, real *x) { or_lu_solve(h->n[d], h->p, h->MDLU[d], x); return OR_OK; }

/* set_state: R1 half-kick start (C2): a0 = D^-1 (F(0) - K u0), V0 = udot0 + tau/2 a0. */
int or_pw_set_state(or_pwave *h, const real *u, const real *udot) {
    long N = or_pw_size(h);
    const int *n = h->n;
    for (int k = 0; k < n[2]; ++k)
        for (int j = 0; j < n[1]; ++j)
            for (int i = 0; i < n[0]; ++i) {
                long q = ((long)k * n[1] + j) * n[0] + i;
                int bnd = (h->bcd[0] && (i == 0 || i == n[0] - 1)) || (h->bcd[1] && (j == 0 || j == n[1] - 1)) ||
                          (h->bcd[2] && (k == 0 || k == n[2] - 1));
                h->U[q] = bnd ? 0.0 : u[q];
                h->V[q] = bnd ? 0.0 : (udot ? udot[q] : 0.0);
            }
    h->step = 0;
    if (h->scheme == 1) {
        pw_rhs(h, 0.0, h->U, h->a);
        kron3_solve(n, h->p, h->LU, h->a);
        for (long q = 0; q < N; ++q) h->V[q] += 0.5 * h->tau * h->a[q];
    } else {
        for (long q = 0; q < N; ++q) h->a[q] = 0.0;
    }
    return OR_OK;
}

/* One time step n -> n+1.
 * R1: P = U + tau V;  a = D^-1 (F(t_{n+1}) - K P);  V += tau a;  U = P.
 * R0 (literal Eq. 16):
 *     Udd = D^-1 (-K(U + tau Udot) + F_{n+1});  Udot' = Udot + tau/2 Udd;
 *     U' = U + tau Udot' - tau^2/2 Udd. */
static void pw_step1(or_pwave *h) {
    long N = or_pw_size(h);
    real tau = h->tau;
    real t1 = (real)(h->step + 1) * tau;
    real *P = h->w1;
    for (long q = 0; q < N; ++q) P[q] = h->U[q] + tau * h->V[q];
    pw_rhs(h, t1, P, h->a);
    kron3_solve(h->n, h->p, h->LU, h->a);
    if (h->scheme == 1) {
        for (long q = 0; q < N; ++q) {
            h->V[q] = h->V[q] + tau * h->a[q];
            h->U[q] = P[q];
        }
    } else {
        for (long q = 0; q < N; ++q) {
            real vd = h->V[q] + 0.5 * tau * h->a[q];
            h->U[q] = h->U[q] + tau * vd - 0.5 * tau * tau * h->a[q];
            h->V[q] = vd;
        }
    }
    h->step += 1;
}

int or_pw_step(or_pwave *h, int nsteps) {
    if (nsteps < 0) return OR_E_INVAL;
    for (int s = 0; s < nsteps; ++s) pw_step1(h);
    return OR_OK;
}

/* get_state: U_n and udot_n = V_{n+1/2} - tau/2 a_n (R1); a_n.  Any pointer may be NULL. */
int or_pw_get_state(or_pwave *h, real *u, real *udot, real *a) {
    long N = or_pw_size(h);
    for (long q = 0; q < N; ++q) {
        if (u) u[q] = h->U[q];
        if (udot) udot[q] = (h->scheme == 1) ? h->V[q] - 0.5 * h->tau * h->a[q] : h->V[q];
        if (a) a[q] = h->a[q];
    }
    return OR_OK;
}

/* Raw state (U, V as stored, a). */
int or_pw_get_raw(or_pwave *h, real *U, real *V, real *a) {
    long N = or_pw_size(h);
    if (U) memcpy(U, h->U, sizeof(real) * N);
    if (V) memcpy(V, h->V, sizeof(real) * N);
    if (a) memcpy(a, h->a, sizeof(real) * N);
    return OR_OK;
}

real or_pw_time(or_pwave *h) { return (real)h->step * h->tau; }

/* Energies (C6): out[0] kinetic 1/2 v'Mv with v = V - tau/2 a,
 * out[1] potential 1/2 U'KU, out[2] invariant 1/2 V'DV + 1/2 U_n' K U_{n+1}. */
int or_pw_energy(or_pwave *h, real out[3]) {
    long N = or_pw_size(h);
    real *v = h->w1, *Mv = h->w2;
    for (long q = 0; q < N; ++q) v[q] = (h->scheme == 1) ? h->V[q] - 0.5 * h->tau * h->a[q] : h->V[q];
    or_pw_mapply(h, v, Mv);
    out[0] = 0.5 * dot(N, v, Mv);
    real *KU = h->w2;
    or_pw_kapply(h, h->U, KU);
    out[1] = 0.5 * dot(N, h->U, KU);
    if (h->scheme == 1) {
        real *DV = h->w1;
        or_pw_dapply(h, h->V, DV);
        real e = 0.5 * dot(N, h->V, DV);
        /* U_{n+1} = U_n + tau V */
        real *P = h->w1;
        for (long q = 0; q < N; ++q) P[q] = h->U[q] + h->tau * h->V[q];
        or_pw_kapply(h, P, KU);
        out[2] = e + 0.5 * dot(N, h->U, KU);
    } else {
        out[2] = NAN;
    }
    return OR_OK;
}

/* Dense 1D matrices of the handle (for tests): which 0=M 1=K 2=A 3=LU. */
int or_pw_matrix(or_pwave *h, int d, int which, real *out) {
    int n = h->n[d];
    const real *src = which == 0 ? h->M[d] : which == 1 ? h->K[d] : which == 2 ? h->A[d] : h->LU[d];
    memcpy(out, src, sizeof(real) * n * n);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* 3D isotropic linear elasticity (3D per C10/C11/C12)     */
/*                                                                          */
/* a(w,u) = int mu grad w : grad u + mu grad w : (grad u)^T + lam div w div u */
/* (from (w_(i,j), sigma_ij)).  Block (i,k), test     */
/* component i, trial component k:                                          */
/*   Ups_ii = (2mu+lam) K_(i) + mu sum_{d!=i} K_(d)                          */
/*   Ups_ik = mu [B]_k [B^T]_i + lam [B]_i [B^T]_k      (M in the third dir) */
/* where K_(d) is K in direction d and M elsewhere; B(a,c) = int N'_a N_c.   */
/* Split factors S_i = rho (x)_d (M_d + c_{i,d} K_d),                        */
/*   c_{i,d} = tau^2/(4 rho) (2mu+lam if d==i else mu). */
/* Step (delta form of Eqs. 35/36 with the split of Eq. 37):                 */
/*   P = U + tau V; r = f - Ups P;                                           */
/*   predictor i = x,y,z:  S_i w_i = r_i - tau^2/2 sum_{j<i} Ups_ij w_j      */
/*   corrector i = z,y,x:  S_i z_i = rho M w_i - tau^2/2 sum_{j>i} Ups_ij z_j */
/*   V += tau z;  U = P.                                                     */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n[3], p, bc;
    int bcd[3];                        /* zero Dirichlet on direction d (the 2D axis has none) */
    real tau, lam, mu, rho;
    long step;
    real *M[3], *K[3], *B[3], *BT[3];
    real *SL[3], *SS[3];   /* LU of M_d + c K_d: SL with (2mu+lam), SS with mu */
    real *MDLU[3];
    real *U[3], *V[3], *z[3];
    real *w[3], *r[3], *P[3], *t1, *t2, *t3;
} or_elastic;

static void el_free(or_elastic *h) {
    if (!h) return;
    for (int d = 0; d < 3; ++d) {
        free(h->M[d]); free(h->K[d]); free(h->B[d]); free(h->BT[d]);
        free(h->SL[d]); free(h->SS[d]); free(h->MDLU[d]);
        free(h->U[d]); free(h->V[d]); free(h->z[d]); free(h->w[d]); free(h->r[d]); free(h->P[d]);
    }
    free(h->t1); free(h->t2); free(h->t3);
    free(h);
}

long or_el_size(const or_elastic *h) { return (long)h->n[0] * h->n[1] * h->n[2]; }

int or_el_create(or_elastic **out, int nelx, int nely, int nelz, int p, real tau, int bc,
                 real lam, real mu, real rho) {
    *out = NULL;
    /* nelz = 0: the 2D (plane-strain) problem PAPER.md:362-387 on the same code -- a third axis with
     * one function, M_z = 1, K_z = B_z = 0 and no boundary.  The blocks Ups_xz, Ups_yz vanish
     * (B_z = 0), so (u_x, u_y) evolve by the 2D blocks Ups_xx = (2mu+lam) Kx(x)My + mu Mx(x)Ky,
     * Ups_xy = mu [B]_y [B^T]_x + lam [B]_x [B^T]_y, and u_z (antiplane, Ups_zz = mu (Kx My + Mx Ky))
     * stays what it starts as (0 for the paper's 2D problem). */
    if (p < 1 || p > 5 || nelx < 1 || nely < 1 || nelz < 0 || !(tau > 0.0) || (bc != 0 && bc != 1) ||
        !(mu > 0.0) || !(rho > 0.0) || !(lam >= 0.0))
        return OR_E_INVAL;
    or_elastic *h = (or_elastic *)calloc(1, sizeof(or_elastic));
    int nel[3] = {nelx, nely, nelz};
    h->p = p; h->bc = bc; h->tau = tau; h->lam = lam; h->mu = mu; h->rho = rho;
    real cl = tau * tau / (4.0 * rho) * (2.0 * mu + lam), cs = tau * tau / (4.0 * rho) * mu;
    for (int d = 0; d < 3; ++d) {
        int n = nel[d] == 0 ? 1 : nel[d] + p;
        h->n[d] = n;
        h->bcd[d] = nel[d] == 0 ? 0 : bc;
        h->M[d] = (real *)malloc(sizeof(real) * n * n);
        h->K[d] = (real *)malloc(sizeof(real) * n * n);
        h->B[d] = (real *)malloc(sizeof(real) * n * n);
        h->BT[d] = (real *)malloc(sizeof(real) * n * n);
        h->SL[d] = (real *)malloc(sizeof(real) * n * n);
        h->SS[d] = (real *)malloc(sizeof(real) * n * n);
        h->MDLU[d] = (real *)malloc(sizeof(real) * n * n);
        or_matrices_1d(p, nel[d], bc, h->M[d], h->K[d], h->B[d]);
        for (int a = 0; a < n; ++a)
            for (int c = 0; c < n; ++c) h->BT[d][a * n + c] = h->B[d][c * n + a];
        for (int q = 0; q < n * n; ++q) {
            h->SL[d][q] = h->M[d][q] + cl * h->K[d][q];
            h->SS[d][q] = h->M[d][q] + cs * h->K[d][q];
            h->MDLU[d][q] = h->M[d][q];
        }
        if (h->bcd[d] == 1) {
            h->SL[d][0] = h->SS[d][0] = h->MDLU[d][0] = 1.0;
            h->SL[d][n * n - 1] = h->SS[d][n * n - 1] = h->MDLU[d][n * n - 1] = 1.0;
        }
        int rc = or_banded_lu(n, p, h->SL[d]);
        if (rc == OR_OK) rc = or_banded_lu(n, p, h->SS[d]);
        if (rc == OR_OK) rc = or_banded_lu(n, p, h->MDLU[d]);
        if (rc != OR_OK) { el_free(h); return rc; }
    }
    long N = or_el_size(h);
    for (int c = 0; c < 3; ++c) {
        h->U[c] = (real *)calloc(N, sizeof(real));
        h->V[c] = (real *)calloc(N, sizeof(real));
        h->z[c] = (real *)calloc(N, sizeof(real));
        h->w[c] = (real *)calloc(N, sizeof(real));
        h->r[c] = (real *)calloc(N, sizeof(real));
        h->P[c] = (real *)calloc(N, sizeof(real));
    }
    h->t1 = (real *)calloc(N, sizeof(real));
    h->t2 = (real *)calloc(N, sizeof(real));
    h->t3 = (real *)calloc(N, sizeof(real));
    *out = h;
    return OR_OK;
}

void or_el_destroy(or_elastic *h) { el_free(h); }

/* out += coef * Ups_ik in   (block (i,k) of the elasticity operator) */
static void el_block_acc(or_elastic *h, int i, int k, real coef, const real *in, real *out) {
    const real *F[3];
    if (i == k) {
        for (int d = 0; d < 3; ++d) {
            real c = (d == i) ? (2.0 * h->mu + h->lam) : h->mu;
            for (int e = 0; e < 3; ++e) F[e] = (e == d) ? h->K[e] : h->M[e];
            kron3_acc(h->n, h->p, F[0], F[1], F[2], coef * c, in, out, h->t1, h->t2);
        }
    } else {
        /* mu [B]_k [B^T]_i */
        for (int e = 0; e < 3; ++e) F[e] = (e == k) ? h->B[e] : (e == i) ? h->BT[e] : h->M[e];
        kron3_acc(h->n, h->p, F[0], F[1], F[2], coef * h->mu, in, out, h->t1, h->t2);
        /* lam [B]_i [B^T]_k */
        for (int e = 0; e < 3; ++e) F[e] = (e == i) ? h->B[e] : (e == k) ? h->BT[e] : h->M[e];
        kron3_acc(h->n, h->p, F[0], F[1], F[2], coef * h->lam, in, out, h->t1, h->t2);
    }
}

/* out_i = sum_k Ups_ik in_k  (component-major arrays of 3N) */
int or_el_apply(or_elastic *h, const real *in, real *out) {
    long N = or_el_size(h);
    for (int i = 0; i < 3; ++i) {
        for (long q = 0; q < N; ++q) out[i * N + q] = 0.0;
        for (int k = 0; k < 3; ++k) el_block_acc(h, i, k, 1.0, in + k * N, out + i * N);
    }
    return OR_OK;
}

static void el_S_solve(or_elastic *h, int i, real *x) {
    real *LU[3];
    for (int d = 0; d < 3; ++d) LU[d] = (d == i) ? h->SL[d] : h->SS[d];
    kron3_solve(h->n, h->p, LU, x);
    long N = or_el_size(h);
    for (long q = 0; q < N; ++q) x[q] /= h->rho;
}

/* x <- D~^-1 x with D~ = L~ (rho M)^-1 L~^T  (3N, component-major) */
static void el_dsolve_comp(or_elastic *h, real *const x[3]) {
    long N = or_el_size(h);
    real hh = 0.5 * h->tau * h->tau;
    /* predictor: S_i w_i = x_i - tau^2/2 sum_{j<i} Ups_ij w_j */
    for (int i = 0; i < 3; ++i) {
        real *wi = h->w[i];
        memcpy(wi, x[i], sizeof(real) * N);
        for (int j = 0; j < i; ++j) el_block_acc(h, i, j, -hh, h->w[j], wi);
        el_S_solve(h, i, wi);
    }
    /* corrector: S_i z_i = rho M w_i - tau^2/2 sum_{j>i} Ups_ij z_j */
    for (int i = 2; i >= 0; --i) {
        real *zi = x[i];
        for (long q = 0; q < N; ++q) zi[q] = 0.0;
        kron3_acc(h->n, h->p, h->M[0], h->M[1], h->M[2], h->rho, h->w[i], zi, h->t1, h->t2);
        for (int j = i + 1; j < 3; ++j) el_block_acc(h, i, j, -hh, x[j], zi);
        el_S_solve(h, i, zi);
    }
}

int or_el_dsolve(or_elastic *h, real *x) {
    long N = or_el_size(h);
    real *xs[3] = {x, x + N, x + 2 * N};
    el_dsolve_comp(h, xs);
    return OR_OK;
}

/* set_state with the half-kick start (C13): V0 = udot0 + tau/2 D~^-1 (f(0) - Ups U0), f = 0. */
int or_el_set_state(or_elastic *h, const real *u, const real *udot) {
    long N = or_el_size(h);
    const int *n = h->n;
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < n[2]; ++k)
            for (int j = 0; j < n[1]; ++j)
                for (int i = 0; i < n[0]; ++i) {
                    long q = ((long)k * n[1] + j) * n[0] + i;
                    int bnd = (h->bcd[0] && (i == 0 || i == n[0] - 1)) || (h->bcd[1] && (j == 0 || j == n[1] - 1)) ||
                              (h->bcd[2] && (k == 0 || k == n[2] - 1));
                    h->U[c][q] = bnd ? 0.0 : u[c * N + q];
                    h->V[c][q] = bnd ? 0.0 : (udot ? udot[c * N + q] : 0.0);
                }
    h->step = 0;
    for (int i = 0; i < 3; ++i) {
        for (long q = 0; q < N; ++q) h->z[i][q] = 0.0;
        for (int k = 0; k < 3; ++k) el_block_acc(h, i, k, -1.0, h->U[k], h->z[i]);
    }
    el_dsolve_comp(h, h->z);
    for (int c = 0; c < 3; ++c)
        for (long q = 0; q < N; ++q) h->V[c][q] += 0.5 * h->tau * h->z[c][q];
    return OR_OK;
}

int or_el_step(or_elastic *h, int nsteps) {
    long N = or_el_size(h);
    real tau = h->tau;
    for (int s = 0; s < nsteps; ++s) {
        for (int c = 0; c < 3; ++c)
            for (long q = 0; q < N; ++q) h->P[c][q] = h->U[c][q] + tau * h->V[c][q];
        for (int i = 0; i < 3; ++i) {
            for (long q = 0; q < N; ++q) h->z[i][q] = 0.0;
            for (int k = 0; k < 3; ++k) el_block_acc(h, i, k, -1.0, h->P[k], h->z[i]);
        }
        el_dsolve_comp(h, h->z);
        for (int c = 0; c < 3; ++c)
            for (long q = 0; q < N; ++q) {
                h->V[c][q] += tau * h->z[c][q];
                h->U[c][q] = h->P[c][q];
            }
        h->step += 1;
    }
    return OR_OK;
}

int or_el_get_state(or_elastic *h, real *u, real *udot, real *a) {
    long N = or_el_size(h);
    for (int c = 0; c < 3; ++c)
        for (long q = 0; q < N; ++q) {
            if (u) u[c * N + q] = h->U[c][q];
            if (udot) udot[c * N + q] = h->V[c][q] - 0.5 * h->tau * h->z[c][q];
            if (a) a[c * N + q] = h->z[c][q];
        }
    return OR_OK;
}

/* Energies: kinetic 1/2 rho v'Mv, potential 1/2 U'Ups U,
 * invariant 1/2 V'D~V + 1/2 U_n' Ups U_{n+1}  with D~ = L~ (rho M)^-1 L~^T. */
int or_el_energy(or_elastic *h, real out[3]) {
    long N = or_el_size(h);
    real *v = (real *)malloc(sizeof(real) * 3 * N);
    real *y = (real *)malloc(sizeof(real) * 3 * N);
    real *U = (real *)malloc(sizeof(real) * 3 * N);
    real *P = (real *)malloc(sizeof(real) * 3 * N);
    for (int c = 0; c < 3; ++c)
        for (long q = 0; q < N; ++q) {
            v[c * N + q] = h->V[c][q] - 0.5 * h->tau * h->z[c][q];
            U[c * N + q] = h->U[c][q];
            P[c * N + q] = h->U[c][q] + h->tau * h->V[c][q];
        }
    real ek = 0.0;
    for (int c = 0; c < 3; ++c) {
        for (long q = 0; q < N; ++q) h->t3[q] = 0.0;
        kron3_acc(h->n, h->p, h->M[0], h->M[1], h->M[2], h->rho, v + c * N, h->t3, h->t1, h->t2);
        ek += dot(N, v + c * N, h->t3);
    }
    out[0] = 0.5 * ek;
    or_el_apply(h, U, y);
    out[1] = 0.5 * dot(3 * N, U, y);
    /* V' D~ V = (L~^T V)' (rho M)^-1 (L~^T V) */
    real hh = 0.5 * h->tau * h->tau;
    real inv = 0.0;
    for (int i = 0; i < 3; ++i) {
        real *g = y + i * N;   /* g_i = S_i V_i + tau^2/2 sum_{j>i} Ups_ij V_j */
        for (long q = 0; q < N; ++q) g[q] = 0.0;
        /* S_i V_i: rho (x)_d (M_d + c_{i,d} K_d) applied as a Kronecker product */
        {
            real cl = h->tau * h->tau / (4.0 * h->rho) * (2.0 * h->mu + h->lam);
            real cs = h->tau * h->tau / (4.0 * h->rho) * h->mu;
            int n0 = h->n[0], n1 = h->n[1], n2 = h->n[2];
            real *Sd[3];
            int nn[3] = {n0, n1, n2};
            for (int d = 0; d < 3; ++d) {
                int n = nn[d];
                Sd[d] = (real *)malloc(sizeof(real) * n * n);
                real c = (d == i) ? cl : cs;
                for (int q = 0; q < n * n; ++q) Sd[d][q] = h->M[d][q] + c * h->K[d][q];
                if (h->bcd[d] == 1) { Sd[d][0] = 1.0; Sd[d][n * n - 1] = 1.0; }
            }
            kron3_acc(h->n, h->p, Sd[0], Sd[1], Sd[2], h->rho, h->V[i], g, h->t1, h->t2);
            for (int d = 0; d < 3; ++d) free(Sd[d]);
        }
        for (int j = i + 1; j < 3; ++j) el_block_acc(h, i, j, hh, h->V[j], g);
        memcpy(h->t3, g, sizeof(real) * N);
        kron3_solve(h->n, h->p, h->MDLU, h->t3);
        for (long q = 0; q < N; ++q) h->t3[q] /= h->rho;
        inv += dot(N, g, h->t3);
    }
    or_el_apply(h, P, y);
    out[2] = 0.5 * inv + 0.5 * dot(3 * N, U, y);
    free(v); free(y); free(U); free(P);
    return OR_OK;
}

real or_el_time(or_elastic *h) { return (real)h->step * h->tau; }
