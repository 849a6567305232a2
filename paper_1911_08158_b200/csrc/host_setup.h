// host_setup.h -- host-side (once per ads_create) 1D discretisation and
// factor tables for the B200 ADS solver.  Independent of oracle/ (no shared
// code): B-spline values by de Boor's triangular scheme, Gauss-Legendre by
// Newton on the Bonnet recurrence, Gram matrices accumulated in band storage,
// banded LU in band storage, partitioned-elimination (SPIKE-style) tables.
#pragma once
#include <vector>

namespace ads {

// Band storage of an n x n matrix with half-bandwidth p:
// band[i*(2p+1) + (j - i + p)] = A(i, j) for |i-j| <= p (0 outside the matrix).
struct Band {
    int n = 0, p = 0;
    std::vector<double> v;
    Band() = default;
    Band(int n_, int p_) : n(n_), p(p_), v((size_t)n_ * (2 * p_ + 1), 0.0) {}
    double &at(int i, int j) { return v[(size_t)i * (2 * p + 1) + (j - i + p)]; }
    double get(int i, int j) const {
        if (i < 0 || j < 0 || i >= n || j >= n || j - i > p || i - j > p) return 0.0;
        return v[(size_t)i * (2 * p + 1) + (j - i + p)];
    }
};

// 1D open-uniform B-spline space on [0,1] with its Gram matrices
// M = (N_a, N_c), K = (N'_a, N'_c), B = (N'_a, N_c).
struct Space1D {
    int p = 0, nel = 0, n = 0, bc = 0;
    std::vector<double> knots;
    Band M, K, B;
};

int gauss_legendre(int m, double *x, double *w);
// Nonzero basis values/derivatives at x in knot span `span` (p <= span < n):
// N[0..p], dN[0..p] belong to functions span-p .. span.
void basis_and_derivs(const std::vector<double> &t, int p, int span, double x, double *N, double *dN);
int build_space(int p, int nel, int bc, Space1D &s);
// Stiffness rows in plane-difference form (the operator kernel's Kz, kernels.cuh KopArgs::wz):
// (K T)_k = sum_{m < 2p} w[k*2p + m] (T_{k-p+m+1} - T_{k-p+m}) for every T of the space, using
// the row sums the exact matrix has -- zero for every row of the unrestricted space (K 1 = 0);
// on zero-Dirichlet rows next to a boundary the removed column's share, with T = 0 on the
// boundary function.  Computed in extended precision from the band of s.K.
void diff_weights(const Space1D &s, std::vector<double> &w);
// The 2D scheme's third axis (ads_create with nz = 0; PAPER.md:123-143 as printed in 2D): one
// function, M = 1, K = B = 0, no boundary -- K = Kx(x)My + Mx(x)Ky and D = Ax(x)Ay exactly.
void trivial_space(int p, Space1D &s);
// b_a = int f N_a over [0,1], 8-point Gauss per element; func 0 sin(pi x), 1 Gaussian.
void load_vector(const Space1D &s, int func, double c, double sigma, double *out);

// Banded LU without pivoting of A (n x n, half-bandwidth p), returned as
//   l[i*p + (k-1)]  = L(i, i-k)            (unit lower)
//   us[i*p + (k-1)] = U(i, i+k) / U(i, i)  (row-scaled upper)
//   dinv[i]         = 1 / U(i, i)
// Returns 0, or -2 if a pivot falls below 1e-14 * max|A|.
//
// With freeze = true the rows of the factors that have converged in the
// Toeplitz interior of A (entries changing by < 2 ulp over p+1 consecutive
// rows) are replaced by one constant row for i in [i_lo, i_hi); rows from
// i_hi on (where A stops being Toeplitz) are recomputed by the row-wise
// Doolittle recurrence from the frozen rows.  The result is an LU
// factorisation of A to rounding; it is accepted only if
// max |(LU - A)_ij| <= 1e-14 max|A| (else the plain factors are kept and
// i_lo = i_hi = 0).  Kernels keep the constant row in registers.
struct LUFactors {
    int n = 0, p = 0;
    std::vector<double> l, us, dinv;
    int i_lo = 0, i_hi = 0;  // frozen (uniform) rows [i_lo, i_hi)
    double residual = 0.0;   // max |(LU - A)_ij| / max |A|
};
int banded_lu(const Band &A, LUFactors &f, bool freeze = false);
void lu_solve_host(const LUFactors &f, double *x);  // in place, one vector

// Partitioned elimination tables for one direction: every line (padded with
// identity rows to C*L rows) is cut into C chunks of L rows solved
// independently, then coupled through the chunk boundary states.
//   gf[i*p + m]   response of the forward (L) recurrence at i to incoming
//                 state y_{s-1-m} = 1 (s = start of i's chunk)
//   gb[i*p + m]   response of the backward (U) recurrence at i to incoming
//                 state x_{e+m} = 1 (e = end of i's chunk)
//   Tf[c*p*p + a*p + b] = gf[(e_c-1-a)*p + b]   forward chunk transfer map
//   Rb[c*p*p + a*p + b] = gb[(s_c+a)*p + b]     backward chunk transfer map
// The incoming state of chunk c is in_c = Tf_{c-1} in_{c-1} + h_{c-1}
// (h = outgoing state of the zero-incoming pass).  Kf is the number of
// preceding chunks the device folds in: the smallest k with
// ||Tf_{c-1} ... Tf_{c-k}||_inf < 2^-64 for every c (contributions of older
// chunks are below 2^-64 of the state, i.e. no bit of an fp64 result), or C-1
// (the complete chain) if no such k exists.  Kb likewise for Rb.
struct PartTables {
    int n = 0, p = 0, C = 0, L = 0, Kf = 0, Kb = 0;
    std::vector<double> gf, gb, Tf, Rb;
};
// Chunk length: the smallest value of kChunkLens with C*L >= n and L >= p
// (0 if none).  Odd lengths keep the x-tile shared-memory reads conflict-free.
constexpr int kChunkLens[] = {1, 3, 5, 9, 17, 33};
int choose_chunk_len(int n, int p, int C);
// f: factors padded to C*L rows (identity rows beyond n)
void build_part_tables(const LUFactors &f, int C, int L, PartTables &t);

}  // namespace ads

namespace ads {

// ---- z-slab decomposition (multi-GPU) ----
// Balanced split of n planes over G slabs: slab j = [z0[j], z0[j] + nl[j]).
void slab_plan(int n, int G, std::vector<int> &z0, std::vector<int> &nl);

// Distributed exact SPIKE for A (global band, Dirichlet rows set) cut into slabs:
//   x_j = xloc_j - V_j u_{j+1} - W_j b_{j-1},  xloc_j = A_jj^-1 r_j,
//   V_j = A_jj^-1 [0; B_j], W_j = A_jj^-1 [C_j; 0]   (p spike columns, [nl][p] row-major),
// u_{j+1} = first p values of x_{j+1}, b_{j-1} = last p values of x_{j-1}.  Interface j|j+1:
//   [b_j; u_{j+1}] = Q_j [bl_j; ul_{j+1}],  Q_j = inverse of [[I, Vbot_j], [Wtop_{j+1}, I]]
// which is exact when the dropped couplings W_j(bottom p rows) and V_{j+1}(top p rows) are
// below 2^-64 (certified: `certified`), i.e. the spikes decay across a slab.
struct SlabSpikes {
    LUFactors lu;             // (unused by the device: tables are rebuilt from `block`)
    Band block;               // A_jj
    std::vector<double> V, W; // [nl][p]
};
int build_slab_spikes(const Band &A, int z0, int nl, SlabSpikes &s);
// Q_j (2p x 2p row-major) from slab j and j+1; returns the max dropped coupling entry.
double interface_inverse(const SlabSpikes &sj, const SlabSpikes &sj1, int p, std::vector<double> &Q);

}  // namespace ads

namespace ads {

// ---- modal basis of one direction (Eqs. 17-18) ----
// Generalised symmetric-definite eigenproblem of the 1D pencil on the active DOFs (all n for
// bc = 0, the n - 2 interior ones for bc = 1): K phi = lambda M phi with Phi^T M Phi = I.
// Dense Cholesky M = L L^T, C = L^-1 K L^-T, Householder tridiagonalisation, implicit QL,
// Phi = L^-T Z.  lam ascending; phi row-major, phi[i * na + k] = component i of eigenvector k.
// Returns 0, or -1 (M not positive definite, QL not converged, no active DOF).
// The reversal symmetry of the uniform basis splits the pencil into even and odd blocks solved
// separately; parity (if non-null) receives +1 / -1 per eigenvector (exact by construction).
int modal_basis(const Space1D &s, std::vector<double> &lam, std::vector<double> &phi,
                std::vector<int> *parity = nullptr);

}  // namespace ads
