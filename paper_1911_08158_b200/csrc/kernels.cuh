// kernels.cuh -- device kernel interfaces of the B200 ADS solver (sm_100a, fp64).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace ads {

// Banded 1D matrix on the device: b[i*(2p+1) + c] = A(i, i - p + c).
// Factor tables of A_d = M_d + tau^2/4 K_d (see host_setup.h LUFactors/PartTables),
// padded with identity rows to C*L rows (C = kSweepChunks chunks of L rows).
// Rows [i_lo, i_hi) (whole chunks) are one constant row (lc, usc, dic): warps
// whose chunks all lie inside read their coefficients from the kernel's
// constant bank instead of memory.
constexpr int kMaxP = 5;
constexpr int kSweepChunks = 32;
constexpr int kMaxChunkLen = 33;
struct SolveTab {
    const double *l = nullptr, *us = nullptr, *dinv = nullptr;  // [C*L][p], [C*L][p], [C*L]
    const double *Tf = nullptr, *Rb = nullptr;                  // [C][p][p] chunk transfer maps
    int n = 0, L = 0, Kf = 0, Kb = 0;
    int C = kSweepChunks;  // chunks per line: 32, or 16 (chunks of <= 17 rows) when that pads less
    int c_lo = 0, c_hi = 0;  // uniform chunks [c_lo, c_hi): rows [c_lo L, c_hi L) are (lc, usc, dic)
    double lc[kMaxP] = {0, 0, 0, 0, 0}, usc[kMaxP] = {0, 0, 0, 0, 0}, dic = 0.0;
    // responses of a uniform chunk at local row j to a unit incoming state m:
    // Gf (forward, y_{-1-m} = 1) and Gb (backward, x_{L+m} = 1)
    double Gf[kMaxChunkLen][kMaxP] = {}, Gb[kMaxChunkLen][kMaxP] = {};
};

// Geometry of a field: x-fastest, sy = row stride, sz = plane stride (elements).
struct Geom {
    int n0 = 0, n1 = 0, n2 = 0;
    long sy = 0, sz = 0;
};

// r = g * (bx (x) by (x) bz) + sign * K P,  P = U + tau V  (P written to Pout if non-null).
// K = Kx(x)My(x)Mz + Mx(x)Ky(x)Mz + Mx(x)My(x)Kz by sum factorisation.
// Rows [ilo[d], ihi[d]] of M_d, K_d are the Toeplitz row (mc[d], kc[d]) bitwise (uniform mesh,
// host_setup build_space); tiles/planes inside read these from the constant bank.
struct KopArgs {
    const double *U = nullptr, *V = nullptr;
    double *Pout = nullptr, *r = nullptr;
    double tau = 0.0, g = 0.0, sign = -1.0;
    const double *bx = nullptr, *by = nullptr, *bz = nullptr;
    const double *mx = nullptr, *kx = nullptr, *my = nullptr, *ky = nullptr, *mz = nullptr, *kz = nullptr;
    Geom geo;
    int zlen = 0;
    int ilo[3] = {1, 1, 1}, ihi[3] = {0, 0, 0};
    double mc[3][2 * kMaxP + 1] = {}, kc[3][2 * kMaxP + 1] = {};
    // weight of each direction's K term: K = kw0 Kx My Mz + kw1 Mx Ky Mz + kw2 Mx My Kz (1 for the
    // P-wave; elasticity's diagonal blocks mu K + (mu + lam) K_(i)).  The interior rows kc[d]
    // arrive pre-scaled; boundary rows are scaled where they are staged.
    double kw[3] = {1.0, 1.0, 1.0};
    // Kz in plane-difference form (kop v4): (Kz T)_k = sum_m wz[k][m] (T_{k-p+m+1} - T_{k-p+m}),
    // m < 2p, rows global (table [n2 global][2p]); wzc: the Toeplitz interior row, pre-scaled by kw[2]
    const double *wz = nullptr;
    double wzc[2 * kMaxP] = {};
    // global planes whose P counts as zero in those differences (zero-Dirichlet z faces; -1: none)
    int zd0 = -1, zd1 = -1;
    // z-slabs: the halo planes (outside [0, n2)) hold the neighbours' drifted field P itself in Ph
    // (exchanged instead of U and V); the kernel reads them there (nullptr: U + tau V everywhere)
    const double *Ph = nullptr;
    // z-slabs: local plane k is global row k + zoff of Mz, Kz (and of bz); input planes
    // [zv0, zv1) exist in memory (halo planes of a slab); outputs are planes [0, n2)
    int zoff = 0, zv0 = 0, zv1 = -1;
    // device-side source time (CUDA graphs): when dstep is set, g = amp R((*dstep + 1) tau_g)
    // (R = Ricker if wav, else 1) replaces the host value g
    const long *dstep = nullptr;
    int wav = 0;
    bool pdl = false;  // programmatic dependent launch (the elastic step)
    double f0 = 0.0, t0 = 0.0, amp = 0.0, tau_g = 0.0;
};

// Distributed z-solve (exact SPIKE, host_setup.h build_slab_spikes) on the owned planes of a
// slab j (geometry g, n2 = nl), X = local solution of the slab's diagonal block:
//   stage 1 (launch_zint):  b0 = Qt[0:p, :] [tip_prev; X(first p)]     -> b0buf  (= b_{j-1}^0)
//                           u0 = Qb[p:2p, :] [X(last p); tip_next]      -> u0buf  (= u_{j+1}^0)
//   exchange: b0buf -> slab j+1 (its b0_prev2), u0buf -> slab j-1 (its u0_next2)
//   stage 2 (launch_zfix): one Jacobi refinement of both interface systems with the couplings
//   to the next interfaces (Wbot, Vtop p x p), then x = X - W b_{j-1} - V u_{j+1} and the kick
//   Vf += kick x (A = x if non-null).
// tip_prev / tip_next: p planes (plane stride sz) received from the neighbours (null: none).
struct ZfixArgs {
    const double *X = nullptr, *tip_prev = nullptr, *tip_next = nullptr;
    const double *b0_prev2 = nullptr, *u0_next2 = nullptr;  // stage-1 values of slabs j-1 / j+1
    double *b0buf = nullptr, *u0buf = nullptr;              // this slab's stage-1 values
    const double *Vsp = nullptr, *Wsp = nullptr;            // [nl][p]
    double *Vf = nullptr, *A = nullptr;
    double kick = 0.0;
    double qt[2 * kMaxP][2 * kMaxP] = {}, qb[2 * kMaxP][2 * kMaxP] = {};
    // couplings dropped by stage 1: top interface (j-1|j): Wbot_{j-1}, Vtop_j;
    // bottom interface (j|j+1): Wbot_j, Vtop_{j+1}
    double wbp[kMaxP][kMaxP] = {}, vtm[kMaxP][kMaxP] = {}, wbm[kMaxP][kMaxP] = {}, vtn[kMaxP][kMaxP] = {};
    Geom geo;
};
int launch_zint(int p, const ZfixArgs &a, cudaStream_t s);
int launch_zfix(int p, const ZfixArgs &a, cudaStream_t s);

// Batched banded solve along direction dir of every line of `in`.
// mode 0: out = A^-1 in; mode 1: V += kick * (A^-1 in) and out = A^-1 in if out != nullptr.
struct SweepArgs {
    const double *in = nullptr;
    double *out = nullptr;
    double *V = nullptr;
    double kick = 0.0;
    SolveTab t;
    Geom geo;
    int dir = 0;
    int mode = 0;
    // y/z sweeps: TMA descriptors of `in` and `V` (3D, boxes of 16 lines x rb rows), filled by
    // the launcher; nbox boxes of rb rows cover the C L (identity-padded) rows of a line
    alignas(64) CUtensorMap tm_in;
    alignas(64) CUtensorMap tm_v;
    alignas(64) CUtensorMap tm_out;  // x sweep: TMA stores of the solved tile
    int rb = 0, nbox = 0;
    // y/z sweeps: number of output (or V) tile buffers, 1 or 2 (set by the launcher when the
    // shared memory holds a second one: a TMA store is then waited for two tiles later)
    bool pdl = false;  // programmatic dependent launch (the elastic step)
    int vbufs = 1;
    long *dstep_inc = nullptr;  // y/z: block 0 increments the device step counter (graph steps)
};

int launch_kop(int p, const KopArgs &a, cudaStream_t s);
// Modal propagation (§3, reading R1): for every mode (i, j, k)
// of the padded layout (i < n0), L = lx_i + ly_j + lz_k, delta = (1 + eta lx_i)(1 + eta ly_j)
// (1 + eta lz_k), eta = tau^2/4.  g == nullptr: [cU; cV] <- A^n [cU; cV],
// A = [[1, tau], [-tau L/delta, 1 - tau^2 L/delta]] by repeated squaring, ca = -(L/delta) cU;
// else n R1 steps cP = cU + tau cV, ca = (g[s] fx_i fy_j fz_k - L cP)/delta, cV += tau ca, cU = cP.
int launch_modal(double *cU, double *cV, double *ca, const double *lx, const double *ly, const double *lz,
                 const double *fx, const double *fy, const double *fz, const double *g, long nsteps, double tau,
                 const Geom &geo, cudaStream_t s);
void launch_set_long(long *dst, long value, cudaStream_t s);
// The folded modal transforms along one axis as FP64 tensor-core GEMMs (modal_tc.cu, f3):
// forward out[slots] = [Q_e fold_e(in); Q_o fold_o(in); 0], inverse out = unfold(P_e in_e, P_o in_o).
// Element k of line l in batch b at k ks + l ls + b bs (nl lines, nb batches); maps column-major.
struct ModalGemmArgs {
    const double *in = nullptr;
    double *out = nullptr;
    long ks = 1, ls = 1, bs = 0;
    int nl = 0, nb = 1;
    int n = 0, ne = 0, no = 0, H = 0, hh = 0;
    const double *Qe = nullptr, *Qo = nullptr, *Pe = nullptr, *Po = nullptr;
    int inverse = 0;
    // tensor-core path: the same maps column-major with even leading dimensions (TMA strides are
    // 16-byte multiples) -- Q_e with its middle column (n odd) halved: the fold loads u(h) twice
    const double *Qe2 = nullptr, *Qo2 = nullptr, *Pe2 = nullptr, *Po2 = nullptr;
    int lqe = 0, lqo = 0, lpe = 0, lpo = 0;
    // the addressing as a 3D tensor (for the TMA maps): element (k, l, b) of the axis view
    long td[3] = {0, 0, 0}, ts1 = 0, ts2 = 0;
    int kdim = 0;  // which tensor dimension is k (0: x lines, k contiguous; 1: y / z)
    int tail_only = 0;  // run only the CUDA-core tail rows (the tensor-core path did the full tiles)
    int fuse_tail = 0;  // the TMA kernels' last full-tile CTAs also compute the (<= 4) tail rows
};
int encode_map_3d(CUtensorMap *m, const double *base, long d0, long d1, long d2, long s1, long s2, unsigned b0,
                  unsigned b1, unsigned b2);
int launch_modal_gemm(const ModalGemmArgs &g, cudaStream_t s);
// dense caller layout (n0 n1 n2, x fastest) <-> pitched field (sy, sz): to_pitched = 1 unpacks
void launch_repack(const double *src, double *dst, const Geom &g, int to_pitched, cudaStream_t s);
// Solve along a direction of line length 1 (the 2D scheme's third axis): x = scale in, then the
// sweep's epilogue -- out = x (if out), V += kick x (if V), *inc += 1 (if inc).  Elementwise.
void launch_line1(const double *in, double *out, double *V, double scale, double kick, long *inc, const Geom &g,
                  cudaStream_t s);
int launch_sweep(int p, const SweepArgs &a, cudaStream_t s);
// Short lines along y (dir 1) or z (dir 2): one thread per line running the sequential banded LU
// recurrences of the factors in a.t (rows [0, t.n)), threads of a block on adjacent x-lines
// (coalesced rows); y is kept in `out` between the forward and the backward pass.  Same modes
// as launch_sweep (kick, dstep_inc).  Used for the z blocks of thin slabs (at most kLineSweepMax
// planes), where the partitioned kernel's per-tile overheads dominate (c4 as 8 slabs of 65
// planes: 6.49 -> 6.03 ms of summed work); slower than it from ~65-row lines of a whole grid up.
constexpr int kLineSweepMax = 96;
int launch_line_sweep(int p, const SweepArgs &a, cudaStream_t s);
// dynamic shared memory (bytes) a sweep along dir needs for these tables (one output buffer)
long sweep_smem_bytes(int p, const SolveTab &t, int dir);
constexpr long kMaxSmemPerCta = 227L * 1024;

// Small helpers (diagnostics / state I/O, not on the per-step path).
// out = alpha (A along axis d) in + beta out (band table [n_d][2p+1]; beta == 0: out not read).
// Along z: band row of local plane k is global row k + zoff; input planes [zv0, zv1) exist
// (default: [0, n2)).
int launch_axis_apply(int p, int d, const double *band, const double *in, double *out, const Geom &g, double alpha,
                      double beta, cudaStream_t s, int zoff = 0, int zv0 = 0, int zv1 = -1);
// out = alpha (Fx (x) Fy (x) Fz) in + beta out in one z-marching pass (beta == 0: out not read)
// Kronecker triples sharing input and output (elasticity):
//   out = beta out + sum_{t < nterms} alpha_t (Fx_t (x) Fy_t (x) Fz_t) in,  bands [n_d][2p+1]
struct KronTerms {
    int nterms = 1;
    const double *fx[2] = {nullptr, nullptr}, *fy[2] = {nullptr, nullptr}, *fz[2] = {nullptr, nullptr};
    double alpha[2] = {0.0, 0.0};
    const double *addend = nullptr;  // beta multiplies this field instead of out (nullptr: out)
    // rows [fylo[t], fyhi[t]] of Fy_t are the row fyrow[t] bitwise (uniform-mesh interior): tiles
    // inside take the y-pass coefficients from the kernel parameters (lo > hi: none)
    int fylo[2] = {1, 1}, fyhi[2] = {0, 0};
    double fyrow[2][2 * kMaxP + 1] = {};
};
int launch_kron3(int p, const double *in, double *out, const KronTerms &k3, double beta, const Geom &g,
                 cudaStream_t s);
// y = alpha x + beta y over N elements
int launch_axpby(long N, double alpha, const double *x, double beta, double *y, cudaStream_t s, bool pdl = false);
// u_c = sum_{t: comp_t = c} amp_t sx_t (x) sy_t (x) sz_t for every component c < ncomp (component stride
// cstride), zero on the Dirichlet faces (mx, my; ngz > 0: global z faces), in one pass.  f holds per
// term [amp, comp, sx (n0f), sy (n1f), sz (nzf, global z)]; local plane k is global plane k + zoff.
void launch_set_separable(double *u, long cstride, int ncomp, int nterms, const double *f, int n0f, int n1f, int nzf,
                          const Geom &g, int zoff, int mx, int my, int ngz, cudaStream_t s);
// P = U + tau V over N contiguous elements (the drift of a slab's edge planes)
void launch_drift(const double *U, const double *V, double tau, double *P, long N, cudaStream_t s);
// all-to-all z solve (ads_set_zsolve): kick from the returned pencil blocks.  arecv holds, for each
// y block q (rows [py0[q], py0[q+1])), the slab's solution a as [k][j - py0[q]][i] (row pitch g.sy)
// at offset g.n2 py0[q] g.sy; V += kick a and A = a (A may be null) on the slab's owned planes.
constexpr int kMaxA2A = 64;
struct KickA2AArgs {
    const double *arecv = nullptr;
    double *V = nullptr, *A = nullptr;
    double kick = 0.0;
    Geom geo;
    int nq = 1;
    int py0[kMaxA2A + 1] = {};
};
int launch_kick_a2a(const KickA2AArgs &a, cudaStream_t s);
// zero the boundary faces of a field (Dirichlet masking)
// (slabs: local plane k is global plane k + zoff of ngz; default the field is the whole grid)
int launch_mask_boundary(double *u, const Geom &g, cudaStream_t s, int zoff = 0, int ngz = -1);
// deterministic dot product: partial sums into `partial` (>= 1024 doubles), result into *res (device)
int launch_dot(long N, const double *x, const double *y, double *partial, double *res, cudaStream_t s);

}  // namespace ads
