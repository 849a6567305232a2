/*
 * ads.h -- C ABI of the B200-native alternating-direction-split (ADS)
 * isogeometric implicit wave solver (hot path of arXiv:1911.08158).
 *
 * The library implements, on one NVIDIA B200 (sm_100a), in fp64, the time step
 * of the paper's split scheme (Eq. 16, read as R1 -- see
 * DESIGN.md §3) on a tensor-product B-spline grid of degree p on [0,1]^3:
 *
 *   P   = U_n + tau V_n                         drift (= U_{n+1})
 *   r   = F(t_{n+1}) - K P                      K = Kx(x)My(x)Mz + Mx(x)Ky(x)Mz + Mx(x)My(x)Kz
 *                                               (Eq. 14, 3D)
 *   a   = (A_x (x) A_y (x) A_z)^{-1} r          A_d = M_d + tau^2/4 K_d
 *                                               three sweeps of banded solves
 *                                               (Appendix)
 *   V_{n+1} = V_n + tau a ;  U_{n+1} = P        kick (R1)
 *
 * and the 3D elasticity variant (DESIGN.md §3 E1).
 *
 * Conventions
 *  - Every function returns an int status: ADS_OK (0) or a negative ADS_E_*.
 *    Nothing throws across the ABI.  After ADS_E_CUDA the handle is sticky-
 *    failed: every call except ads_destroy / ads_last_error returns ADS_E_STATE.
 *  - nx, ny, nz are numbers of ELEMENTS per direction.  The number of DOFs per
 *    direction is n_d = n_el,d + p and arrays hold N = n_x n_y n_z doubles
 *    (3N for elasticity, component-major), x fastest:
 *        u[(k * n_y + j) * n_x + i].
 *    With ADS_BC_DIRICHLET0 the boundary entries are ignored on input and are
 *    0 on output (interior restriction of each 1D space, C3).
 *  - Memory: `mem` = ADS_MEM_HOST (pageable or pinned host pointer) or
 *    ADS_MEM_DEVICE (a device pointer on the handle's device).  The library owns
 *    all its device buffers and copies caller arrays in/out; the caller owns
 *    every pointer it passes.
 *  - Streams: all device work is ordered on the handle's stream (default: a
 *    blocking stream the library creates, so it is ordered against CUDA's legacy
 *    default stream -- PyTorch's default stream; ads_set_stream attaches a caller
 *    stream, e.g. torch.cuda.current_stream().cuda_stream).  ads_step is
 *    asynchronous; ads_energy / ads_get_state synchronise the stream.
 *  - Device: every call works on the device that was current at ads_create.
 *  - A handle is single-writer (not thread-safe).
 */
#ifndef ADS_B200_H
#define ADS_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ads_ctx *ads_handle;

enum { ADS_BC_NATURAL = 0, ADS_BC_DIRICHLET0 = 1 };
enum {
    ADS_OK = 0,
    ADS_E_INVAL = -1,    /* invalid argument (SPEC.md exit 2) */
    ADS_E_SINGULAR = -2, /* banded LU pivot < 1e-14 max|band| */
    ADS_E_CUDA = -3,     /* CUDA runtime error (sticky) */
    ADS_E_NCCL = -4,     /* NCCL error (distributed handles) */
    ADS_E_NOMEM = -5,    /* device or host allocation failed */
    ADS_E_STATE = -6     /* handle is failed or call out of order */
};
enum { ADS_MEM_HOST = 0, ADS_MEM_DEVICE = 1 };
enum { ADS_FUNC_SIN = 0, ADS_FUNC_GAUSS = 1 };
enum { ADS_WAVELET_NONE = 0, ADS_WAVELET_RICKER = 1 };

/* Create a scalar P-wave solver.
 *   p in [1,5]; nx,ny,nz >= 1 (Dirichlet needs n_d >= 3); tau finite > 0;
 *   bc in {ADS_BC_NATURAL, ADS_BC_DIRICHLET0}; n_d = n_el,d + p <= 1056 (lines are cut into
 *   16, 32 or 64 chunks of at most 33 rows, whichever fits a CTA's shared memory and pads least;
 *   ADS_E_INVAL beyond).
 *   nz = 0: the 2D scheme as the paper prints it (Eqs. 14-16; SURVEY.md §8
 *   row f2): the third axis carries one function with M = 1, K = 0 and no boundary, so that
 *   K = Kx(x)My + Mx(x)Ky and D = Ax(x)Ay exactly; arrays are 1 x n_y x n_x, load/source
 *   vectors along z are [1].  Single-GPU P-wave handles only.
 * Assembles M_d, K_d by Gauss quadrature, factors
 * A_d = M_d + tau^2/4 K_d by banded LU without pivoting, builds
 * the partitioned-elimination tables, allocates device fields on the current
 * CUDA device.  State is zero, t = 0.  Errors: ADS_E_INVAL, ADS_E_SINGULAR,
 * ADS_E_NOMEM, ADS_E_CUDA.  On error *h is NULL. */
int ads_create(ads_handle *h, int nx, int ny, int nz, int p, double tau, int bc);

/* Create a 3D isotropic elasticity solver, 3 components,
 * Lame lambda >= 0, mu > 0, density rho > 0.  Same grid rules as ads_create. */
int ads_create_elastic(ads_handle *h, int nx, int ny, int nz, int p, double tau, int bc,
                       double lambda, double mu, double rho);

/* ---- z-slab decomposition over GPUs ----
 * The grid is cut along z into `world` slabs of balanced plane counts (slab r owns global
 * planes [z_begin, z_begin + z_count), ads_slab_plan).  Per step each slab exchanges p halo
 * planes of U and V with its neighbours (operator z-pass), runs the x and y
 * sweeps locally, solves its diagonal block of A_z, exchanges p "tip" planes and applies the
 * exact SPIKE correction (interface systems 2p x 2p per line; the couplings dropped between
 * non-adjacent interfaces are certified < 2^-64 at create, else ADS_E_INVAL) fused with the
 * kick.  P-wave handles only.
 *
 * ads_get_unique_id: NCCL unique id (128 bytes, caller-owned) for ads_create_dist; rank 0
 *   creates it and broadcasts it (e.g. with torch.distributed).  Host-only call.
 * ads_slab_plan: host-only slab extent of `rank` for nz ELEMENTS (nz + p planes).
 * ads_create_dist: one slab per process/GPU; collective over the `world` ranks (NCCL
 *   communicator on `device`).  State I/O (set_state/get_state) uses the LOCAL planes
 *   (z_count x n_y x n_x doubles); ads_energy returns the global energies (NCCL allreduce).
 * ads_create_virtual: all `nslabs` slabs on the current device in one handle, exchanging by
 *   device copies -- runs the distributed algorithm on one GPU (parity tests); state I/O
 *   uses the global arrays.
 * ads_local_extent: the handle's owned global planes. */
/* Change the step size to tau > 0 at the current step n: the factor tables
 * of A_d = M_d + tau^2/4 K_d are rebuilt and the run continues from the
 * same physical state (U_n, udot_n) at the same time t_n: the half-kick start is redone at t_n,
 * a_n = D^-1 (F(t_n) - K U_n), V = udot_n + tau/2 a_n (C2).  Later steps use
 * t_m = t_n + (m - n) tau (ads_time).  Without a state only the tables change.  Single-GPU
 * P-wave handles only.  Errors: ADS_E_INVAL (tau <= 0, elasticity, slabs), ADS_E_SINGULAR. */
int ads_set_tau(ads_handle h, double tau);

/* Time scheme (readings R1 and R0).  scheme = 1 (default): reading R1.
 * scheme = 0: the literal Eq. 16, kept to reproduce the printed scheme:
 *   a_{n+1} = D^-1 (F(t_{n+1}) - K (U_n + tau V_n)),  V_{n+1} = V_n + tau/2 a_{n+1},
 *   U_{n+1} = U_n + tau V_{n+1} - tau^2/2 a_{n+1}  (= U_n + tau V_n),  V_0 = udot_0, a_0 = 0,
 * which is inconsistent (continuum limit u'' = Laplace(u)/2; R1).  Under scheme 0
 * ads_get_state returns udot = V and ads_energy's third value is kinetic + potential.  Single-GPU
 * P-wave handles only; the state is invalidated (call ads_set_state again).
 * Errors: ADS_E_INVAL (scheme not 0/1, scheme 0 on elasticity or slabs). */
int ads_set_scheme(ads_handle h, int scheme);

/* ---- exact-in-time modal propagator (§3) ----
 * The split scheme is diagonal in the tensor eigenbasis of the 1D pencils: with
 * K_d Phi_d = M_d Phi_d Lambda_d and Phi_d^T M_d Phi_d = I (Eqs. 17-18), a state
 * maps to modal coordinates c = (Phi_x (x) Phi_y (x) Phi_z)^T M U (load vectors: Phi^T b, no M)
 * and every mode advances on its own by the R1 step:
 *   cP = cU + tau cV;  ca = (g(t_{n+1}) cF - L cP) / delta;  cV += tau ca;  cU = cP,
 *   L = l_i + l_j + l_k,  delta = (1 + eta l_i)(1 + eta l_j)(1 + eta l_k),  eta = tau^2/4
 * (delta is the diagonal of D = A_x (x) A_y (x) A_z).
 *
 * ads_modal_basis: host-only.  The basis of one direction on its active DOFs, na = nel + p
 *   (bc = ADS_BC_NATURAL) or nel + p - 2 (ADS_BC_DIRICHLET0, interior restriction C3):
 *   lambda[na] ascending, phi[na * na] row-major, phi[i * na + k] = entry i of eigenvector k
 *   (caller-owned host arrays).  Dense Cholesky of M, Householder tridiagonalisation, implicit QL.
 *   Errors: ADS_E_INVAL (sizes, NULL), ADS_E_SINGULAR (M not SPD or no convergence).
 * ads_modal_advance: advance the handle's state (U, V, a) by nsteps R1 steps in modal space --
 *   the same result as ads_step(h, nsteps) up to rounding.  Without a source the time does not
 *   depend on nsteps (every mode's 2x2 amplification matrix is raised to the nsteps-th power by
 *   repeated squaring); with a source it is linear in nsteps (per-mode recurrence, no sweeps).
 *   Each field is mapped by three dense n_d x n_d products along x, y, z (cuBLAS DGEMM on the FP64
 *   tensor cores): U, V in and out; a_n = D^-1 (F(t_n) - K U_n) by the step's own kernels.  The
 *   bases are computed on the first call (host).
 *   Single-GPU P-wave handles only.  Errors: ADS_E_INVAL (nsteps < 0, elasticity, slabs),
 *   ADS_E_STATE (no state), ADS_E_SINGULAR, ADS_E_CUDA. */
int ads_modal_basis(int nel, int p, int bc, double *lambda, double *phi);
int ads_modal_advance(ads_handle h, long nsteps);

int ads_get_unique_id(unsigned char uid[128]);
int ads_slab_plan(int nz, int p, int world, int rank, int *z_begin, int *z_count);
int ads_create_dist(ads_handle *h, int nx, int ny, int nz, int p, double tau, int bc, int rank, int world,
                    const unsigned char uid[128], int device);
int ads_create_virtual(ads_handle *h, int nx, int ny, int nz, int p, double tau, int bc, int nslabs);
int ads_local_extent(ads_handle h, int *z_begin, int *z_count);

/* z-direction solve of the slab decomposition (north_star: "an NCCL all-to-all transpose or a
 * distributed SPIKE reduced system, whichever measures faster"; the z-line solves are the third
 * sweep).  mode ADS_ZSOLVE_SPIKE (default): each slab solves its diagonal block
 * of A_z and the exact SPIKE correction couples the slabs (above).  mode ADS_ZSOLVE_ALLTOALL:
 * after the local x and y sweeps the right-hand side is transposed -- slab r receives y block
 * [r n_y / G, (r+1) n_y / G) of every global plane (one grouped NCCL send/recv per peer; device
 * copies in a virtual group) --, solved along complete z-lines with the single-GPU factors of
 * A_z, transposed back and applied by the kick.  Both give the same result up to rounding.  The
 * first switch to ADS_ZSOLVE_ALLTOALL allocates 3 slab-sized buffers per slab (4 on an NCCL rank).
 * Collective on NCCL slabs (every rank must call it with the same mode).  Errors: ADS_E_INVAL
 * (not a slab handle, bad mode, more than 64 slabs or fewer y rows than slabs). */
#define ADS_ZSOLVE_SPIKE 0
#define ADS_ZSOLVE_ALLTOALL 1
int ads_set_zsolve(ads_handle h, int mode);

/* Attach a CUDA stream (cudaStream_t passed as void*).  NULL (which is also what
 * torch.cuda.current_stream().cuda_stream is for PyTorch's default stream) selects the
 * library's own stream, a blocking stream that is ordered against the legacy default
 * stream: work PyTorch queues there before/after a call is seen by/sees the library's. */
int ads_set_stream(ads_handle h, void *cuda_stream);

/* Host-side 1D helpers for separable data (L2 projection).
 * ads_load_vector: out[a] = int_0^1 f(x) N_a(x) dx in direction d (0=x,1=y,2=z),
 *   f = sin(pi x) (ADS_FUNC_SIN) or exp(-(x-c)^2/(2 sigma^2)) (ADS_FUNC_GAUSS),
 *   8 Gauss points per element (C4); Dirichlet entries zeroed.
 *   out: host array of n_d doubles.
 * ads_mass_solve_1d: x <- M_d^{-1} x in place (host array of n_d doubles), with
 *   the Dirichlet identity rows when bc = ADS_BC_DIRICHLET0. */
int ads_load_vector(ads_handle h, int d, int func, double c, double sigma, double *out);
int ads_mass_solve_1d(ads_handle h, int d, double *x);

/* Separable source F(t) = amp g(t) (b_x (x) b_y (x) b_z) (C14):
 * bx,by,bz host arrays of n_d doubles (load vectors, dual -- not projected);
 * g = Ricker (1 - 2 pi^2 f0^2 (t-t0)^2) exp(-pi^2 f0^2 (t-t0)^2) or 1 (NONE).
 * F is evaluated at t_{n+1} = (n+1) tau by step n -> n+1.  bx = NULL clears. */
int ads_set_source(ads_handle h, const double *bx, const double *by, const double *bz,
                   int wavelet, double f0, double t0, double amp);

/* Set the state (u0, udot0) and reset t = 0 (C2, half-kick start):
 *   a0 = D^{-1}(F(0) - K u0),  V0 = udot0 + tau/2 a0   (P-wave)
 *   V0 = udot0 + tau/2 D~^{-1}(f(0) - Ups u0)          (elasticity)
 * u: N (3N) doubles; udot may be NULL (= 0).  mem: ADS_MEM_HOST/DEVICE. */
int ads_set_state(ads_handle h, const double *u, const double *udot, int mem);

/* u0 = sum_t amp[t] sx_t (x) sy_t (x) sz_t on component comp[t] (NULL comp = 0),
 * udot0 = 0; then as ads_set_state.  sx: nterms*n_x host doubles (term-major),
 * likewise sy, sz.  The outer products are expanded on the device. */
int ads_set_state_separable(ads_handle h, int nterms, const double *amp, const int *comp,
                            const double *sx, const double *sy, const double *sz);

/* Advance nsteps >= 0 time steps (asynchronous on the handle's stream). */
int ads_step(ads_handle h, int nsteps);

/* Energies (C6), synchronising: out[0] kinetic 1/2 v'Mv with
 * v = V - tau/2 a (rho M for elasticity), out[1] potential 1/2 U'KU (U'Ups U),
 * out[2] the conserved invariant 1/2 V'DV + 1/2 U_n' K U_{n+1}.
 * out: host array of 3 doubles.  Deterministic (fixed reduction order). */
int ads_energy(ads_handle h, double out[3]);

/* Copy out U_n, udot_n = V_n - tau/2 a_n and a_n (any pointer may be NULL).
 * Synchronising.  mem: ADS_MEM_HOST/DEVICE. */
int ads_get_state(ads_handle h, double *u, double *udot, double *a, int mem);

/* Simulation time t_n (n tau, or t_m + (n - m) tau after ads_set_tau changed the step at step
 * m), and step count n. */
double ads_time(ads_handle h);
long ads_step_count(ads_handle h);

/* Grid query: n_d per direction, number of components. */
int ads_dims(ads_handle h, int *nx, int *ny, int *nz, int *ncomp);

/* Unit operations on device arrays of N doubles (for kernel-level parity
 * tests; asynchronous on the handle's stream):
 *   ads_apply_k:   out = K x                  (P-wave operator, fused kernel)
 *   ads_solve_d:   out = (A_x(x)A_y(x)A_z)^{-1} x  (three partitioned sweeps)
 *   ads_sweep:     out = A_d^{-1} x along direction d only
 * x and out must not alias for ads_apply_k. */
int ads_apply_k(ads_handle h, const double *x_dev, double *out_dev);
int ads_solve_d(ads_handle h, const double *x_dev, double *out_dev);
int ads_sweep(ads_handle h, int d, const double *x_dev, double *out_dev);

/* Number of kernel launches issued by the library so far (instrumentation). */
long ads_launch_count(ads_handle h);

/* Per-kernel-class timing with CUDA events recorded on the handle's stream
 * around every launch of the step kernels (instrumentation for bench.py).
 * Classes: 0 = kop (drift+source+K), 1 = sweep x, 2 = sweep y, 3 = sweep z+kick,
 * 4 = modal transform (ads_modal_advance, one launch per direction).
 * ads_profile_enable(h, 1) clears and starts recording; ads_profile_read
 * synchronises and returns total milliseconds and launch counts per class
 * (host arrays of ADS_NPROF entries). */
#define ADS_NPROF 5
int ads_profile_enable(ads_handle h, int on);
int ads_profile_read(ads_handle h, double *ms, long *count);

/* Algorithmic HBM bytes per DOF of one launch of each step kernel class of this handle's
 * P-wave step (host array of ADS_NPROF entries; the roofline numerators of bench.py):
 * kop 32 (reads U, V; writes P, r), sweep x 16, sweep y 16, sweep z + kick 24 (+8 on the last
 * step of a batch, which keeps a).  Zeros for elasticity handles. */
int ads_step_bytes(ads_handle h, double *bytes_per_dof);

/* Last error message of the handle ("" if none); valid until the next call. */
const char *ads_last_error(ads_handle h);

/* Free device memory and the handle.  h may be NULL. */
int ads_destroy(ads_handle h);

#ifdef __cplusplus
}
#endif
#endif /* ADS_B200_H */
