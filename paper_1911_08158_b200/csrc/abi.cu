// abi.cu -- C ABI of the B200 ADS solver (declared in include/ads.h).
//
// Per-step device work on the handle's stream (P-wave, reading R1):
//   kop    (U, V) -> P = U + tau V (into the ping-pong U buffer), r = F(t_{n+1}) - K P
//   sweep x   r -> w          sweep y   w -> r          sweep z + kick   r -> V += tau a (a kept on the last step)
// Four kernel launches per step, no host synchronisation.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <new>
#include <string>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges appear in nsys / ncu when a tool is attached

#include "../../include/ads.h"
#include "host_setup.h"
#include "kernels.cuh"

using namespace ads;

namespace {

struct DirDev {
    double *mband = nullptr, *kband = nullptr, *aband = nullptr;  // [n][2p+1]
    double *bband = nullptr, *btband = nullptr;                    // elasticity: B, B^T
    double *wzband = nullptr;                                      // K in difference form [n][2p]
    double wzrow[2 * kMaxP] = {};                                  // its Toeplitz interior row
    double *slband = nullptr, *ssband = nullptr;                   // elasticity: M + c K (apply)
    int t_lo = 1, t_hi = 0;  // rows [t_lo, t_hi] of M, K are the Toeplitz row (mrow, krow)
    double mrow[2 * kMaxP + 1] = {}, krow[2 * kMaxP + 1] = {};
    SolveTab tab;               // P-wave: A_d = M_d + tau^2/4 K_d
    SolveTab tabL, tabS, tabM;  // elasticity: M + c_L K, M + c_S K, M
};

}  // namespace

struct ads_ctx {
    int nel[3] = {0, 0, 0}, n[3] = {0, 0, 0};
    int p = 0, bc = 0, ncomp = 1;
    // time scheme (ads_set_scheme): 1 = reading R1 (default), 0 = the literal Eq. 16 (reading R0:
    // kick tau/2, no half-kick start, V reported as the velocity; single-GPU P-wave only)
    int scheme = 1;
    // time origin (ads_set_tau): t_n = t_base + (n - n_base) tau; set_state resets it to (0, 0)
    double t_base = 0.0;
    long n_base = 0;
    double tau = 0.0;
    double lam = 0.0, mu = 0.0, rho = 1.0;  // elasticity (ncomp = 3)
    long step = 0;
    bool failed = false, have_state = false;
    std::string err;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int device = 0;
    long launches = 0;
    Geom geo;
    long N = 0;       // logical DOFs n0 n1 n2 (dense caller arrays)
    long Nalloc = 0;  // device field length sz * n2 (rows padded to a multiple of 8 doubles)
    Space1D sp[3];
    LUFactors mass_lu[3];
    DirDev dd[3];
    // fields
    // fields (ncomp components each, component-major, Nalloc doubles per component)
    double *U = nullptr, *U2 = nullptr, *V = nullptr, *A = nullptr, *R = nullptr, *Wk = nullptr;
    double *W = nullptr, *T1 = nullptr, *T2 = nullptr, *T3 = nullptr;  // elasticity scratch
    // z-slab decomposition: dist = 1 NCCL slab (one per process/GPU),
    // 2 virtual group (all slabs of the grid on this device, exchanges by device copies),
    // 3 member slab of a virtual group.  This slab owns global planes [zbeg, zbeg + n[2]);
    // fields carry p halo planes below and above the owned planes (pointers are to the
    // first owned plane).
    int dist = 0, rank = 0, world = 1, zbeg = 0, ngz = 0, halo = 0;
    bool has_prev = false, has_next = false;
    SolveTab tabZ;                                   // A_z restricted to the slab (diagonal block)
    double *Vsp = nullptr, *Wsp = nullptr;           // SPIKE columns [nl][p]
    double *tip_prev = nullptr, *tip_next = nullptr; // p planes received from the neighbours
    double *b0buf = nullptr, *u0buf = nullptr;       // stage-1 interface values (p planes)
    double *b0_prev2 = nullptr, *u0_next2 = nullptr; // the neighbours' stage-1 values
    double qt[2 * kMaxP][2 * kMaxP] = {}, qb[2 * kMaxP][2 * kMaxP] = {};
    double wbp[kMaxP][kMaxP] = {}, vtm[kMaxP][kMaxP] = {}, wbm[kMaxP][kMaxP] = {}, vtn[kMaxP][kMaxP] = {};
    ncclComm_t comm = nullptr;
    // all-to-all z solve (ads_set_zsolve, zsolve = 1): the slab's y block [py0[r], py0[r+1]) of every
    // global plane (the "pencil", geometry pgeo) is gathered from all slabs, solved along z with the
    // global A_z table tabG, and returned into arecv ([q][k][row][x] blocks) for the kick
    int zsolve = 0;
    std::vector<int> py0, z0s, nls;
    Geom pgeo;
    SolveTab tabG;
    double *pen_in = nullptr, *pen_out = nullptr, *arecv = nullptr, *a2a_send = nullptr;
    std::vector<ads_ctx *> members;                  // dist = 2
    ads_ctx *prev = nullptr, *next = nullptr;        // dist = 3
    double *dpartial = nullptr, *dres = nullptr;
    double *stage = nullptr;  // dense staging buffer of host copies (N doubles, first use)
    // CUDA graphs of two P-wave steps (one per U/U2 parity) replayed by ads_step; the source
    // time comes from a device step counter the z sweep increments
    long *dstep = nullptr;
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    double *gU[2] = {nullptr, nullptr};
    long glaunch[2] = {0, 0};  // kernel launches in each graph (two steps)
    bool graphs_off = false;
    // exact-in-time modal propagator (ads_modal_advance).  The uniform basis is
    // mirror-symmetric, so every mode is even or odd under i <-> n-1-i and each direction's maps
    // split in halves acting on the folded line (t = [u + Ju | u - Ju], folded inside modal_tc.cu):
    //   forward  Q_e (ne x H), Q_o (no x h) of Q = Phi^T M;  inverse  P_e (H x ne), P_o (h x no)
    // (column-major; h = n/2, H = h + n%2).  Modal coordinates along d are ordered [even | odd |
    // unused], eigenvalues mlam in that order (0 on unused), mord = the active mode at each slot.
    bool modal_ready = false;
    double *mQe[3] = {}, *mQo[3] = {}, *mPe[3] = {}, *mPo[3] = {};
    // the same maps for the TMA-fed kernels: leading dimensions padded to multiples of 4 (16-byte
    // TMA strides), Q_e's middle column (odd n) halved (the fold loads u(h) twice)
    double *mQe2[3] = {}, *mQo2[3] = {}, *mPe2[3] = {}, *mPo2[3] = {};
    int mlqe[3] = {}, mlqo[3] = {}, mlpe[3] = {}, mlpo[3] = {};
    int mne[3] = {0, 0, 0}, mno[3] = {0, 0, 0};
    double *mlam[3] = {nullptr, nullptr, nullptr}, *mf[3] = {nullptr, nullptr, nullptr};
    std::vector<double> mphi_h[3];  // active-block eigenvectors (host, for the load vectors)
    std::vector<int> mord[3];
    double *mg = nullptr;           // g(t_{n+s}) of the forced recurrence
    long mg_cap = 0;
    // source
    double *src[3] = {nullptr, nullptr, nullptr};
    std::vector<double> src_h[3];  // host copies of the load vectors
    bool has_src = false;
    int wavelet = 0;
    double f0 = 0, t0 = 0, amp = 0;
    // elasticity: two side streams and a pool of events for the independent launches of a step
    // (fork/join; inside a graph capture they become parallel branches)
    cudaStream_t side[2] = {nullptr, nullptr};
    cudaEvent_t fev[8] = {};
    std::vector<void *> allocs;
    // bands whose interior rows are one row bitwise (device pointer -> rows [lo, hi], the row):
    // the Kronecker kernel takes a tile's y-pass coefficients from its parameters there
    struct ToepRow {
        const double *dev;
        int lo, hi;
        double row[2 * kMaxP + 1];
    };
    std::vector<ToepRow> toep;
    // profiling (ads_profile_enable): event pairs per kernel class
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_rec;
};

namespace {

int fail(ads_ctx *h, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (h) {
        h->err = buf;
        if (code == ADS_E_CUDA) h->failed = true;
    }
    return code;
}

#define CUDA_TRY(h, call)                                                                        \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess) return fail(h, ADS_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

int dalloc(ads_ctx *h, void **p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();
        return fail(h, ADS_E_NOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    }
    h->allocs.push_back(*p);
    return ADS_OK;
}

// release one dalloc'd buffer (after the stream has drained: launches may still read it)
int dfree(ads_ctx *h, const void *p) {
    for (size_t i = 0; i < h->allocs.size(); ++i)
        if (h->allocs[i] == p) {
            if (h->stream) cudaStreamSynchronize(h->stream);
            cudaFree(h->allocs[i]);
            h->allocs.erase(h->allocs.begin() + (long)i);
            return ADS_OK;
        }
    return ADS_E_INVAL;
}

template <class T>
int upload(ads_ctx *h, T **dst, const std::vector<T> &v) {
    size_t bytes = sizeof(T) * (v.empty() ? 1 : v.size());
    int rc = dalloc(h, (void **)dst, bytes);
    if (rc) return rc;
    if (!v.empty()) CUDA_TRY(h, cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return ADS_OK;
}

cudaEvent_t next_event(ads_ctx *h) {
    if (h->ev_used == h->ev_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        h->ev_pool.push_back(e);
    }
    return h->ev_pool[h->ev_used++];
}

// bracket one launch of kernel class `cls` with events on the handle's stream
struct ProfScope {
    ads_ctx *h;
    int cls;
    cudaEvent_t e0 = nullptr;
    ProfScope(ads_ctx *h_, int cls_) : h(h_), cls(cls_) {
        if (h->prof && (e0 = next_event(h))) cudaEventRecord(e0, h->stream);
    }
    ~ProfScope() {
        if (!e0) return;
        cudaEvent_t e1 = next_event(h);
        if (!e1) return;
        cudaEventRecord(e1, h->stream);
        h->prof_rec.push_back({cls, {e0, e1}});
    }
};

int check_launch(ads_ctx *h, const char *what) {
    h->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(h, ADS_E_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
    return ADS_OK;
}

double ricker(double t, double f0, double t0) {
    const double kPi = 3.141592653589793238462643383;
    double x = kPi * f0 * (t - t0);
    x = x * x;
    return (1.0 - 2.0 * x) * std::exp(-x);
}

// global plane count for the Dirichlet mask of z, 0 when z has no boundary (2D axis)
int zmask(const ads_ctx *m) { return m->sp[2].bc == ADS_BC_DIRICHLET0 ? m->ngz : 0; }

// time of step n (the step size may have changed at n_base, ads_set_tau)
double time_at(const ads_ctx *h, long n) { return h->t_base + (double)(n - h->n_base) * h->tau; }

// kick coefficient of V += c a and the offset of the reported velocity udot = V - c' a
double kick_coef(const ads_ctx *h) { return h->scheme == 1 ? h->tau : 0.5 * h->tau; }
double vel_corr(const ads_ctx *h) { return h->scheme == 1 ? 0.5 * h->tau : 0.0; }

double source_g(const ads_ctx *h, double t) {
    if (!h->has_src) return 0.0;
    return h->wavelet == ADS_WAVELET_RICKER ? h->amp * ricker(t, h->f0, h->t0) : h->amp;
}

// Factor A (band, Dirichlet identity rows already set) and build the device tables of
// the partitioned sweeps (host_setup.h PartTables; kernels.cuh SolveTab).
int dfree(ads_ctx *h, const void *p);

int make_solve_tab(ads_ctx *h, const Band &A, const char *what, SolveTab &tab) {
    const int n = A.n, p = A.p;
    LUFactors f;
    if (banded_lu(A, f, /*freeze=*/true)) return fail(h, ADS_E_SINGULAR, "%s singular", what);
    // chunking: 32 chunks, or 16 chunks of at most 17 rows when that pads the line less (e.g.
    // 258 rows: 16 x 17 instead of 32 x 9 -- per-tile overheads are amortised over longer chunks),
    // or 64 chunks of at most 17 rows for lines beyond 544 rows (33-row chunks held in registers
    // ran at a third of the bandwidth) when their tables fit the shared memory of a CTA (the
    // identity-padded rows of 64 x 17 land in the edge-record table: p = 4, 5 lines of 577..865
    // rows do not fit and keep 32 x 33)
    const int L32 = choose_chunk_len(n, p, kSweepChunks);
    const int L16 = choose_chunk_len(n, p, 16), L64 = choose_chunk_len(n, p, 64);
    std::vector<std::pair<int, int>> cand;  // (C, L) in order of preference
    if (L16 != 0 && L16 <= 17 && (L32 == 0 || 16 * L16 < kSweepChunks * L32)) cand.push_back({16, L16});
    else if ((L32 == 0 || L32 > 17) && L64 != 0 && L64 <= 17) cand.push_back({64, L64});
    if (L32 != 0) cand.push_back({kSweepChunks, L32});
    if (cand.empty()) return fail(h, ADS_E_INVAL, "%s: n = %d has no supported chunking", what, n);
    for (size_t ci = 0; ci < cand.size(); ++ci) {
        const int C = cand[ci].first, L = cand[ci].second;
        // pad the factors to C*L rows with identity rows: every chunk has length L
        const int npad = C * L;
        LUFactors fp = f;
        fp.n = npad;
        fp.l.resize((size_t)npad * p, 0.0);
        fp.us.resize((size_t)npad * p, 0.0);
        fp.dinv.resize(npad, 1.0);
        PartTables pt;
        build_part_tables(fp, C, L, pt);
        SolveTab t;
        t.n = n;
        t.L = L;
        t.C = C;
        t.Kf = pt.Kf;
        t.Kb = pt.Kb;
        // uniform region aligned to whole chunks: chunks [c_lo, c_hi) lie inside [i_lo, i_hi)
        const int c_lo = (f.i_lo + L - 1) / L, c_hi = f.i_hi / L;
        t.c_lo = c_hi > c_lo ? c_lo : 0;
        t.c_hi = c_hi > c_lo ? c_hi : 0;
        if (t.c_hi > t.c_lo) {
            for (int k = 0; k < p; ++k) {
                t.lc[k] = f.l[(size_t)f.i_lo * p + k];
                t.usc[k] = f.us[(size_t)f.i_lo * p + k];
            }
            t.dic = f.dinv[f.i_lo];
            const int s0 = t.c_lo * L;  // any uniform chunk: its responses are bitwise identical
            for (int j = 0; j < L; ++j)
                for (int m = 0; m < p; ++m) {
                    t.Gf[j][m] = pt.gf[(size_t)(s0 + j) * p + m];
                    t.Gb[j][m] = pt.gb[(size_t)(s0 + j) * p + m];
                }
        }
        const long need = std::max(sweep_smem_bytes(p, t, 0), sweep_smem_bytes(p, t, 1));
        if (need < 0 || need > kMaxSmemPerCta) {
            if (ci + 1 < cand.size()) continue;
            return fail(h, ADS_E_INVAL, "%s: n = %d needs %ld B of shared memory per sweep tile", what, n, need);
        }
        int rc;
        double *l, *us, *dinv, *Tf, *Rb;
        if ((rc = upload(h, &l, fp.l)) || (rc = upload(h, &us, fp.us)) || (rc = upload(h, &dinv, fp.dinv)) ||
            (rc = upload(h, &Tf, pt.Tf)) || (rc = upload(h, &Rb, pt.Rb)))
            return rc;
        // tables this handle built before (ads_set_tau rebuilds them): released, not leaked
        for (const double *old : {tab.l, tab.us, tab.dinv, tab.Tf, tab.Rb})
            if (old) dfree(h, old);
        t.l = l;
        t.us = us;
        t.dinv = dinv;
        t.Tf = Tf;
        t.Rb = Rb;
        tab = t;
        return ADS_OK;
    }
    return fail(h, ADS_E_INVAL, "%s: no chunking", what);
}

// M + c K with the Dirichlet identity rows (the matrices the sweeps invert)
Band shifted(const Space1D &s, double c, int bc) {
    Band A(s.n, s.p);
    for (size_t q = 0; q < A.v.size(); ++q) A.v[q] = s.M.v[q] + c * s.K.v[q];
    if (bc == ADS_BC_DIRICHLET0) {
        A.at(0, 0) = 1.0;
        A.at(s.n - 1, s.n - 1) = 1.0;
    }
    return A;
}

// z-slab tables of this slab (distributed exact SPIKE, host_setup.h build_slab_spikes): the
// diagonal block's sweep tables, its spike columns, and the interface inverses towards the
// neighbours.  Every rank recomputes its neighbours' spikes (1D, cheap): no setup traffic.
int build_slab_tables(ads_ctx *h, const Band &A) {
    std::vector<int> z0s, nls;
    slab_plan(h->ngz, h->world, z0s, nls);
    const int r = h->rank, p = h->p, G = h->world, m = 2 * p;
    for (int j = 0; j < G; ++j)
        if (nls[j] < 2 * p + 1) return fail(h, ADS_E_INVAL, "slab %d has %d < 2p+1 planes", j, nls[j]);
    // every rank builds every slab's spikes (1D, cheap) so all ranks take the same decision
    std::vector<SlabSpikes> S(G);
    for (int j = 0; j < G; ++j)
        if (build_slab_spikes(A, z0s[j], nls[j], S[j])) return fail(h, ADS_E_SINGULAR, "slab block %d singular", j);
    std::vector<std::vector<double>> Q(G > 1 ? G - 1 : 0);
    for (int j = 0; j + 1 < G; ++j) {
        const double d = interface_inverse(S[j], S[j + 1], p, Q[j]);
        double qn = 0.0;
        for (int a = 0; a < m; ++a) {
            double rs = 0.0;
            for (int b = 0; b < m; ++b) rs += std::fabs(Q[j][a * m + b]);
            qn = std::max(qn, rs);
        }
        // stage 1 drops couplings of size <= p d; one Jacobi refinement leaves (|Q| p d)^2
        const double e = qn * p * d;
        if (!(e * e < std::ldexp(1.0, -64)))
            return fail(h, ADS_E_INVAL, "slabs too thin for the spike decay (interface %d: %.3g)", j, e * e);
    }
    int rc;
    if ((rc = make_solve_tab(h, S[r].block, "A_z slab", h->tabZ))) return rc;
    if ((rc = upload(h, &h->Vsp, S[r].V)) || (rc = upload(h, &h->Wsp, S[r].W))) return rc;
    auto wbot = [&](int j, double (&o)[kMaxP][kMaxP]) {  // last p rows of W_j
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b) o[a][b] = S[j].W[(size_t)(nls[j] - p + a) * p + b];
    };
    auto vtop = [&](int j, double (&o)[kMaxP][kMaxP]) {  // first p rows of V_j
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b) o[a][b] = S[j].V[(size_t)a * p + b];
    };
    if (h->has_prev) {
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) h->qt[a][b] = Q[r - 1][a * m + b];
        wbot(r - 1, h->wbp);
        vtop(r, h->vtm);
    }
    if (h->has_next) {
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) h->qb[a][b] = Q[r][a * m + b];
        wbot(r, h->wbm);
        vtop(r + 1, h->vtn);
    }
    return ADS_OK;
}

// rows of a band [n][2p+1] equal to its middle row bitwise: the largest range around the middle
void note_toeplitz(ads_ctx *h, const double *dev, const std::vector<double> &b, int n) {
    const int W = 2 * h->p + 1, mid = n / 2;
    auto same = [&](int i) {
        for (int c = 0; c < W; ++c)
            if (b[(size_t)i * W + c] != b[(size_t)mid * W + c]) return false;
        return true;
    };
    ads_ctx::ToepRow r{dev, mid, mid, {}};
    while (r.lo > 0 && same(r.lo - 1)) --r.lo;
    while (r.hi < n - 1 && same(r.hi + 1)) ++r.hi;
    for (int c = 0; c < W; ++c) r.row[c] = b[(size_t)mid * W + c];
    if (n < 3) r.lo = 1, r.hi = 0;
    h->toep.push_back(r);
}

int build_direction(ads_ctx *h, int d) {
    Space1D &s = h->sp[d];
    const int p = h->p;
    if (h->nel[d] == 0) trivial_space(p, s);  // 2D: the third axis (ads_create nz = 0)
    else if (build_space(p, h->nel[d], h->bc, s)) return fail(h, ADS_E_INVAL, "bad 1D space");
    const int n = s.n, W = 2 * p + 1;
    Band Mm = shifted(s, 0.0, s.bc);
    if (banded_lu(Mm, h->mass_lu[d])) return fail(h, ADS_E_SINGULAR, "M_%d singular", d);
    DirDev &D = h->dd[d];
    // Toeplitz interior of M, K (build_space made rows [2p, n-1-2p] bitwise equal)
    if (n - 1 - 2 * p - 2 * p >= 2) {
        D.t_lo = 2 * p;
        D.t_hi = n - 1 - 2 * p;
        for (int c = 0; c < W; ++c) {
            D.mrow[c] = s.M.v[(size_t)D.t_lo * W + c];
            D.krow[c] = s.K.v[(size_t)D.t_lo * W + c];
        }
        for (int i = D.t_lo; i <= D.t_hi; ++i)
            for (int c = 0; c < W; ++c)
                if (s.M.v[(size_t)i * W + c] != D.mrow[c] || s.K.v[(size_t)i * W + c] != D.krow[c]) {
                    D.t_lo = 1;
                    D.t_hi = 0;
                }
    }
    int rc;
    char what[32];
    if (h->ncomp == 1) {
        // P-wave: A_d = M_d + tau^2/4 K_d (eta = tau^2/4 PAPER.md:173)
        const double eta = h->tau * h->tau / 4.0;
        Band A = shifted(s, eta, s.bc);
        snprintf(what, sizeof what, "A_%d", d);
        if (d == 2 && h->dist) {
            if ((rc = build_slab_tables(h, A))) return rc;
        } else if ((rc = make_solve_tab(h, A, what, D.tab))) {
            return rc;
        }
        if ((rc = upload(h, &D.aband, A.v))) return rc;
    } else {
        // elasticity: S_i = rho (x)_d (M_d + c_{i,d} K_d), c = tau^2/(4 rho) (2mu+lam | mu)
        // (Eq. 37, 3D reading DESIGN.md E1); B_d for the coupling blocks
        const double cl = h->tau * h->tau / (4.0 * h->rho) * (2.0 * h->mu + h->lam);
        const double cs = h->tau * h->tau / (4.0 * h->rho) * h->mu;
        Band AL = shifted(s, cl, s.bc), AS = shifted(s, cs, s.bc);
        if (d == 0)  // S_i = rho (x)_d (...): the density goes into the x factor, (rho A)^-1 = A^-1 / rho
            for (auto *B : {&AL, &AS})
                for (double &v : B->v) v *= h->rho;
        snprintf(what, sizeof what, "SL_%d", d);
        if ((rc = make_solve_tab(h, AL, what, D.tabL))) return rc;
        snprintf(what, sizeof what, "SS_%d", d);
        if ((rc = make_solve_tab(h, AS, what, D.tabS))) return rc;
        snprintf(what, sizeof what, "M_%d", d);
        if ((rc = make_solve_tab(h, Mm, what, D.tabM))) return rc;
        Band BT(n, p);
        for (int i = 0; i < n; ++i)
            for (int j = i - p; j <= i + p; ++j)
                if (j >= 0 && j < n) BT.at(i, j) = s.B.get(j, i);
        // the apply bands: boundary rows/columns stay zero (inputs and outputs vanish there)
        Band SLa(n, p), SSa(n, p);
        for (size_t q = 0; q < SLa.v.size(); ++q) {
            SLa.v[q] = s.M.v[q] + cl * s.K.v[q];
            SSa.v[q] = s.M.v[q] + cs * s.K.v[q];
        }
        if ((rc = upload(h, &D.bband, s.B.v)) || (rc = upload(h, &D.btband, BT.v)) ||
            (rc = upload(h, &D.slband, SLa.v)) || (rc = upload(h, &D.ssband, SSa.v)))
            return rc;
        note_toeplitz(h, D.bband, s.B.v, n);
        note_toeplitz(h, D.btband, BT.v, n);
        note_toeplitz(h, D.slband, SLa.v, n);
        note_toeplitz(h, D.ssband, SSa.v, n);
    }
    std::vector<double> mb(s.M.v), kb(s.K.v), wz;
    diff_weights(s, wz);
    if (D.t_hi > D.t_lo)
        for (int m = 0; m < 2 * p; ++m) D.wzrow[m] = wz[(size_t)D.t_lo * 2 * p + m];
    if ((rc = upload(h, &D.mband, mb)) || (rc = upload(h, &D.kband, kb)) || (rc = upload(h, &D.wzband, wz))) return rc;
    note_toeplitz(h, D.mband, mb, n);
    return ADS_OK;
}

// NVTX range over an ABI call (a no-op without an attached tool)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// every ABI entry works on the handle's device (the one current at ads_create), and restores the
// caller's current device on return
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(const ads_ctx *h) {
        int cur = 0;
        if (h && cudaGetDevice(&cur) == cudaSuccess && cur != h->device && cudaSetDevice(h->device) == cudaSuccess)
            prev = cur;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int guard(ads_ctx *h) {
    if (!h) return ADS_E_INVAL;
    if (h->failed) return ADS_E_STATE;
    return ADS_OK;
}

// ---- step pieces ----
int run_kop(ads_ctx *h, const double *U, const double *V, double tau_d, double g, double sign, double *Pout,
            double *r, bool devsrc = false, const double *kw = nullptr, const double *Ph = nullptr) {
    KopArgs a;
    a.Ph = Ph;
    a.U = U;
    a.V = V;
    a.Pout = Pout;
    a.r = r;
    a.tau = tau_d;
    a.g = g;
    a.sign = sign;
    if (h->has_src && (g != 0.0 || devsrc)) {
        a.bx = h->src[0];
        a.by = h->src[1];
        a.bz = h->src[2];
        if (devsrc) {  // g from the device step counter at replay time
            a.dstep = h->dstep;
            a.wav = h->wavelet == ADS_WAVELET_RICKER;
            a.f0 = h->f0;
            // device time (n + 1) tau_g; shifting the wavelet centre moves the time origin
            a.t0 = h->t0 - (h->t_base - (double)h->n_base * h->tau);
            a.amp = h->amp;
            a.tau_g = h->tau;
        }
    }
    a.mx = h->dd[0].mband;
    a.kx = h->dd[0].kband;
    a.my = h->dd[1].mband;
    a.ky = h->dd[1].kband;
    a.mz = h->dd[2].mband;
    a.kz = h->dd[2].kband;
    a.geo = h->geo;
    a.zlen = 0;
    if (h->halo) {  // slab: band rows / source entries are global rows, halo planes exist
        a.zoff = h->zbeg;
        a.zv0 = -h->halo;
        a.zv1 = h->n[2] + h->halo;
    }
    for (int d = 0; d < 3; ++d) {
        a.ilo[d] = h->dd[d].t_lo;
        a.ihi[d] = h->dd[d].t_hi;
        a.kw[d] = kw ? kw[d] : 1.0;
        for (int c = 0; c < 2 * h->p + 1; ++c) {
            a.mc[d][c] = h->dd[d].mrow[c];
            a.kc[d][c] = a.kw[d] * h->dd[d].krow[c];
        }
    }
    a.wz = h->dd[2].wzband;
    a.pdl = h->ncomp == 3;  // the elastic step launches with programmatic dependencies
    if (h->sp[2].bc == ADS_BC_DIRICHLET0) {
        a.zd0 = 0;
        a.zd1 = h->ngz - 1;
    }
    for (int m = 0; m < 2 * h->p; ++m) a.wzc[m] = a.kw[2] * h->dd[2].wzrow[m];
    ProfScope ps(h, 0);
    const int lr = launch_kop(h->p, a, h->stream);
    if (lr == -2) return fail(h, ADS_E_CUDA, "kop: TMA descriptor encoding failed");
    if (lr) return fail(h, ADS_E_INVAL, "kop: unsupported p");
    return check_launch(h, "kop");
}

int run_sweep_tab(ads_ctx *h, int d, const SolveTab &tab, const double *in, double *out, double *V, double kick,
                  long *inc = nullptr, const Geom *geo = nullptr) {
    SweepArgs a;
    a.dstep_inc = inc;
    a.in = in;
    a.out = out;
    a.V = V;
    a.kick = kick;
    a.t = tab;
    a.geo = geo ? *geo : h->geo;
    a.dir = d;
    a.mode = V ? 1 : 0;
    a.pdl = h->ncomp == 3;
    ProfScope ps(h, 1 + d);
    if (tab.n == 1) {  // the 2D axis: a 1 x 1 system per line (P-wave A_z = M_z + eta K_z = 1)
        const double a00 = h->sp[d].M.get(0, 0) + 0.25 * h->tau * h->tau * h->sp[d].K.get(0, 0);
        launch_line1(in, out, V, 1.0 / a00, kick, inc, h->geo, h->stream);
        return check_launch(h, "line1");
    }
    // the z blocks of thin slabs: one thread per line (ADS_LINE_SWEEP=0 disables)
    static const bool line_ok = [] {
        const char *e = std::getenv("ADS_LINE_SWEEP");
        return !(e && e[0] == '0');
    }();
    if (line_ok && &tab == &h->tabZ && out && tab.n <= kLineSweepMax && launch_line_sweep(h->p, a, h->stream) == 0)
        return check_launch(h, "line sweep");
    const int lr = launch_sweep(h->p, a, h->stream);
    if (lr == -2) return fail(h, ADS_E_CUDA, "sweep: TMA descriptor encoding failed");
    if (lr) return fail(h, ADS_E_INVAL, "sweep: unsupported p/chunk");
    return check_launch(h, "sweep");
}

int run_sweep(ads_ctx *h, int d, const double *in, double *out, double *V, double kick) {
    return run_sweep_tab(h, d, h->dd[d].tab, in, out, V, kick);
}

int run_solve(ads_ctx *h, const double *r_in, double *scratch, double *r2, double *aout, double *V, double kick) {
    int rc;
    if ((rc = run_sweep(h, 0, r_in, scratch, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 1, scratch, r2, nullptr, 0.0))) return rc;
    return run_sweep_tab(h, 2, h->dd[2].tab, r2, aout, V, kick, h->dstep);
}

// one single-GPU P-wave step n -> n+1 (drift + RHS, three sweeps, kick); devsrc: source time
// from the device step counter (graph capture), else from the host counter
int enqueue_step(ads_ctx *h, bool keepA, bool devsrc) {
    const double t1 = time_at(h, h->step + 1);  // F at t_{n+1} (C14)
    int rc;
    if ((rc = run_kop(h, h->U, h->V, h->tau, devsrc ? 0.0 : source_g(h, t1), -1.0, h->U2, h->R, devsrc))) return rc;
    if ((rc = run_solve(h, h->R, h->Wk, h->R, keepA ? h->A : nullptr, h->V, kick_coef(h)))) return rc;
    std::swap(h->U, h->U2);
    return ADS_OK;
}

int el_step(ads_ctx *h);

// graph of two steps for the current U/U2 parity (captured once, replayed); *nl = its launches
int step_graph(ads_ctx *h, cudaGraphExec_t *out, long *nl) {
    const int par = h->U == h->gU[1] ? 1 : (h->U == h->gU[0] ? 0 : -1);
    if (par >= 0 && h->gexec[par]) {
        *out = h->gexec[par];
        *nl = h->glaunch[par];
        return ADS_OK;
    }
    const int slot = h->gexec[0] ? 1 : 0;
    double *u0 = h->U;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return ADS_E_CUDA;
    const long launches = h->launches;
    // P-wave: source time from the device step counter; elasticity has no source term
    auto one = [&] { return h->ncomp == 3 ? el_step(h) : enqueue_step(h, false, true); };
    int rc = one();
    if (rc == ADS_OK) rc = one();
    const long captured = h->launches - launches;
    h->launches = launches;
    const cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    if (rc != ADS_OK || e != cudaSuccess || !g) {
        cudaGetLastError();
        if (g) cudaGraphDestroy(g);
        h->err.clear();
        h->failed = false;
        h->graphs_off = true;  // fall back to direct launches for good
        return ADS_E_CUDA;
    }
    cudaGraphExec_t ex = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) {
        cudaGetLastError();
        h->graphs_off = true;
        return ADS_E_CUDA;
    }
    h->gexec[slot] = ex;
    h->gU[slot] = u0;
    h->glaunch[slot] = captured;
    *out = ex;
    *nl = captured;
    return ADS_OK;
}

void drop_graphs(ads_ctx *h) {
    for (int i = 0; i < 2; ++i) {
        if (h->gexec[i]) cudaGraphExecDestroy(h->gexec[i]);
        h->gexec[i] = nullptr;
        h->gU[i] = nullptr;
    }
}

int dist_solve(ads_ctx *G, double tau_d, double g, double kick, bool keepA);

int init_state(ads_ctx *h) {
    // half-kick start (C2): a0 = D^-1 (F(0) - K u0); V0 = udot0 + tau/2 a0
    int rc;
    if (h->dist) {
        if ((rc = dist_solve(h, 0.0, source_g(h, 0.0), 0.5 * h->tau, true))) return rc;
    } else if (h->scheme == 0) {  // literal Eq. 16 (R0): no start procedure, a_0 = 0, V_0 = udot_0
        CUDA_TRY(h, cudaMemsetAsync(h->A, 0, sizeof(double) * h->Nalloc, h->stream));
        CUDA_TRY(h, cudaMemsetAsync(h->dstep, 0, sizeof(long), h->stream));
    } else {
        if ((rc = run_kop(h, h->U, h->V, 0.0, source_g(h, 0.0), -1.0, nullptr, h->R))) return rc;
        if ((rc = run_sweep(h, 0, h->R, h->Wk, nullptr, 0.0))) return rc;
        if ((rc = run_sweep(h, 1, h->Wk, h->R, nullptr, 0.0))) return rc;
        if ((rc = run_sweep(h, 2, h->R, h->A, h->V, 0.5 * h->tau))) return rc;
        CUDA_TRY(h, cudaMemsetAsync(h->dstep, 0, sizeof(long), h->stream));  // device step counter n = 0
    }
    h->step = 0;
    h->t_base = 0.0;
    h->n_base = 0;
    h->have_state = true;
    for (ads_ctx *m : h->members) {
        m->step = 0;
        m->have_state = true;
    }
    return ADS_OK;
}

// ---------------------------------------------------------------------------------------
// 3D isotropic elasticity (readings C10-C13, E1).  Fields are
// component-major: component c of a field F is F + c * Nalloc.
//   Ups_ii = (2mu+lam) K_(i) + mu sum_{d != i} K_(d) = mu K + (mu+lam) K_(i)
//   Ups_ik = mu [B]_k [B^T]_i + lam [B]_i [B^T]_k      (i != k, M in the third direction)
// where [F]_d is F acting along direction d.  Kronecker triples run as three banded axis
// passes (T1, T2 scratch); K = Kx My Mz + ... runs in the fused operator kernel.
// ---------------------------------------------------------------------------------------
double *comp(double *f, const ads_ctx *h, int c) { return f + (long)c * h->Nalloc; }

// Kronecker y factors: the Toeplitz interior of each Fy_t (ads_ctx::toep) into the kernel arguments
void set_yrows(const ads_ctx *h, KronTerms &k3) {
    for (int t = 0; t < k3.nterms; ++t)
        for (const auto &r : h->toep)
            if (r.dev == k3.fy[t]) {
                k3.fylo[t] = r.lo;
                k3.fyhi[t] = r.hi;
                for (int c = 0; c < 2 * h->p + 1; ++c) k3.fyrow[t][c] = r.row[c];
            }
}

// out = alpha (Fx (x) Fy (x) Fz) in + beta out   (Fd: band [n_d][2p+1], acting along d)
int tri(ads_ctx *h, double *out, const double *in, const double *fx, const double *fy, const double *fz,
        double alpha, double beta) {
    KronTerms k3;
    k3.fx[0] = fx, k3.fy[0] = fy, k3.fz[0] = fz, k3.alpha[0] = alpha;
    set_yrows(h, k3);
    if (launch_kron3(h->p, in, out, k3, beta, h->geo, h->stream)) return fail(h, ADS_E_INVAL, "kron3: unsupported p");
    return check_launch(h, "kron3");
}

// out = (addend or out) + coef Ups_ik in   (i != k): mu [B]_k [B^T]_i + lam [B]_i [B^T]_k, M in
// the third direction -- both triples act on the same input and output: one fused pass
int ups_offdiag(ads_ctx *h, int i, int k, const double *in, double *out, double coef,
                const double *addend = nullptr) {
    KronTerms k3;
    k3.nterms = 2;
    k3.addend = addend;
    const double **F[3] = {k3.fx, k3.fy, k3.fz};
    for (int e = 0; e < 3; ++e) {
        F[e][0] = e == k ? h->dd[e].bband : e == i ? h->dd[e].btband : h->dd[e].mband;
        F[e][1] = e == i ? h->dd[e].bband : e == k ? h->dd[e].btband : h->dd[e].mband;
    }
    k3.alpha[0] = coef * h->mu;
    k3.alpha[1] = coef * h->lam;
    set_yrows(h, k3);
    if (launch_kron3(h->p, in, out, k3, 1.0, h->geo, h->stream)) return fail(h, ADS_E_INVAL, "kron3: unsupported p");
    return check_launch(h, "kron3");
}

// Concurrency of the elastic step: lane 0 is the handle's stream, lanes 1, 2 its side streams.
// after(h, to, from): lane `to` waits for everything enqueued so far on lane `from` (an event);
// on(h, lane, f): run f with the handle's launches going to that lane.
cudaStream_t lane_stream(ads_ctx *h, int lane) { return lane == 0 ? h->stream : h->side[lane - 1]; }
int after(ads_ctx *h, int to, int from, int ev) {
    CUDA_TRY(h, cudaEventRecord(h->fev[ev], lane_stream(h, from)));
    CUDA_TRY(h, cudaStreamWaitEvent(lane_stream(h, to), h->fev[ev], 0));
    return ADS_OK;
}
template <class F>
int on(ads_ctx *h, int lane, F f) {
    cudaStream_t keep = h->stream;
    h->stream = lane_stream(h, lane);
    const int rc = f();
    h->stream = keep;
    return rc;
}

// out_i (+)= coef (Ups in)_i for all i.  The diagonal blocks go through the fused operator
// kernel: out_i = coef mu K (in_i + tau_d v_i) with the drift written to pout_i if non-null.
// The three components run on three lanes (the off-diagonal blocks read every component's drift,
// so the lanes join between the two phases).
int ups_apply(ads_ctx *h, const double *in, const double *v, double tau_d, double *pout, double *out, double coef) {
    int rc;
    if ((rc = after(h, 1, 0, 0)) || (rc = after(h, 2, 0, 1))) return rc;
    // diagonal blocks Ups_ii = mu K + (mu + lam) K_(i): the operator kernel with direction i's K
    // term weighted (2 mu + lam) / mu
    for (int i = 0; i < 3; ++i) {
        double kw[3] = {1.0, 1.0, 1.0};
        kw[i] = (2.0 * h->mu + h->lam) / h->mu;
        if ((rc = on(h, i, [&] {
                 return run_kop(h, comp((double *)in, h, i), comp((double *)v, h, i), tau_d, 0.0, coef * h->mu,
                                pout ? comp(pout, h, i) : nullptr, comp(out, h, i), false, kw);
             })))
            return rc;
    }
    // every lane waits for every drift: lane 0 joins lanes 1, 2, then lanes 1, 2 wait for lane 0
    if ((rc = after(h, 0, 1, 2)) || (rc = after(h, 0, 2, 3)) || (rc = after(h, 1, 0, 4)) || (rc = after(h, 2, 0, 5)))
        return rc;
    const double *P = pout ? pout : in;  // the drifted field the blocks act on
    for (int i = 0; i < 3; ++i)
        if ((rc = on(h, i, [&] {
                 for (int k = 0; k < 3; ++k) {
                     int r = k != i ? ups_offdiag(h, i, k, comp((double *)P, h, k), comp(out, h, i), coef) : 0;
                     if (r) return r;
                 }
                 return 0;
             })))
            return rc;
    if ((rc = after(h, 0, 1, 6)) || (rc = after(h, 0, 2, 7))) return rc;
    return ADS_OK;
}

// x <- S_i^-1 in (in == nullptr: in place),  S_i = rho (x)_d (M_d + c_{i,d} K_d)  (PAPER.md:415-422
// Eq. 37); the x tables carry the factor rho (build_direction)
int s_solve(ads_ctx *h, int i, double *x, const double *in = nullptr) {
    int rc;
    for (int d = 0; d < 3; ++d)
        if ((rc = run_sweep_tab(h, d, d == i ? h->dd[d].tabL : h->dd[d].tabS, d == 0 && in ? in : x, x, nullptr, 0.0)))
            return rc;
    return ADS_OK;
}

// X <- D~^-1 X, D~ = L~ (rho M)^-1 L~^T: predictor x -> y -> z, corrector z -> y -> x
// (Eqs. 35-36 in delta form, E1).  W: 3-component scratch.
int el_dsolve(ads_ctx *h, double *X) {
    const double hh = -0.5 * h->tau * h->tau;
    int rc;
    double *w0 = comp(h->W, h, 0), *w1 = comp(h->W, h, 1), *w2 = comp(h->W, h, 2);
    double *z0 = comp(X, h, 0), *z1 = comp(X, h, 1), *z2 = comp(X, h, 2);
    auto rhoM = [&](double *z, const double *w) {
        return tri(h, z, w, h->dd[0].mband, h->dd[1].mband, h->dd[2].mband, h->rho, 0.0);
    };
    // predictor: w_i = S_i^-1 (X_i - tau^2/2 sum_{j<i} Ups_ij w_j) (the first coupling reads X_i);
    // w_2's coupling to w_0 runs on lane 1 while lane 0 finishes w_1
    if ((rc = s_solve(h, 0, w0, z0))) return rc;
    if ((rc = after(h, 1, 0, 0))) return rc;
    if ((rc = on(h, 1, [&] { return ups_offdiag(h, 2, 0, w0, w2, hh, z2); }))) return rc;
    if ((rc = ups_offdiag(h, 1, 0, w0, w1, hh, z1)) || (rc = s_solve(h, 1, w1))) return rc;
    if ((rc = after(h, 0, 1, 1))) return rc;
    if ((rc = ups_offdiag(h, 2, 1, w1, w2, hh)) || (rc = s_solve(h, 2, w2))) return rc;
    // corrector: z_i = S_i^-1 (rho M w_i - tau^2/2 sum_{j>i} Ups_ij z_j); z_1, z_0's mass products
    // on lanes 1, 2 from the start, z_0's coupling to z_2 on lane 2 once z_2 is final
    if ((rc = after(h, 1, 0, 2)) || (rc = after(h, 2, 0, 3))) return rc;
    if ((rc = on(h, 1, [&] { return rhoM(z1, w1); })) || (rc = on(h, 2, [&] { return rhoM(z0, w0); }))) return rc;
    if ((rc = rhoM(z2, w2)) || (rc = s_solve(h, 2, z2))) return rc;
    if ((rc = after(h, 2, 0, 4)) || (rc = on(h, 2, [&] { return ups_offdiag(h, 0, 2, z2, z0, hh); }))) return rc;
    if ((rc = after(h, 0, 1, 5))) return rc;
    if ((rc = ups_offdiag(h, 1, 2, z2, z1, hh)) || (rc = s_solve(h, 1, z1))) return rc;
    if ((rc = after(h, 0, 2, 6))) return rc;
    if ((rc = ups_offdiag(h, 0, 1, z1, z0, hh)) || (rc = s_solve(h, 0, z0))) return rc;
    return ADS_OK;
}

// one elastic step: P = U + tau V (-> U2), A = -Ups P, A <- D~^-1 A, V += tau A, U <- P
int el_step(ads_ctx *h) {
    int rc;
    if ((rc = ups_apply(h, h->U, h->V, h->tau, h->U2, h->A, -1.0))) return rc;
    if ((rc = el_dsolve(h, h->A))) return rc;
    launch_axpby(3 * h->Nalloc, h->tau, h->A, 1.0, h->V, h->stream, true);
    if ((rc = check_launch(h, "axpby"))) return rc;
    std::swap(h->U, h->U2);
    return ADS_OK;
}

// half-kick start: V0 = udot0 + tau/2 D~^-1 (-Ups U0)   (C13)
int el_init(ads_ctx *h) {
    int rc;
    if ((rc = ups_apply(h, h->U, h->U, 0.0, nullptr, h->A, -1.0))) return rc;
    if ((rc = el_dsolve(h, h->A))) return rc;
    launch_axpby(3 * h->Nalloc, 0.5 * h->tau, h->A, 1.0, h->V, h->stream);
    if ((rc = check_launch(h, "axpby"))) return rc;
    h->step = 0;
    h->have_state = true;
    return ADS_OK;
}

// energies (C6 for elasticity): kinetic 1/2 rho v'Mv (v = V - tau/2 a),
// potential 1/2 U'Ups U, invariant 1/2 V'D~V + 1/2 U'Ups(U + tau V) with
// V'D~V = sum_i g_i' (rho M)^-1 g_i, g_i = S_i V_i + tau^2/2 sum_{j>i} Ups_ij V_j.
int el_energy(ads_ctx *h, double res[3]) {
    const long N3 = 3 * h->Nalloc;
    const long fb = sizeof(double) * h->Nalloc;
    int rc;
    // the 8 dot products land in dres[0..7] on the stream; one copy and one host wait at the end
    // (summed on the host in the same order as before)
    auto dot = [&](long n, const double *x, const double *y, int slot) -> int {
        launch_dot(n, x, y, h->dpartial, h->dres + slot, h->stream);
        return ADS_OK;
    };
    // kinetic
    CUDA_TRY(h, cudaMemcpyAsync(h->W, h->V, sizeof(double) * N3, cudaMemcpyDeviceToDevice, h->stream));
    launch_axpby(N3, -0.5 * h->tau, h->A, 1.0, h->W, h->stream);
    for (int c = 0; c < 3; ++c) {
        if ((rc = tri(h, h->T3, comp(h->W, h, c), h->dd[0].mband, h->dd[1].mband, h->dd[2].mband, h->rho, 0.0)))
            return rc;
        if ((rc = dot(h->Nalloc, comp(h->W, h, c), h->T3, c))) return rc;
    }
    // potential
    if ((rc = ups_apply(h, h->U, h->U, 0.0, nullptr, h->W, 1.0))) return rc;
    if ((rc = dot(N3, h->U, h->W, 3))) return rc;
    // invariant: U' Ups (U + tau V)
    if ((rc = ups_apply(h, h->U, h->V, h->tau, h->U2, h->W, 1.0))) return rc;
    if ((rc = dot(N3, h->U, h->W, 4))) return rc;
    for (int i = 0; i < 3; ++i) {
        double *g = comp(h->W, h, i);
        const double *F[3];
        for (int d = 0; d < 3; ++d) F[d] = d == i ? h->dd[d].slband : h->dd[d].ssband;
        if ((rc = tri(h, g, comp(h->V, h, i), F[0], F[1], F[2], h->rho, 0.0))) return rc;
        for (int j = i + 1; j < 3; ++j)
            if ((rc = ups_offdiag(h, i, j, comp(h->V, h, j), g, 0.5 * h->tau * h->tau))) return rc;
        CUDA_TRY(h, cudaMemcpyAsync(h->T3, g, fb, cudaMemcpyDeviceToDevice, h->stream));
        for (int d = 0; d < 3; ++d)
            if ((rc = run_sweep_tab(h, d, h->dd[d].tabM, h->T3, h->T3, nullptr, 0.0))) return rc;
        launch_axpby(h->Nalloc, 1.0 / h->rho, h->T3, 0.0, h->T3, h->stream);
        if ((rc = dot(h->Nalloc, g, h->T3, 5 + i))) return rc;
    }
    double d[8];
    CUDA_TRY(h, cudaMemcpyAsync(d, h->dres, sizeof d, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    double acc[3] = {0, 0, 0}, inv = 0.0;
    for (int c = 0; c < 3; ++c) acc[0] += d[c];
    acc[1] += d[3];
    acc[2] += d[4];
    for (int i = 0; i < 3; ++i) inv += d[5 + i];
    res[0] = 0.5 * acc[0];
    res[1] = 0.5 * acc[1];
    res[2] = 0.5 * inv + 0.5 * acc[2];
    return ADS_OK;
}

// ---------------------------------------------------------------------------------------
// z-slab decomposition.  Per step, on every slab:
//   1. halo exchange of U, V (p planes per side)       -- NCCL send/recv, or device copies
//   2. fused operator (drift + source + K P) on the owned planes, reading the halos
//   3. x, y sweeps (local), z sweep of the slab's diagonal block (local solve, zero tips)
//   4. tip exchange (first/last p planes of the local z solution)
//   5. exact SPIKE fix-up of the slab (interface inverses, spike columns) fused with the kick
// The dropped couplings of the interface systems are certified < 2^-64 at create.
// ---------------------------------------------------------------------------------------
std::vector<ads_ctx *> slabs_of(ads_ctx *h) {
    if (h->dist == 2) return h->members;
    return {h};
}

#define NCCL_TRY(h, call)                                                                       \
    do {                                                                                        \
        ncclResult_t r_ = (call);                                                               \
        if (r_ != ncclSuccess) return fail(h, ADS_E_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
    } while (0)

// Exchanges between neighbouring z-slabs as one schedule both back ends run: every entry moves
// `count` doubles from region `sr` of slab `src` to region `dr` of slab `dst`.  An NCCL rank posts
// the entries it takes part in (send or receive, one group on its stream); a virtual group copies
// every entry on the device.  The tested virtual path therefore exercises exactly the pairing the
// NCCL path uses.
struct Xfer {
    int src, dst, sr, dr;
    long count;
};
template <class Resolve>
int run_schedule(ads_ctx *G, const std::vector<Xfer> &xs, Resolve res) {
    if (G->dist == 2) {
        for (const Xfer &x : xs) {
            ads_ctx *ms = G->members[x.src], *md = G->members[x.dst];
            CUDA_TRY(md, cudaMemcpyAsync(res(md, x.dr), res(ms, x.sr), sizeof(double) * x.count, cudaMemcpyDeviceToDevice,
                                         md->stream));
        }
    } else if (G->dist == 1) {
        NCCL_TRY(G, ncclGroupStart());
        for (const Xfer &x : xs) {
            if (x.src == G->rank) NCCL_TRY(G, ncclSend(res(G, x.sr), x.count, ncclDouble, x.dst, G->comm, G->stream));
            if (x.dst == G->rank) NCCL_TRY(G, ncclRecv(res(G, x.dr), x.count, ncclDouble, x.src, G->comm, G->stream));
        }
        NCCL_TRY(G, ncclGroupEnd());
    }
    return ADS_OK;
}

// the world's slabs and their plane counts (every rank knows the whole plan)
int slab_count(const ads_ctx *G) { return G->dist == 2 ? (int)G->members.size() : G->world; }

// halo exchange of a field: slab j's last p owned planes -> slab j+1's lower halo, slab j+1's first
// p owned planes -> slab j's upper halo
enum { RG_LOW_OWNED, RG_HIGH_OWNED, RG_LOW_HALO, RG_HIGH_HALO };
int exch_halo(ads_ctx *G, double *ads_ctx::*F) {
    std::vector<Xfer> xs;
    const long hp = (long)G->p * (G->dist == 2 ? G->members[0]->geo.sz : G->geo.sz);
    for (int j = 0; j + 1 < slab_count(G); ++j) {
        xs.push_back({j, j + 1, RG_HIGH_OWNED, RG_LOW_HALO, hp});
        xs.push_back({j + 1, j, RG_LOW_OWNED, RG_HIGH_HALO, hp});
    }
    return run_schedule(G, xs, [F](ads_ctx *m, int r) -> double * {
        const long sz = m->geo.sz, nl = m->n[2], p = m->p;
        double *f = m->*F;
        switch (r) {
            case RG_LOW_OWNED: return f;
            case RG_HIGH_OWNED: return f + (nl - p) * sz;
            case RG_LOW_HALO: return f - p * sz;
            default: return f + nl * sz;
        }
    });
}

// tips of the local z solution X = Wk: tip_prev <- previous slab's last p planes,
// tip_next <- next slab's first p planes
enum { RG_WK_LOW, RG_WK_HIGH, RG_TIP_PREV, RG_TIP_NEXT };
int exch_tips(ads_ctx *G) {
    std::vector<Xfer> xs;
    const long hp = (long)G->p * (G->dist == 2 ? G->members[0]->geo.sz : G->geo.sz);
    for (int j = 0; j + 1 < slab_count(G); ++j) {
        xs.push_back({j, j + 1, RG_WK_HIGH, RG_TIP_PREV, hp});
        xs.push_back({j + 1, j, RG_WK_LOW, RG_TIP_NEXT, hp});
    }
    return run_schedule(G, xs, [](ads_ctx *m, int r) -> double * {
        const long sz = m->geo.sz, nl = m->n[2], p = m->p;
        switch (r) {
            case RG_WK_LOW: return m->Wk;
            case RG_WK_HIGH: return m->Wk + (nl - p) * sz;
            case RG_TIP_PREV: return m->tip_prev;
            default: return m->tip_next;
        }
    });
}

void zargs(ads_ctx *m, ZfixArgs &a) {
    a.X = m->Wk;
    a.tip_prev = m->has_prev ? m->tip_prev : nullptr;
    a.tip_next = m->has_next ? m->tip_next : nullptr;
    a.b0_prev2 = m->rank >= 2 ? m->b0_prev2 : nullptr;
    a.u0_next2 = m->rank + 2 < m->world ? m->u0_next2 : nullptr;
    a.b0buf = m->b0buf;
    a.u0buf = m->u0buf;
    a.Vsp = m->Vsp;
    a.Wsp = m->Wsp;
    a.Vf = m->V;
    for (int i = 0; i < 2 * kMaxP; ++i)
        for (int j = 0; j < 2 * kMaxP; ++j) {
            a.qt[i][j] = m->qt[i][j];
            a.qb[i][j] = m->qb[i][j];
        }
    for (int i = 0; i < kMaxP; ++i)
        for (int j = 0; j < kMaxP; ++j) {
            a.wbp[i][j] = m->wbp[i][j];
            a.vtm[i][j] = m->vtm[i][j];
            a.wbm[i][j] = m->wbm[i][j];
            a.vtn[i][j] = m->vtn[i][j];
        }
    a.geo = m->geo;
}

int run_zint(ads_ctx *m) {
    ZfixArgs a;
    zargs(m, a);
    ProfScope ps(m, 3);
    if (launch_zint(m->p, a, m->stream)) return fail(m, ADS_E_INVAL, "zint: unsupported p");
    return check_launch(m, "zint");
}

int run_zfix(ads_ctx *m, double *Aout, double kick) {
    ZfixArgs a;
    zargs(m, a);
    a.A = Aout;
    a.kick = kick;
    ProfScope ps(m, 3);
    if (launch_zfix(m->p, a, m->stream)) return fail(m, ADS_E_INVAL, "zfix: unsupported p");
    return check_launch(m, "zfix");
}

// stage-1 values: b0buf -> next slab's b0_prev2, u0buf -> previous slab's u0_next2 (slab j+1 needs
// b_{j-1}^0, which exists for j >= 1; slab j-1 needs u_{j+1}^0, which exists for j <= G-2)
enum { RG_B0, RG_U0, RG_B0_PREV2, RG_U0_NEXT2 };
int exch_stage1(ads_ctx *G) {
    std::vector<Xfer> xs;
    const int W = slab_count(G);
    const long hp = (long)G->p * (G->dist == 2 ? G->members[0]->geo.sz : G->geo.sz);
    for (int j = 1; j + 1 < W; ++j) {
        xs.push_back({j, j + 1, RG_B0, RG_B0_PREV2, hp});
        xs.push_back({j, j - 1, RG_U0, RG_U0_NEXT2, hp});
    }
    return run_schedule(G, xs, [](ads_ctx *m, int r) -> double * {
        switch (r) {
            case RG_B0: return m->b0buf;
            case RG_U0: return m->u0buf;
            case RG_B0_PREV2: return m->b0_prev2;
            default: return m->u0_next2;
        }
    });
}

// All-to-all z solve (ads_set_zsolve(h, ADS_ZSOLVE_ALLTOALL)), after the local x and y sweeps left
// each slab's right-hand side in R: (1) transpose -- slab s sends the rows of y block q of its
// owned planes to slab q, which stacks them by global plane into its pencil (the full z extent of
// y block q); (2) every pencil solves A_z along its complete z-lines (the single-GPU table); (3) the
// planes of slab s in pencil q return to slab s (arecv block q); (4) kick V += kick a, A = a.
// NCCL ranks pack their strided send blocks with a 2D device copy; a virtual group copies directly.
int a2a_zsolve(ads_ctx *G, double kick, bool keepA) {
    const int W = slab_count(G);
    auto pny = [](const ads_ctx *m, int q) { return m->py0[q + 1] - m->py0[q]; };
    if (G->dist == 2) {
        for (ads_ctx *s_ : G->members)
            for (int q = 0; q < W; ++q) {
                ads_ctx *t = G->members[q];
                const size_t w = sizeof(double) * pny(s_, q) * s_->geo.sy;
                CUDA_TRY(G, cudaMemcpy2DAsync(t->pen_in + (long)s_->zbeg * t->pgeo.sz, sizeof(double) * t->pgeo.sz,
                                              s_->R + (long)s_->py0[q] * s_->geo.sy, sizeof(double) * s_->geo.sz, w,
                                              s_->n[2], cudaMemcpyDeviceToDevice, G->stream));
            }
    } else {
        const int me = G->rank, nl = G->n[2];
        const long sy = G->geo.sy;
        for (int q = 0; q < W; ++q) {
            const size_t w = sizeof(double) * pny(G, q) * sy;
            double *dst = q == me ? G->pen_in + (long)G->zbeg * G->pgeo.sz : G->a2a_send + (long)nl * G->py0[q] * sy;
            CUDA_TRY(G, cudaMemcpy2DAsync(dst, q == me ? sizeof(double) * G->pgeo.sz : w, G->R + (long)G->py0[q] * sy,
                                          sizeof(double) * G->geo.sz, w, nl, cudaMemcpyDeviceToDevice, G->stream));
        }
        NCCL_TRY(G, ncclGroupStart());
        for (int q = 0; q < W; ++q) {
            if (q == me) continue;
            NCCL_TRY(G, ncclSend(G->a2a_send + (long)nl * G->py0[q] * sy, (size_t)nl * pny(G, q) * sy, ncclDouble, q,
                                 G->comm, G->stream));
            NCCL_TRY(G, ncclRecv(G->pen_in + (long)G->z0s[q] * G->pgeo.sz, (size_t)G->nls[q] * G->pgeo.sz, ncclDouble,
                                 q, G->comm, G->stream));
        }
        NCCL_TRY(G, ncclGroupEnd());
    }
    int rc;
    for (ads_ctx *m : slabs_of(G))
        if ((rc = run_sweep_tab(m, 2, m->tabG, m->pen_in, m->pen_out, nullptr, 0.0, nullptr, &m->pgeo))) return rc;
    if (G->dist == 2) {
        for (ads_ctx *s_ : G->members)
            for (int q = 0; q < W; ++q) {
                ads_ctx *t = G->members[q];
                CUDA_TRY(G, cudaMemcpyAsync(s_->arecv + (long)s_->n[2] * s_->py0[q] * s_->geo.sy,
                                            t->pen_out + (long)s_->zbeg * t->pgeo.sz,
                                            sizeof(double) * s_->n[2] * t->pgeo.sz, cudaMemcpyDeviceToDevice, G->stream));
            }
    } else {
        const int me = G->rank, nl = G->n[2];
        const long sy = G->geo.sy;
        CUDA_TRY(G, cudaMemcpyAsync(G->arecv + (long)nl * G->py0[me] * sy, G->pen_out + (long)G->zbeg * G->pgeo.sz,
                                    sizeof(double) * nl * G->pgeo.sz, cudaMemcpyDeviceToDevice, G->stream));
        NCCL_TRY(G, ncclGroupStart());
        for (int q = 0; q < W; ++q) {
            if (q == me) continue;
            NCCL_TRY(G, ncclSend(G->pen_out + (long)G->z0s[q] * G->pgeo.sz, (size_t)G->nls[q] * G->pgeo.sz, ncclDouble,
                                 q, G->comm, G->stream));
            NCCL_TRY(G, ncclRecv(G->arecv + (long)nl * G->py0[q] * sy, (size_t)nl * pny(G, q) * sy, ncclDouble, q,
                                 G->comm, G->stream));
        }
        NCCL_TRY(G, ncclGroupEnd());
    }
    for (ads_ctx *m : slabs_of(G)) {
        KickA2AArgs k;
        k.arecv = m->arecv;
        k.V = m->V;
        k.A = keepA ? m->A : nullptr;
        k.kick = kick;
        k.geo = m->geo;
        k.nq = W;
        for (int q = 0; q <= W; ++q) k.py0[q] = m->py0[q];
        ProfScope ps(m, 3);
        if (launch_kick_a2a(k, m->stream)) return fail(m, ADS_E_INVAL, "kick_a2a: too many slabs");
        if ((rc = check_launch(m, "kick_a2a"))) return rc;
    }
    return ADS_OK;
}

// One drift + solve + kick over all slabs: A = D^-1 (F(t) - K (U + tau_d V)), V += kick A,
// U <- U + tau_d V when tau_d != 0 (the step) -- with tau_d = 0 this is the half-kick init.
int dist_solve(ads_ctx *G, double tau_d, double g, double kick, bool keepA) {
    int rc;
    // only the drifted field crosses the interfaces: each slab forms P = U + tau V on its p first
    // and last owned planes (into U2, where the operator kernel writes P anyway), the P planes are
    // exchanged into U2's halos, and the operator kernel reads its halo planes from there -- half
    // the bytes of exchanging U and V (the half-kick start, tau_d = 0, exchanges U alone)
    if (tau_d != 0.0) {
        for (ads_ctx *m : slabs_of(G)) {
            const long hp = (long)m->p * m->geo.sz, nl = m->n[2];
            launch_drift(m->U, m->V, tau_d, m->U2, hp, m->stream);
            launch_drift(m->U + (nl - m->p) * m->geo.sz, m->V + (nl - m->p) * m->geo.sz, tau_d,
                         m->U2 + (nl - m->p) * m->geo.sz, hp, m->stream);
            if ((rc = check_launch(m, "drift edges"))) return rc;
        }
        if ((rc = exch_halo(G, &ads_ctx::U2))) return rc;
    } else if ((rc = exch_halo(G, &ads_ctx::U))) {
        return rc;
    }
    for (ads_ctx *m : slabs_of(G)) {
        if ((rc = run_kop(m, m->U, m->V, tau_d, g, -1.0, tau_d != 0.0 ? m->U2 : nullptr, m->R, false, nullptr,
                          tau_d != 0.0 ? m->U2 : nullptr)))
            return rc;
        if ((rc = run_sweep(m, 0, m->R, m->Wk, nullptr, 0.0)) || (rc = run_sweep(m, 1, m->Wk, m->R, nullptr, 0.0)) ||
            (!G->zsolve && (rc = run_sweep_tab(m, 2, m->tabZ, m->R, m->Wk, nullptr, 0.0))))
            return rc;
    }
    if (G->zsolve) {
        if ((rc = a2a_zsolve(G, kick, keepA))) return rc;
        if (tau_d != 0.0)
            for (ads_ctx *m : slabs_of(G)) std::swap(m->U, m->U2);
        return ADS_OK;
    }
    if ((rc = exch_tips(G))) return rc;
    if (G->world > 2) {  // interface refinement needs the neighbours' stage-1 values
        for (ads_ctx *m : slabs_of(G))
            if ((rc = run_zint(m))) return rc;
        if ((rc = exch_stage1(G))) return rc;
    }
    for (ads_ctx *m : slabs_of(G)) {
        if ((rc = run_zfix(m, keepA ? m->A : nullptr, kick))) return rc;
        if (tau_d != 0.0) std::swap(m->U, m->U2);
    }
    return ADS_OK;
}

// partial energy dots of one slab (or the single-GPU field) into m->dres[0..3]:
//   v'Mv (v = V - tau/2 a), U'KU, V'DV, U'K(U + tau V); x/y passes run over the halo planes
//   so that the z pass sees its neighbours (needs the U, V, R halos exchanged)
int energy_partials(ads_ctx *m) {
    const Geom &g = m->geo;
    const long hl = (long)m->halo * g.sz, N = m->Nalloc;
    Geom ge = g;
    ge.n2 = g.n2 + 2 * m->halo;
    const int zv0 = -m->halo, zv1 = g.n2 + m->halo;
    int rc;
    // kinetic (R = v already formed on owned planes, halos exchanged)
    if (launch_axis_apply(m->p, 0, m->dd[0].mband, m->R - hl, m->Wk - hl, ge, 1.0, 0.0, m->stream) ||
        launch_axis_apply(m->p, 1, m->dd[1].mband, m->Wk - hl, m->U2 - hl, ge, 1.0, 0.0, m->stream) ||
        launch_axis_apply(m->p, 2, m->dd[2].mband, m->U2, m->Wk, g, 1.0, 0.0, m->stream, m->zbeg, zv0, zv1))
        return fail(m, ADS_E_INVAL, "axis apply: unsupported p");
    if ((rc = check_launch(m, "axis_apply"))) return rc;
    launch_dot(N, m->R, m->Wk, m->dpartial, m->dres + 0, m->stream);
    // potential
    if ((rc = run_kop(m, m->U, m->V, 0.0, 0.0, 1.0, nullptr, m->R))) return rc;
    launch_dot(N, m->U, m->R, m->dpartial, m->dres + 1, m->stream);
    // invariant
    if (launch_axis_apply(m->p, 0, m->dd[0].aband, m->V - hl, m->Wk - hl, ge, 1.0, 0.0, m->stream) ||
        launch_axis_apply(m->p, 1, m->dd[1].aband, m->Wk - hl, m->U2 - hl, ge, 1.0, 0.0, m->stream) ||
        launch_axis_apply(m->p, 2, m->dd[2].aband, m->U2, m->Wk, g, 1.0, 0.0, m->stream, m->zbeg, zv0, zv1))
        return fail(m, ADS_E_INVAL, "axis apply: unsupported p");
    launch_dot(N, m->V, m->Wk, m->dpartial, m->dres + 2, m->stream);
    if ((rc = run_kop(m, m->U, m->V, m->tau, 0.0, 1.0, nullptr, m->R))) return rc;
    launch_dot(N, m->U, m->R, m->dpartial, m->dres + 3, m->stream);
    return check_launch(m, "dot");
}

int pwave_energy(ads_ctx *G, double res[3]) {
    int rc;
    if ((rc = exch_halo(G, &ads_ctx::U)) || (rc = exch_halo(G, &ads_ctx::V))) return rc;
    for (ads_ctx *m : slabs_of(G)) {
        CUDA_TRY(m, cudaMemcpyAsync(m->R, m->V, sizeof(double) * m->Nalloc, cudaMemcpyDeviceToDevice, m->stream));
        launch_axpby(m->Nalloc, -vel_corr(m), m->A, 1.0, m->R, m->stream);
        if ((rc = check_launch(m, "axpby"))) return rc;
    }
    if ((rc = exch_halo(G, &ads_ctx::R))) return rc;
    double d4[4] = {0, 0, 0, 0};
    for (ads_ctx *m : slabs_of(G)) {
        if ((rc = energy_partials(m))) return rc;
        if (m->dist == 1) NCCL_TRY(m, ncclAllReduce(m->dres, m->dres, 4, ncclDouble, ncclSum, m->comm, m->stream));
        double e[4];
        CUDA_TRY(m, cudaMemcpyAsync(e, m->dres, sizeof(double) * 4, cudaMemcpyDeviceToHost, m->stream));
        CUDA_TRY(m, cudaStreamSynchronize(m->stream));
        for (int i = 0; i < 4; ++i) d4[i] += e[i];
    }
    res[0] = 0.5 * d4[0];
    res[1] = 0.5 * d4[1];
    // R0 conserves no such quantity: the third slot reports kinetic + potential instead
    res[2] = G->scheme == 1 ? 0.5 * d4[2] + 0.5 * d4[3] : res[0] + res[1];
    return ADS_OK;
}

// Host arrays move as one contiguous copy through a dense device staging buffer and are
// repacked on the device (pitched host<->device 2D copies ran at ~28 GB/s against ~56 GB/s
// contiguous on this box, scripts/copy_probe.py); device arrays use a 2D device copy.
int stage_buffer(ads_ctx *h) {
    return h->stage ? ADS_OK : dalloc(h, (void **)&h->stage, sizeof(double) * (size_t)h->N);
}

int copy_in(ads_ctx *h, double *dst, const double *src, int mem) {
    if (mem == ADS_MEM_DEVICE) {  // dense caller array -> pitched device field
        CUDA_TRY(h, cudaMemcpy2DAsync(dst, sizeof(double) * h->geo.sy, src, sizeof(double) * h->n[0],
                                      sizeof(double) * h->n[0], (size_t)h->n[1] * h->n[2], cudaMemcpyDeviceToDevice,
                                      h->stream));
        return ADS_OK;
    }
    int rc;
    if ((rc = stage_buffer(h))) return rc;
    CUDA_TRY(h, cudaMemcpyAsync(h->stage, src, sizeof(double) * (size_t)h->N, cudaMemcpyHostToDevice, h->stream));
    launch_repack(h->stage, dst, h->geo, 1, h->stream);
    return check_launch(h, "repack");
}

int copy_out(ads_ctx *h, double *dst, const double *src, int mem) {
    if (mem == ADS_MEM_DEVICE) {
        CUDA_TRY(h, cudaMemcpy2DAsync(dst, sizeof(double) * h->n[0], src, sizeof(double) * h->geo.sy,
                                      sizeof(double) * h->n[0], (size_t)h->n[1] * h->n[2], cudaMemcpyDeviceToDevice,
                                      h->stream));
        return ADS_OK;
    }
    int rc;
    if ((rc = stage_buffer(h))) return rc;
    launch_repack(src, h->stage, h->geo, 0, h->stream);
    if ((rc = check_launch(h, "repack"))) return rc;
    CUDA_TRY(h, cudaMemcpyAsync(dst, h->stage, sizeof(double) * (size_t)h->N, cudaMemcpyDeviceToHost, h->stream));
    return ADS_OK;
}

// ---------------------------------------------------------------------------------------
// exact-in-time modal propagator (§3 decomposition):
// c = (Q_x (x) Q_y (x) Q_z) U with Q_d = Phi_d^T M_d, per-mode R1 recurrence, U = P3 c.
// The three directional transforms are dense products on the FP64 tensor cores, hand-written
// (modal_tc.cu) with the mirror fold of the even / odd bases fused into them.
// ---------------------------------------------------------------------------------------

int modal_prepare(ads_ctx *h) {
    if (h->modal_ready) return ADS_OK;
    int rc;
    for (int d = 0; d < 3; ++d) {
        const int o = h->sp[d].bc == ADS_BC_DIRICHLET0 ? 1 : 0;
        const int n = h->n[d], na = n - 2 * o, hh = n / 2, H = hh + (n & 1);
        int e = -1;  // an earlier direction with the same 1D space
        for (int c = 0; c < d; ++c)
            if (h->nel[c] == h->nel[d] && h->sp[c].bc == h->sp[d].bc) e = c;
        if (e >= 0) {
            h->mQe[d] = h->mQe[e], h->mQo[d] = h->mQo[e], h->mPe[d] = h->mPe[e], h->mPo[d] = h->mPo[e];
            h->mQe2[d] = h->mQe2[e], h->mQo2[d] = h->mQo2[e], h->mPe2[d] = h->mPe2[e], h->mPo2[d] = h->mPo2[e];
            h->mlqe[d] = h->mlqe[e], h->mlqo[d] = h->mlqo[e], h->mlpe[d] = h->mlpe[e], h->mlpo[d] = h->mlpo[e];
            h->mne[d] = h->mne[e], h->mno[d] = h->mno[e], h->mlam[d] = h->mlam[e];
            h->mphi_h[d] = h->mphi_h[e], h->mord[d] = h->mord[e];
            continue;
        }
        std::vector<double> lam, phi;
        std::vector<int> par;  // exact parity of each mode (even / odd blocks solved apart)
        if (modal_basis(h->sp[d], lam, phi, &par))
            return fail(h, ADS_E_SINGULAR, "modal basis of direction %d: eigensolver failed", d);
        std::vector<int> E, O;
        for (int k = 0; k < na; ++k) (par[k] > 0 ? E : O).push_back(k);
        const int ne = (int)E.size(), no = (int)O.size();
        // Q(k, i) = sum_j phi(j, k) M(j + o, i) at extended position i; Phi(i, k) likewise
        auto Qf = [&](int k, int i) {
            const int ia = i - o;
            if (ia < 0 || ia >= na) return 0.0;
            double q = 0.0;
            for (int j = std::max(0, ia - h->p); j <= std::min(na - 1, ia + h->p); ++j)
                q += phi[(size_t)j * na + k] * h->sp[d].M.get(j + o, i);
            return q;
        };
        auto Pf = [&](int i, int k) { return (i - o >= 0 && i - o < na) ? phi[(size_t)(i - o) * na + k] : 0.0; };
        std::vector<double> Qe((size_t)std::max(1, ne * H)), Qo((size_t)std::max(1, no * hh)),
            Pe((size_t)std::max(1, H * ne)), Po((size_t)std::max(1, hh * no)), le(n, 0.0);
        for (int a = 0; a < ne; ++a) {
            for (int i = 0; i < H; ++i) Qe[(size_t)a + (size_t)i * ne] = Qf(E[a], i);
            for (int i = 0; i < H; ++i) Pe[(size_t)i + (size_t)a * H] = Pf(i, E[a]);
            le[a] = lam[E[a]];
        }
        for (int b = 0; b < no; ++b) {
            for (int i = 0; i < hh; ++i) Qo[(size_t)b + (size_t)i * no] = Qf(O[b], i);
            for (int i = 0; i < hh; ++i) Po[(size_t)i + (size_t)b * hh] = Pf(i, O[b]);
            le[ne + b] = lam[O[b]];
        }
        // padded copies (column-major, leading dimension a multiple of 4)
        auto padded = [](const std::vector<double> &a, int rows, int cols, int &ld, int halve_col) {
            ld = std::max(4, (rows + 3) / 4 * 4);
            std::vector<double> b((size_t)ld * std::max(cols, 1), 0.0);
            for (int c = 0; c < cols; ++c)
                for (int r = 0; r < rows; ++r) b[(size_t)r + (size_t)c * ld] = a[(size_t)r + (size_t)c * rows] * (c == halve_col ? 0.5 : 1.0);
            return b;
        };
        std::vector<double> Qe2 = padded(Qe, ne, H, h->mlqe[d], (n & 1) ? H - 1 : -1);
        std::vector<double> Qo2 = padded(Qo, no, hh, h->mlqo[d], -1);
        std::vector<double> Pe2 = padded(Pe, H, ne, h->mlpe[d], -1);
        std::vector<double> Po2 = padded(Po, hh, no, h->mlpo[d], -1);
        double **dsts[9] = {&h->mQe[d], &h->mQo[d], &h->mPe[d], &h->mPo[d], &h->mlam[d],
                            &h->mQe2[d], &h->mQo2[d], &h->mPe2[d], &h->mPo2[d]};
        const std::vector<double> *srcs[9] = {&Qe, &Qo, &Pe, &Po, &le, &Qe2, &Qo2, &Pe2, &Po2};
        for (int q = 0; q < 9; ++q) {
            if ((rc = dalloc(h, (void **)dsts[q], sizeof(double) * srcs[q]->size()))) return rc;
            CUDA_TRY(h, cudaMemcpy(*dsts[q], srcs[q]->data(), sizeof(double) * srcs[q]->size(), cudaMemcpyHostToDevice));
        }
        h->mne[d] = ne;
        h->mno[d] = no;
        h->mphi_h[d] = phi;
        h->mord[d] = E;
        h->mord[d].insert(h->mord[d].end(), O.begin(), O.end());
    }
    h->modal_ready = true;
    return ADS_OK;
}

// forward (modal coordinates) or inverse map of a whole field along x, y, z: in -> b, scratch a
// (in is only read).  Each direction is one launch of the folded tensor-core GEMMs (modal_tc.cu):
// the mirror fold / unfold happens in the operand loads / the epilogue.
int modal_transform(ads_ctx *h, bool inverse, const double *in, double *a, double *b) {
    const Geom &g = h->geo;
    const double *src = in;
    double *dsts[3] = {b, a, b};  // in -> b -> a -> b
    for (int d = 0; d < 3; ++d) {
        ModalGemmArgs m;
        m.in = src;
        m.out = dsts[d];
        m.n = h->n[d];
        m.hh = m.n / 2;
        m.H = m.hh + (m.n & 1);
        m.ne = h->mne[d];
        m.no = h->mno[d];
        m.Qe = h->mQe[d], m.Qo = h->mQo[d], m.Pe = h->mPe[d], m.Po = h->mPo[d];
        m.Qe2 = h->mQe2[d], m.Qo2 = h->mQo2[d], m.Pe2 = h->mPe2[d], m.Po2 = h->mPo2[d];
        m.lqe = h->mlqe[d], m.lqo = h->mlqo[d], m.lpe = h->mlpe[d], m.lpo = h->mlpo[d];
        m.inverse = inverse ? 1 : 0;
        if (d == 0) {         // x lines: contiguous rows of pitch sy
            m.ks = 1, m.ls = g.sy, m.nl = g.n1 * g.n2, m.bs = 0, m.nb = 1;
            m.kdim = 0, m.td[0] = g.n0, m.td[1] = (long)g.n1 * g.n2, m.td[2] = 1, m.ts1 = g.sy, m.ts2 = g.sz * g.n2;
        } else if (d == 1) {  // y lines: adjacent in x, one batch per plane
            m.ks = g.sy, m.ls = 1, m.nl = g.n0, m.bs = g.sz, m.nb = g.n2;
            m.kdim = 1, m.td[0] = g.n0, m.td[1] = g.n1, m.td[2] = g.n2, m.ts1 = g.sy, m.ts2 = g.sz;
        } else {              // z lines: every (x, y) position of a plane, row padding included (zero)
            m.ks = g.sz, m.ls = 1, m.nl = (int)g.sz, m.bs = 0, m.nb = 1;
            m.kdim = 1, m.td[0] = g.sz, m.td[1] = g.n2, m.td[2] = 1, m.ts1 = g.sz, m.ts2 = g.sz * g.n2;
        }
        ProfScope ps(h, 4);
        const int lr = launch_modal_gemm(m, h->stream);
        if (lr == -2) return fail(h, ADS_E_CUDA, "modal transform: TMA descriptor encoding failed");
        if (lr) return fail(h, ADS_E_INVAL, "modal transform: grid too large");
        int rc;
        if ((rc = check_launch(h, "modal transform"))) return rc;
        src = dsts[d];
    }
    return ADS_OK;
}

}  // namespace

extern "C" {

// dist: 0 single GPU; 1 NCCL slab `rank` of `world`; 3 member slab of a virtual group
static int create_common(ads_handle *out, int nx, int ny, int nz, int p, double tau, int bc, int ncomp,
                         double lam, double mu, double rho, int dist = 0, int rank = 0, int world = 1,
                         ncclComm_t comm = nullptr) {
    if (!out) return ADS_E_INVAL;
    *out = nullptr;
    // nz = 0: the 2D scheme (single-GPU handles; trivial_space): P-wave, or plane-strain elasticity
    // (u_z decouples: B_z = 0)
    if (p < 1 || p > 5 || nx < 1 || ny < 1 || nz < 0 || (nz == 0 && dist) || !(tau > 0.0) ||
        !std::isfinite(tau) || (bc != ADS_BC_NATURAL && bc != ADS_BC_DIRICHLET0))
        return ADS_E_INVAL;
    if (bc == ADS_BC_DIRICHLET0 && (nx + p < 3 || ny + p < 3 || (nz > 0 && nz + p < 3))) return ADS_E_INVAL;
    if (nx + p > 1056 || ny + p > 1056) return ADS_E_INVAL;  // n_d <= 32 x 33 (sweep chunking)
    if (world < 1 || rank < 0 || rank >= world) return ADS_E_INVAL;
    ads_ctx *h = new (std::nothrow) ads_ctx;
    if (!h) return ADS_E_NOMEM;
    h->p = p;
    h->bc = bc;
    h->tau = tau;
    h->ncomp = ncomp;
    h->lam = lam;
    h->mu = mu;
    h->rho = rho;
    h->nel[0] = nx;
    h->nel[1] = ny;
    h->nel[2] = nz;
    h->dist = dist;
    h->rank = rank;
    h->world = world;
    h->comm = comm;
    h->ngz = nz == 0 ? 1 : nz + p;
    int rc = ADS_OK;
    if (dist) {
        std::vector<int> z0s, nls;
        slab_plan(h->ngz, world, z0s, nls);
        h->zbeg = z0s[rank];
        h->halo = p;
        h->has_prev = rank > 0;
        h->has_next = rank < world - 1;
        if (ncomp != 1) rc = fail(h, ADS_E_INVAL, "z-slabs: P-wave handles only");
    } else if (nz + p > 1056) {
        rc = ADS_E_INVAL;
    }
    cudaGetDevice(&h->device);
    for (int d = 0; d < 3 && rc == ADS_OK; ++d) {
        h->n[d] = h->nel[d] == 0 ? 1 : h->nel[d] + p;
        rc = build_direction(h, d);
    }
    if (rc == ADS_OK && dist) {
        std::vector<int> z0s, nls;
        slab_plan(h->ngz, world, z0s, nls);
        h->n[2] = nls[rank];  // owned planes
    }
    if (rc == ADS_OK) {
        h->geo.n0 = h->n[0];
        h->geo.n1 = h->n[1];
        h->geo.n2 = h->n[2];
        // rows padded to a multiple of 8 doubles: every 8-line tile row segment of the
        // y/z sweeps is one aligned 64-byte block, x-sweep tiles start 64-byte aligned
        h->geo.sy = (h->n[0] + 7) / 8 * 8;
        h->geo.sz = h->geo.sy * h->n[1];
        h->N = (long)h->n[0] * h->n[1] * h->n[2];
        h->Nalloc = h->geo.sz * h->n[2];
        // every field carries `halo` planes below and above its owned planes
        const long hl = (long)h->halo * h->geo.sz;
        const size_t fb = sizeof(double) * (h->Nalloc + 2 * hl) * ncomp, sb = sizeof(double) * (h->Nalloc + 2 * hl);
        std::vector<std::pair<double **, size_t>> fields = {{&h->U, fb}, {&h->U2, fb}, {&h->V, fb},
                                                            {&h->A, fb}, {&h->R, sb},  {&h->Wk, sb}};
        if (ncomp == 3)
            for (auto f : std::initializer_list<std::pair<double **, size_t>>{
                     {&h->W, fb}, {&h->T1, sb}, {&h->T2, sb}, {&h->T3, sb}})
                fields.push_back(f);
        if (dist)
            for (double **b : {&h->tip_prev, &h->tip_next, &h->b0buf, &h->u0buf, &h->b0_prev2, &h->u0_next2})
                fields.push_back({b, sizeof(double) * p * h->geo.sz});
        for (auto &f : fields)
            if (rc == ADS_OK) rc = dalloc(h, (void **)f.first, f.second);
        if (rc == ADS_OK && (rc = dalloc(h, (void **)&h->dpartial, sizeof(double) * 1024)) == ADS_OK &&
            (rc = dalloc(h, (void **)&h->dres, sizeof(double) * 8)) == ADS_OK &&
            (rc = dalloc(h, (void **)&h->dstep, sizeof(long))) == ADS_OK) {
            cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamDefault);
            if (e != cudaSuccess) rc = fail(h, ADS_E_CUDA, "stream: %s", cudaGetErrorString(e));
            h->own_stream = true;
            if (ncomp == 3 && rc == ADS_OK) {
                for (cudaStream_t &st : h->side)
                    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) rc = ADS_E_CUDA;
                for (cudaEvent_t &ev : h->fev)
                    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) rc = ADS_E_CUDA;
                if (rc) rc = fail(h, ADS_E_CUDA, "elastic side streams");
            }
        }
        if (rc == ADS_OK) {  // zero everything: row padding and domain-boundary halos stay 0 forever
            for (auto &f : fields) cudaMemsetAsync(*f.first, 0, f.second, h->stream);
            cudaMemsetAsync(h->dstep, 0, sizeof(long), h->stream);
            if (cudaStreamSynchronize(h->stream) != cudaSuccess) rc = fail(h, ADS_E_CUDA, "memset failed");
            for (int f = 0; f < 6 + (ncomp == 3 ? 4 : 0); ++f) *fields[f].first += hl;  // owned planes
        }
    }
    if (rc != ADS_OK) {
        h->comm = nullptr;  // owned by the caller of create_common
        ads_destroy(h);
        return rc;
    }
    *out = h;
    return ADS_OK;
}

int ads_create(ads_handle *out, int nx, int ny, int nz, int p, double tau, int bc) {
    return create_common(out, nx, ny, nz, p, tau, bc, 1, 0.0, 0.0, 1.0);
}

int ads_create_elastic(ads_handle *out, int nx, int ny, int nz, int p, double tau, int bc, double lambda, double mu,
                       double rho) {
    if (out) *out = nullptr;
    if (!(lambda >= 0.0) || !(mu > 0.0) || !(rho > 0.0) || !std::isfinite(lambda) || !std::isfinite(mu) ||
        !std::isfinite(rho))
        return ADS_E_INVAL;
    return create_common(out, nx, ny, nz, p, tau, bc, 3, lambda, mu, rho);
}

int ads_get_unique_id(unsigned char uid[128]) {
    if (!uid) return ADS_E_INVAL;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return ADS_E_NCCL;
    std::memcpy(uid, &id, sizeof id);
    return ADS_OK;
}

int ads_slab_plan(int nz, int p, int world, int rank, int *z_begin, int *z_count) {
    if (nz < 1 || p < 1 || world < 1 || rank < 0 || rank >= world || !z_begin || !z_count) return ADS_E_INVAL;
    std::vector<int> z0s, nls;
    slab_plan(nz + p, world, z0s, nls);
    *z_begin = z0s[rank];
    *z_count = nls[rank];
    return ADS_OK;
}

int ads_create_dist(ads_handle *out, int nx, int ny, int nz, int p, double tau, int bc, int rank, int world,
                    const unsigned char uid[128], int device) {
    if (!out || !uid || world < 1 || rank < 0 || rank >= world) return ADS_E_INVAL;
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return ADS_E_CUDA;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    ncclComm_t comm = nullptr;
    if (ncclCommInitRank(&comm, world, id, rank) != ncclSuccess) return ADS_E_NCCL;
    int rc = create_common(out, nx, ny, nz, p, tau, bc, 1, 0.0, 0.0, 1.0, 1, rank, world, comm);
    if (rc != ADS_OK) ncclCommDestroy(comm);
    return rc;
}

int ads_create_virtual(ads_handle *out, int nx, int ny, int nz, int p, double tau, int bc, int nslabs) {
    if (!out || nslabs < 1) return ADS_E_INVAL;
    *out = nullptr;
    ads_ctx *G = new (std::nothrow) ads_ctx;
    if (!G) return ADS_E_NOMEM;
    G->dist = 2;
    G->world = nslabs;
    G->p = p;
    G->bc = bc;
    G->tau = tau;
    G->nel[0] = nx;
    G->nel[1] = ny;
    G->nel[2] = nz;
    for (int d = 0; d < 3; ++d) G->n[d] = G->nel[d] + p;
    G->ngz = G->n[2];
    G->N = (long)G->n[0] * G->n[1] * G->n[2];
    cudaGetDevice(&G->device);
    int rc = ADS_OK;
    if (cudaStreamCreateWithFlags(&G->stream, cudaStreamDefault) != cudaSuccess) rc = ADS_E_CUDA;
    G->own_stream = true;
    for (int r = 0; r < nslabs && rc == ADS_OK; ++r) {
        ads_handle m = nullptr;
        rc = create_common(&m, nx, ny, nz, p, tau, bc, 1, 0.0, 0.0, 1.0, 3, r, nslabs, nullptr);
        if (rc == ADS_OK) {
            G->members.push_back(m);
            rc = ads_set_stream(m, G->stream);  // one stream orders every slab's work
        } else if (m) {
            G->err = m->err;
        }
    }
    for (int r = 0; r < (int)G->members.size(); ++r) {
        G->members[r]->prev = r > 0 ? G->members[r - 1] : nullptr;
        G->members[r]->next = r + 1 < (int)G->members.size() ? G->members[r + 1] : nullptr;
    }
    if (rc != ADS_OK) {
        ads_destroy(G);
        return rc;
    }
    *out = G;
    return ADS_OK;
}

int ads_set_tau(ads_handle h, double tau) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (!(tau > 0.0) || !std::isfinite(tau)) return fail(h, ADS_E_INVAL, "ads_set_tau: tau must be > 0");
    if (h->ncomp != 1 || h->dist) return fail(h, ADS_E_INVAL, "ads_set_tau: single-GPU P-wave handles only");
    if (h->have_state && h->scheme == 1) {  // udot_n = V - tau_old/2 a_n, kept in Wk
        CUDA_TRY(h, cudaMemcpyAsync(h->Wk, h->V, sizeof(double) * h->Nalloc, cudaMemcpyDeviceToDevice, h->stream));
        launch_axpby(h->Nalloc, -vel_corr(h), h->A, 1.0, h->Wk, h->stream);
        if ((rc = check_launch(h, "axpby"))) return rc;
    }
    const double t_now = time_at(h, h->step);
    drop_graphs(h);  // the graphs bake the factor tables
    h->tau = tau;
    h->t_base = t_now;
    h->n_base = h->step;
    for (int d = 0; d < 3; ++d) {  // A_d = M_d + tau^2/4 K_d
        Band A = shifted(h->sp[d], tau * tau / 4.0, h->sp[d].bc);
        char what[32];
        snprintf(what, sizeof what, "A_%d", d);
        if ((rc = make_solve_tab(h, A, what, h->dd[d].tab))) return rc;
        if (h->dd[d].aband) dfree(h, h->dd[d].aband);
        if ((rc = upload(h, &h->dd[d].aband, A.v))) return rc;
    }
    if (h->have_state && h->scheme == 1) {
        // restart at t_n from (U_n, udot_n): a_n = D^-1 (F(t_n) - K U_n), V = udot_n + tau/2 a_n
        CUDA_TRY(h, cudaMemcpyAsync(h->V, h->Wk, sizeof(double) * h->Nalloc, cudaMemcpyDeviceToDevice, h->stream));
        if ((rc = run_kop(h, h->U, h->U, 0.0, source_g(h, t_now), -1.0, nullptr, h->R))) return rc;
        if ((rc = run_sweep(h, 0, h->R, h->Wk, nullptr, 0.0))) return rc;
        if ((rc = run_sweep(h, 1, h->Wk, h->R, nullptr, 0.0))) return rc;
        if ((rc = run_sweep(h, 2, h->R, h->A, h->V, 0.5 * tau))) return rc;
    }
    return ADS_OK;
}

int ads_set_scheme(ads_handle h, int scheme) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (scheme != 0 && scheme != 1) return fail(h, ADS_E_INVAL, "ads_set_scheme: scheme must be 0 or 1");
    if (scheme == 0 && (h->ncomp != 1 || h->dist))
        return fail(h, ADS_E_INVAL, "ads_set_scheme: the literal scheme is for single-GPU P-wave handles");
    drop_graphs(h);  // the graphs bake the kick coefficient
    h->scheme = scheme;
    h->have_state = false;  // V means something else under the other scheme: set the state again
    return ADS_OK;
}

int ads_modal_basis(int nel, int p, int bc, double *lambda, double *phi) {
    if (nel < 1 || p < 1 || p > kMaxP || (bc != ADS_BC_NATURAL && bc != ADS_BC_DIRICHLET0) || !lambda || !phi)
        return ADS_E_INVAL;
    Space1D sp;
    if (build_space(p, nel, bc, sp)) return ADS_E_INVAL;
    std::vector<double> lam, ph;
    if (modal_basis(sp, lam, ph)) return ADS_E_SINGULAR;
    std::memcpy(lambda, lam.data(), sizeof(double) * lam.size());
    std::memcpy(phi, ph.data(), sizeof(double) * ph.size());
    return ADS_OK;
}

int ads_modal_advance(ads_handle h, long nsteps) {
    NvtxRange nv_("ads_modal_advance");
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (nsteps < 0) return fail(h, ADS_E_INVAL, "ads_modal_advance: nsteps < 0");
    if (h->ncomp != 1 || h->dist) return fail(h, ADS_E_INVAL, "ads_modal_advance: single-GPU P-wave handles only");
    if (h->scheme != 1) return fail(h, ADS_E_INVAL, "ads_modal_advance: scheme R1 only");
    if (!h->have_state) return fail(h, ADS_E_STATE, "ads_modal_advance before ads_set_state");
    if (nsteps == 0) return ADS_OK;
    if ((rc = modal_prepare(h))) return rc;
    const double *fvec[3] = {nullptr, nullptr, nullptr};
    const double *gdev = nullptr;
    if (h->has_src) {  // modal load vectors Phi_d^T b_d (dual: no M) and g(t_{n+s}), s = 1..nsteps
        for (int d = 0; d < 3; ++d) {
            const int o = h->sp[d].bc == ADS_BC_DIRICHLET0 ? 1 : 0;
            const int n = h->n[d], na = n - 2 * o;
            std::vector<double> f(n, 0.0);  // in modal slot order (even | odd)
            for (int slot = 0; slot < na; ++slot) {
                const int k = h->mord[d][slot];
                double v = 0.0;
                for (int i = 0; i < na; ++i) v += h->mphi_h[d][(size_t)i * na + k] * h->src_h[d][i + o];
                f[slot] = v;
            }
            if (!h->mf[d] && (rc = dalloc(h, (void **)&h->mf[d], sizeof(double) * n))) return rc;
            CUDA_TRY(h, cudaMemcpyAsync(h->mf[d], f.data(), sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
            CUDA_TRY(h, cudaStreamSynchronize(h->stream));
            fvec[d] = h->mf[d];
        }
        if (nsteps > h->mg_cap) {
            if ((rc = dalloc(h, (void **)&h->mg, sizeof(double) * nsteps))) return rc;
            h->mg_cap = nsteps;
        }
        std::vector<double> gv(nsteps);
        for (long s = 0; s < nsteps; ++s) gv[s] = source_g(h, time_at(h, h->step + s + 1));
        CUDA_TRY(h, cudaMemcpy(h->mg, gv.data(), sizeof(double) * nsteps, cudaMemcpyHostToDevice));
        gdev = h->mg;
    }
    // U -> cU (in R), V -> cV (in U2); modes advance in place; back: cV -> V, cU -> U; then a
    if ((rc = modal_transform(h, false, h->U, h->Wk, h->R))) return rc;
    if ((rc = modal_transform(h, false, h->V, h->Wk, h->U2))) return rc;
    if (launch_modal(h->R, h->U2, h->Wk, h->mlam[0], h->mlam[1], h->mlam[2], fvec[0], fvec[1], fvec[2], gdev, nsteps,
                     h->tau, h->geo, h->stream))
        return fail(h, ADS_E_INVAL, "ads_modal_advance: grid too large for the mode kernel");
    if ((rc = check_launch(h, "modal"))) return rc;
    if ((rc = modal_transform(h, true, h->U2, h->A, h->V))) return rc;
    if ((rc = modal_transform(h, true, h->R, h->A, h->U))) return rc;
    h->step += nsteps;
    // a_n = D^-1 (F(t_n) - K U_n) (= P3 ca exactly; the operator kernel and three sweeps cost
    // less than a fifth transform and compute a as ads_step does)
    if ((rc = run_kop(h, h->U, h->U, 0.0, source_g(h, time_at(h, h->step)), -1.0, nullptr, h->R))) return rc;
    if ((rc = run_sweep(h, 0, h->R, h->Wk, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 1, h->Wk, h->R, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 2, h->R, h->A, nullptr, 0.0))) return rc;
    launch_set_long(h->dstep, h->step, h->stream);  // source time of later graph replays
    return check_launch(h, "set_step");
}

// the pencil buffers and the global A_z table of one slab (first switch to the all-to-all solve)
static int a2a_prepare(ads_ctx *m, int W) {
    if (m->pen_in) return ADS_OK;
    slab_plan(m->ngz, W, m->z0s, m->nls);
    m->py0.assign(W + 1, 0);
    for (int q = 0; q <= W; ++q) m->py0[q] = (int)((long)q * m->n[1] / W);
    for (int q = 0; q < W; ++q)
        if (m->py0[q + 1] <= m->py0[q]) return fail(m, ADS_E_INVAL, "all-to-all: %d slabs exceed n_y = %d", W, m->n[1]);
    m->pgeo = m->geo;
    m->pgeo.n1 = m->py0[m->rank + 1] - m->py0[m->rank];
    m->pgeo.n2 = m->ngz;
    m->pgeo.sz = m->geo.sy * m->pgeo.n1;
    int rc;
    const Band A = shifted(m->sp[2], m->tau * m->tau / 4.0, m->sp[2].bc);
    if ((rc = make_solve_tab(m, A, "A_z (all-to-all pencils)", m->tabG))) return rc;
    const size_t pb = sizeof(double) * m->pgeo.sz * m->pgeo.n2, fb = sizeof(double) * m->Nalloc;
    if ((rc = dalloc(m, (void **)&m->pen_in, pb)) || (rc = dalloc(m, (void **)&m->pen_out, pb)) ||
        (rc = dalloc(m, (void **)&m->arecv, fb)) || (m->dist == 1 && (rc = dalloc(m, (void **)&m->a2a_send, fb))))
        return rc;
    CUDA_TRY(m, cudaMemsetAsync(m->pen_in, 0, pb, m->stream));
    CUDA_TRY(m, cudaMemsetAsync(m->pen_out, 0, pb, m->stream));
    return ADS_OK;
}

int ads_set_zsolve(ads_handle h, int mode) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (!h->dist || h->dist == 3 || (mode != ADS_ZSOLVE_SPIKE && mode != ADS_ZSOLVE_ALLTOALL))
        return fail(h, ADS_E_INVAL, "set_zsolve: slab handles (ads_create_dist / ads_create_virtual), mode 0 or 1");
    const int W = slab_count(h);
    if (mode == ADS_ZSOLVE_ALLTOALL && W > kMaxA2A) return fail(h, ADS_E_INVAL, "all-to-all: at most %d slabs", kMaxA2A);
    if (mode == ADS_ZSOLVE_ALLTOALL)
        for (ads_ctx *m : slabs_of(h))
            if ((rc = a2a_prepare(m, W))) {
                if (m != h) h->err = m->err;
                return m != h ? fail(h, rc, "%s", m->err.c_str()) : rc;
            }
    h->zsolve = mode;
    for (ads_ctx *m : slabs_of(h)) m->zsolve = mode;
    drop_graphs(h);
    return ADS_OK;
}

int ads_local_extent(ads_handle h, int *z_begin, int *z_count) {
    DeviceScope ds_(h);
    if (!h || !z_begin || !z_count) return ADS_E_INVAL;
    *z_begin = h->dist == 2 ? 0 : h->zbeg;
    *z_count = h->dist == 2 ? h->ngz : h->n[2];
    return ADS_OK;
}

int ads_set_stream(ads_handle h, void *stream) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    cudaStream_t old = h->stream, next = old;
    bool own = h->own_stream;
    if (stream) {
        next = (cudaStream_t)stream;
        own = false;
    } else if (!h->own_stream) {
        CUDA_TRY(h, cudaStreamCreateWithFlags(&next, cudaStreamDefault));
        own = true;
    }
    // the members of a virtual slab group run on the group's stream: move them while the old
    // stream still exists, then release it
    for (ads_ctx *m : h->members)
        if ((rc = ads_set_stream(m, next))) return fail(h, rc, "member: %s", m->err.c_str());
    if (h->own_stream && old != next) cudaStreamDestroy(old);
    h->stream = next;
    h->own_stream = own;
    return ADS_OK;
}

int ads_load_vector(ads_handle h, int d, int func, double c, double sigma, double *out) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (d < 0 || d > 2 || !out || (func != ADS_FUNC_SIN && func != ADS_FUNC_GAUSS) ||
        (func == ADS_FUNC_GAUSS && !(sigma > 0.0)))
        return fail(h, ADS_E_INVAL, "ads_load_vector: bad argument");
    load_vector((h->dist == 2 ? h->members[0] : h)->sp[d], func, c, sigma, out);
    return ADS_OK;
}

int ads_mass_solve_1d(ads_handle h, int d, double *x) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (d < 0 || d > 2 || !x) return fail(h, ADS_E_INVAL, "ads_mass_solve_1d: bad argument");
    lu_solve_host((h->dist == 2 ? h->members[0] : h)->mass_lu[d], x);
    return ADS_OK;
}

int ads_set_source(ads_handle h, const double *bx, const double *by, const double *bz, int wavelet, double f0,
                   double t0, double amp) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (!bx) {
        drop_graphs(h);
        h->has_src = false;
        for (ads_ctx *m : h->members) m->has_src = false;
        return ADS_OK;
    }
    if (h->ncomp != 1) return fail(h, ADS_E_INVAL, "ads_set_source: P-wave handles only (elastic f = 0)");
    if (!by || !bz || (wavelet != ADS_WAVELET_NONE && wavelet != ADS_WAVELET_RICKER))
        return fail(h, ADS_E_INVAL, "ads_set_source: bad argument");
    drop_graphs(h);  // the graphs bake the source vectors and wavelet parameters
    for (ads_ctx *m : h->members)
        if ((rc = ads_set_source(m, bx, by, bz, wavelet, f0, t0, amp))) return fail(h, rc, "member: %s", m->err.c_str());
    const double *b[3] = {bx, by, bz};
    for (int d = 0; d < 3 && h->dist != 2; ++d) {
        const int nd = d == 2 ? h->ngz : h->n[d];  // z: global rows (slabs index with zbeg)
        std::vector<double> v(b[d], b[d] + nd);
        if (h->sp[d].bc == ADS_BC_DIRICHLET0) v[0] = v[nd - 1] = 0.0;
        if (!h->src[d]) {
            if ((rc = dalloc(h, (void **)&h->src[d], sizeof(double) * nd))) return rc;
        }
        CUDA_TRY(h, cudaMemcpy(h->src[d], v.data(), sizeof(double) * nd, cudaMemcpyHostToDevice));
        h->src_h[d] = v;
    }
    h->has_src = true;
    h->wavelet = wavelet;
    h->f0 = f0;
    h->t0 = t0;
    h->amp = amp;
    return ADS_OK;
}

int ads_set_state(ads_handle h, const double *u, const double *udot, int mem) {
    NvtxRange nv_("ads_set_state");
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (!u || (mem != ADS_MEM_HOST && mem != ADS_MEM_DEVICE)) return fail(h, ADS_E_INVAL, "ads_set_state: bad argument");
    for (ads_ctx *m : slabs_of(h)) {
        // group members read their planes out of the caller's global arrays
        const long off = h->dist == 2 ? (long)m->zbeg * m->n[0] * m->n[1] : 0;
        for (int c = 0; c < m->ncomp; ++c) {
            if ((rc = copy_in(m, comp(m->U, m, c), u + off + c * m->N, mem))) return rc;
            if (udot) {
                if ((rc = copy_in(m, comp(m->V, m, c), udot + off + c * m->N, mem))) return rc;
            } else {
                CUDA_TRY(m, cudaMemsetAsync(comp(m->V, m, c), 0, sizeof(double) * m->Nalloc, m->stream));
            }
            if (m->bc == ADS_BC_DIRICHLET0) {
                launch_mask_boundary(comp(m->U, m, c), m->geo, m->stream, m->zbeg, zmask(m));
                if ((rc = check_launch(m, "mask"))) return rc;
                launch_mask_boundary(comp(m->V, m, c), m->geo, m->stream, m->zbeg, zmask(m));
                if ((rc = check_launch(m, "mask"))) return rc;
            }
        }
    }
    return h->ncomp == 3 ? el_init(h) : init_state(h);
}

int ads_set_state_separable(ads_handle h, int nterms, const double *amp, const int *cmp, const double *sx,
                            const double *sy, const double *sz) {
    NvtxRange nv_("ads_set_state_separable");
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (nterms < 0 || (nterms > 0 && (!amp || !sx || !sy || !sz)))
        return fail(h, ADS_E_INVAL, "ads_set_state_separable: bad argument");
    for (int t = 0; t < nterms; ++t)
        if (cmp && (cmp[t] < 0 || cmp[t] >= h->ncomp))
            return fail(h, ADS_E_INVAL, "component %d on a handle with %d components", cmp[t], h->ncomp);
    for (ads_ctx *m : slabs_of(h)) {
        // one pass writes every term of every component (zero on the Dirichlet faces); udot0 = 0
        CUDA_TRY(m, cudaMemsetAsync(m->V, 0, sizeof(double) * m->Nalloc * m->ncomp, m->stream));
        const int n0 = m->n[0], n1 = m->n[1], n2 = m->ngz;
        const size_t tl = 2 + (size_t)n0 + n1 + n2;
        std::vector<double> packed((size_t)std::max(nterms, 1) * tl, 0.0);
        for (int t = 0; t < nterms; ++t) {
            double *f = &packed[(size_t)t * tl];
            f[0] = amp[t];
            f[1] = cmp ? cmp[t] : 0;
            std::memcpy(f + 2, sx + (size_t)t * n0, sizeof(double) * n0);
            std::memcpy(f + 2 + n0, sy + (size_t)t * n1, sizeof(double) * n1);
            std::memcpy(f + 2 + n0 + n1, sz + (size_t)t * n2, sizeof(double) * n2);
        }
        // the packed factors go to the work field Wk (free until the start procedure below writes
        // it; stream order), or to a scratch allocation when they do not fit.  A pageable-source
        // copy has consumed the host vector when cudaMemcpyAsync returns.
        const bool fits = packed.size() <= (size_t)m->Nalloc;
        double *d = fits ? m->Wk : nullptr;
        if (!fits && (rc = dalloc(m, (void **)&d, sizeof(double) * packed.size()))) return rc;
        CUDA_TRY(m, cudaMemcpyAsync(d, packed.data(), sizeof(double) * packed.size(), cudaMemcpyHostToDevice, m->stream));
        const bool dir = m->bc == ADS_BC_DIRICHLET0;
        launch_set_separable(m->U, m->Nalloc, m->ncomp, nterms, d, n0, n1, n2, m->geo, m->zbeg, dir ? 1 : 0,
                             dir ? 1 : 0, dir ? zmask(m) : 0, m->stream);
        if ((rc = check_launch(m, "separable"))) return rc;
        if (!fits) {
            CUDA_TRY(m, cudaStreamSynchronize(m->stream));
            dfree(m, d);
        }
    }
    return h->ncomp == 3 ? el_init(h) : init_state(h);
}

int ads_step(ads_handle h, int nsteps) {
    NvtxRange nv_("ads_step");
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (nsteps < 0) return fail(h, ADS_E_INVAL, "nsteps < 0");
    if (!h->have_state) return fail(h, ADS_E_STATE, "ads_step before ads_set_state");
    for (int s = 0; s < nsteps; ++s) {
        cudaGraphExec_t ex = nullptr;
        long nl = 0;
        if (h->ncomp == 3) {  // pairs of elastic steps replay a graph (a is written every step)
            if (!h->prof && !h->graphs_off && nsteps - s >= 2 && step_graph(h, &ex, &nl) == ADS_OK) {
                CUDA_TRY(h, cudaGraphLaunch(ex, h->stream));
                h->launches += nl;
                h->step += 2;
                ++s;
                continue;
            }
            if ((rc = el_step(h))) return rc;
            h->step += 1;
            continue;
        }
        const double t1 = time_at(h, h->step + 1);  // F at t_{n+1} (C14)
        if (h->dist) {
            if ((rc = dist_solve(h, h->tau, source_g(h, t1), h->tau, s == nsteps - 1))) return rc;
            h->step += 1;
            for (ads_ctx *m : h->members) m->step = h->step;
            continue;
        }
        // pairs of steps replay a captured CUDA graph (not while profiling kernels one by one);
        // the last step of the batch runs directly and keeps a
        if (!h->prof && !h->graphs_off && nsteps - s >= 3 && step_graph(h, &ex, &nl) == ADS_OK) {
            CUDA_TRY(h, cudaGraphLaunch(ex, h->stream));
            h->launches += nl;
            h->step += 2;
            ++s;
            continue;
        }
        // drift + RHS: U2 = U + tau V, R = F(t_{n+1}) - K U2; a = D^-1 R; V += tau a
        if ((rc = enqueue_step(h, s == nsteps - 1, false))) return rc;
        h->step += 1;
    }
    return ADS_OK;
}

int ads_energy(ads_handle h, double out[3]) {
    NvtxRange nv_("ads_energy");
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (!out) return fail(h, ADS_E_INVAL, "ads_energy: out is NULL");
    if (!h->have_state) return fail(h, ADS_E_STATE, "ads_energy before ads_set_state");
    double res[3];
    if (h->ncomp == 3) {
        if ((rc = el_energy(h, res))) return rc;
    } else if ((rc = pwave_energy(h, res))) {
        return rc;
    }
    for (int i = 0; i < 3; ++i) {
        if (!std::isfinite(res[i])) return fail(h, ADS_E_STATE, "non-finite energy (NaN/Inf in state)");
        out[i] = res[i];
    }
    return ADS_OK;
}

int ads_get_state(ads_handle h, double *u, double *udot, double *a, int mem) {
    NvtxRange nv_("ads_get_state");
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (mem != ADS_MEM_HOST && mem != ADS_MEM_DEVICE) return fail(h, ADS_E_INVAL, "bad mem");
    for (ads_ctx *m : slabs_of(h)) {
        const long off = h->dist == 2 ? (long)m->zbeg * m->n[0] * m->n[1] : 0;
        for (int c = 0; c < m->ncomp; ++c) {
            if (u && (rc = copy_out(m, u + off + c * m->N, comp(m->U, m, c), mem))) return rc;
            if (udot) {
                CUDA_TRY(m, cudaMemcpyAsync(m->Wk, comp(m->V, m, c), sizeof(double) * m->Nalloc,
                                            cudaMemcpyDeviceToDevice, m->stream));
                launch_axpby(m->Nalloc, -vel_corr(m), comp(m->A, m, c), 1.0, m->Wk, m->stream);
                if ((rc = check_launch(m, "axpby"))) return rc;
                if ((rc = copy_out(m, udot + off + c * m->N, m->Wk, mem))) return rc;
            }
            if (a && (rc = copy_out(m, a + off + c * m->N, comp(m->A, m, c), mem))) return rc;
        }
        CUDA_TRY(m, cudaStreamSynchronize(m->stream));
    }
    return ADS_OK;
}

double ads_time(ads_handle h) { return h ? time_at(h, h->step) : NAN; }
long ads_step_count(ads_handle h) { return h ? h->step : -1; }

int ads_dims(ads_handle h, int *nx, int *ny, int *nz, int *ncomp) {
    DeviceScope ds_(h);
    if (!h) return ADS_E_INVAL;
    if (nx) *nx = h->n[0];
    if (ny) *ny = h->n[1];
    if (nz) *nz = h->n[2];
    if (ncomp) *ncomp = h->ncomp;
    return ADS_OK;
}

// Unit operators act on dense caller device arrays: copy into a pitched work field,
// run the kernels, copy back out.
int ads_apply_k(ads_handle h, const double *x, double *out) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (h->dist) return fail(h, ADS_E_INVAL, "unit operators: single-GPU handles only");
    if (!x || !out || x == out) return fail(h, ADS_E_INVAL, "ads_apply_k: bad pointers");
    // U2 (the drift's ping-pong buffer) and W are scratch between steps: the state (U, V, A) is
    // left intact, so get_state and the energies stay valid after a unit operation
    for (int c = 0; c < h->ncomp; ++c)
        if ((rc = copy_in(h, comp(h->U2, h, c), x + c * h->N, ADS_MEM_DEVICE))) return rc;
    if (h->ncomp == 3) {
        if ((rc = ups_apply(h, h->U2, h->U2, 0.0, nullptr, h->W, 1.0))) return rc;
        for (int c = 0; c < 3; ++c)
            if ((rc = copy_out(h, out + c * h->N, comp(h->W, h, c), ADS_MEM_DEVICE))) return rc;
        return ADS_OK;
    }
    if ((rc = run_kop(h, h->U2, h->U2, 0.0, 0.0, 1.0, nullptr, h->R))) return rc;
    return copy_out(h, out, h->R, ADS_MEM_DEVICE);
}

int ads_solve_d(ads_handle h, const double *x, double *out) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (h->dist) return fail(h, ADS_E_INVAL, "unit operators: single-GPU handles only");
    if (!x || !out) return fail(h, ADS_E_INVAL, "ads_solve_d: bad pointers");
    if (h->ncomp == 3) {  // U2 as the work field (el_dsolve's own scratch is W): A, the state, is kept
        for (int c = 0; c < 3; ++c)
            if ((rc = copy_in(h, comp(h->U2, h, c), x + c * h->N, ADS_MEM_DEVICE))) return rc;
        if ((rc = el_dsolve(h, h->U2))) return rc;
        for (int c = 0; c < 3; ++c)
            if ((rc = copy_out(h, out + c * h->N, comp(h->U2, h, c), ADS_MEM_DEVICE))) return rc;
        return ADS_OK;
    }
    if ((rc = copy_in(h, h->R, x, ADS_MEM_DEVICE))) return rc;
    if ((rc = run_sweep(h, 0, h->R, h->Wk, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 1, h->Wk, h->R, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 2, h->R, h->Wk, nullptr, 0.0))) return rc;
    return copy_out(h, out, h->Wk, ADS_MEM_DEVICE);
}

int ads_sweep(ads_handle h, int d, const double *x, double *out) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (!x || !out || d < 0 || d > 2) return fail(h, ADS_E_INVAL, "ads_sweep: bad argument");
    if (h->ncomp != 1 || h->dist) return fail(h, ADS_E_INVAL, "ads_sweep: single-GPU P-wave handles only");
    if ((rc = copy_in(h, h->R, x, ADS_MEM_DEVICE))) return rc;
    if ((rc = run_sweep(h, d, h->R, h->Wk, nullptr, 0.0))) return rc;
    return copy_out(h, out, h->Wk, ADS_MEM_DEVICE);
}

long ads_launch_count(ads_handle h) {
    if (!h) return -1;
    long n = h->launches;
    for (ads_ctx *m : h->members) n += m->launches;
    return n;
}

int ads_step_bytes(ads_handle h, double bytes_per_dof[ADS_NPROF]) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (!bytes_per_dof) return fail(h, ADS_E_INVAL, "ads_step_bytes: NULL output");
    for (int c = 0; c < ADS_NPROF; ++c) bytes_per_dof[c] = 0.0;
    if (h->ncomp != 1) return ADS_OK;
    // kop: U, V -> P, r; sweeps x, y: in -> out; sweep z + kick: r, V -> V (+8 B when a is kept)
    bytes_per_dof[0] = 32.0, bytes_per_dof[1] = 16.0, bytes_per_dof[2] = 16.0, bytes_per_dof[3] = 24.0;
    return ADS_OK;
}

int ads_profile_enable(ads_handle h, int on) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    for (ads_ctx *m : h->members)
        if ((rc = ads_profile_enable(m, on))) return rc;
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    h->prof = on != 0;
    h->prof_rec.clear();
    h->ev_used = 0;
    return ADS_OK;
}

int ads_profile_read(ads_handle h, double *ms, long *count) {
    DeviceScope ds_(h);
    int rc = guard(h);
    if (rc) return rc;
    if (!ms || !count) return fail(h, ADS_E_INVAL, "ads_profile_read: NULL output");
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    for (int c = 0; c < ADS_NPROF; ++c) {
        ms[c] = 0.0;
        count[c] = 0;
    }
    for (ads_ctx *m : slabs_of(h)) {
        CUDA_TRY(m, cudaStreamSynchronize(m->stream));
        for (auto &r : m->prof_rec) {
            float t = 0.f;
            CUDA_TRY(m, cudaEventElapsedTime(&t, r.second.first, r.second.second));
            ms[r.first] += t;
            count[r.first] += 1;
        }
    }
    return ADS_OK;
}

const char *ads_last_error(ads_handle h) { return h ? h->err.c_str() : "null handle"; }

int ads_destroy(ads_handle h) {
    DeviceScope ds_(h);
    if (!h) return ADS_OK;
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (ads_ctx *m : h->members) ads_destroy(m);
    h->members.clear();
    drop_graphs(h);
    if (h->comm && h->dist == 1) ncclCommDestroy(h->comm);
    for (void *p : h->allocs) cudaFree(p);
    for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    for (cudaStream_t st : h->side)
        if (st) cudaStreamDestroy(st);
    for (cudaEvent_t ev : h->fev)
        if (ev) cudaEventDestroy(ev);
    delete h;
    return ADS_OK;
}

}  // extern "C"
