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
#include <new>
#include <string>
#include <vector>

#include "../../include/ads.h"
#include "host_setup.h"
#include "kernels.cuh"

using namespace ads;

namespace {

struct DirDev {
    double *mband = nullptr, *kband = nullptr, *aband = nullptr;  // [n][2p+1]
    double *l = nullptr, *us = nullptr, *dinv = nullptr, *Tf = nullptr, *Rb = nullptr;
    int t_lo = 1, t_hi = 0;  // rows [t_lo, t_hi] of M, K are the Toeplitz row (mrow, krow)
    double mrow[2 * kMaxP + 1] = {}, krow[2 * kMaxP + 1] = {};
    SolveTab tab;
};

}  // namespace

struct ads_ctx {
    int nel[3] = {0, 0, 0}, n[3] = {0, 0, 0};
    int p = 0, bc = 0, ncomp = 1;
    double tau = 0.0;
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
    double *U = nullptr, *U2 = nullptr, *V = nullptr, *A = nullptr, *R = nullptr, *Wk = nullptr;
    double *dpartial = nullptr, *dres = nullptr;
    // source
    double *src[3] = {nullptr, nullptr, nullptr};
    bool has_src = false;
    int wavelet = 0;
    double f0 = 0, t0 = 0, amp = 0;
    std::vector<void *> allocs;
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

double source_g(const ads_ctx *h, double t) {
    if (!h->has_src) return 0.0;
    return h->wavelet == ADS_WAVELET_RICKER ? h->amp * ricker(t, h->f0, h->t0) : h->amp;
}

int build_direction(ads_ctx *h, int d) {
    Space1D &s = h->sp[d];
    const int p = h->p;
    if (build_space(p, h->nel[d], h->bc, s)) return fail(h, ADS_E_INVAL, "bad 1D space");
    const int n = s.n, W = 2 * p + 1;
    const double eta = h->tau * h->tau / 4.0;
    Band A(n, p), Mm = s.M;
    for (size_t q = 0; q < A.v.size(); ++q) A.v[q] = s.M.v[q] + eta * s.K.v[q];
    if (h->bc == ADS_BC_DIRICHLET0) {
        A.at(0, 0) = 1.0;
        A.at(n - 1, n - 1) = 1.0;
        Mm.at(0, 0) = 1.0;
        Mm.at(n - 1, n - 1) = 1.0;
    }
    LUFactors f;
    if (banded_lu(A, f, /*freeze=*/true)) return fail(h, ADS_E_SINGULAR, "A_%d singular", d);
    if (banded_lu(Mm, h->mass_lu[d])) return fail(h, ADS_E_SINGULAR, "M_%d singular", d);
    const int C = kSweepChunks;
    const int L = choose_chunk_len(n, p, C);
    if (L == 0) return fail(h, ADS_E_INVAL, "n_%d = %d: no supported chunking", d, n);
    // pad the factors to C*L rows with identity rows: every chunk has length L
    const int npad = C * L;
    LUFactors fp = f;
    fp.n = npad;
    fp.l.resize((size_t)npad * p, 0.0);
    fp.us.resize((size_t)npad * p, 0.0);
    fp.dinv.resize(npad, 1.0);
    PartTables pt;
    build_part_tables(fp, C, L, pt);
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
    std::vector<double> mb(s.M.v), kb(s.K.v), ab(A.v);
    (void)W;
    if ((rc = upload(h, &D.mband, mb)) || (rc = upload(h, &D.kband, kb)) || (rc = upload(h, &D.aband, ab)) ||
        (rc = upload(h, &D.l, fp.l)) || (rc = upload(h, &D.us, fp.us)) || (rc = upload(h, &D.dinv, fp.dinv)) ||
        (rc = upload(h, &D.Tf, pt.Tf)) || (rc = upload(h, &D.Rb, pt.Rb)))
        return rc;
    D.tab.l = D.l;
    D.tab.us = D.us;
    D.tab.dinv = D.dinv;
    D.tab.Tf = D.Tf;
    D.tab.Rb = D.Rb;
    D.tab.n = n;
    D.tab.L = L;
    D.tab.Kf = pt.Kf;
    D.tab.Kb = pt.Kb;
    // uniform region aligned to whole chunks: chunks [c_lo, c_hi) lie inside [i_lo, i_hi)
    const int c_lo = (f.i_lo + L - 1) / L, c_hi = f.i_hi / L;
    D.tab.c_lo = c_hi > c_lo ? c_lo : 0;
    D.tab.c_hi = c_hi > c_lo ? c_hi : 0;
    if (D.tab.c_hi > D.tab.c_lo) {
        for (int k = 0; k < p; ++k) {
            D.tab.lc[k] = f.l[(size_t)f.i_lo * p + k];
            D.tab.usc[k] = f.us[(size_t)f.i_lo * p + k];
        }
        D.tab.dic = f.dinv[f.i_lo];
        const int s0 = D.tab.c_lo * L;  // any uniform chunk: its responses are bitwise identical
        for (int j = 0; j < L; ++j)
            for (int m = 0; m < p; ++m) {
                D.tab.Gf[j][m] = pt.gf[(size_t)(s0 + j) * p + m];
                D.tab.Gb[j][m] = pt.gb[(size_t)(s0 + j) * p + m];
            }
    }
    return ADS_OK;
}

int guard(ads_ctx *h) {
    if (!h) return ADS_E_INVAL;
    if (h->failed) return ADS_E_STATE;
    return ADS_OK;
}

// ---- step pieces ----
int run_kop(ads_ctx *h, const double *U, const double *V, double tau_d, double g, double sign, double *Pout,
            double *r) {
    KopArgs a;
    a.U = U;
    a.V = V;
    a.Pout = Pout;
    a.r = r;
    a.tau = tau_d;
    a.g = g;
    a.sign = sign;
    if (h->has_src && g != 0.0) {
        a.bx = h->src[0];
        a.by = h->src[1];
        a.bz = h->src[2];
    }
    a.mx = h->dd[0].mband;
    a.kx = h->dd[0].kband;
    a.my = h->dd[1].mband;
    a.ky = h->dd[1].kband;
    a.mz = h->dd[2].mband;
    a.kz = h->dd[2].kband;
    a.geo = h->geo;
    a.zlen = 0;
    for (int d = 0; d < 3; ++d) {
        a.ilo[d] = h->dd[d].t_lo;
        a.ihi[d] = h->dd[d].t_hi;
        for (int c = 0; c < 2 * h->p + 1; ++c) {
            a.mc[d][c] = h->dd[d].mrow[c];
            a.kc[d][c] = h->dd[d].krow[c];
        }
    }
    ProfScope ps(h, 0);
    if (launch_kop(h->p, a, h->stream)) return fail(h, ADS_E_INVAL, "kop: unsupported p");
    return check_launch(h, "kop");
}

int run_sweep(ads_ctx *h, int d, const double *in, double *out, double *V, double kick) {
    SweepArgs a;
    a.in = in;
    a.out = out;
    a.V = V;
    a.kick = kick;
    a.t = h->dd[d].tab;
    a.geo = h->geo;
    a.dir = d;
    a.mode = V ? 1 : 0;
    ProfScope ps(h, 1 + d);
    if (launch_sweep(h->p, a, h->stream)) return fail(h, ADS_E_INVAL, "sweep: unsupported p/chunk");
    return check_launch(h, "sweep");
}

// a = D^-1 r along x, y, z; z-sweep kicks V += kick * a and stores a into aout (nullable)
int run_solve(ads_ctx *h, const double *r_in, double *scratch, double *r2, double *aout, double *V, double kick) {
    int rc;
    if ((rc = run_sweep(h, 0, r_in, scratch, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 1, scratch, r2, nullptr, 0.0))) return rc;
    return run_sweep(h, 2, r2, aout, V, kick);
}

int init_state(ads_ctx *h) {
    // half-kick start (C2): a0 = D^-1 (F(0) - K u0); V0 = udot0 + tau/2 a0
    int rc;
    if ((rc = run_kop(h, h->U, h->V, 0.0, source_g(h, 0.0), -1.0, nullptr, h->R))) return rc;
    if ((rc = run_sweep(h, 0, h->R, h->Wk, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 1, h->Wk, h->R, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 2, h->R, h->A, h->V, 0.5 * h->tau))) return rc;
    h->step = 0;
    h->have_state = true;
    return ADS_OK;
}

int copy_in(ads_ctx *h, double *dst, const double *src, int mem) {
    cudaMemcpyKind k = mem == ADS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // dense caller array -> pitched device field
    CUDA_TRY(h, cudaMemcpy2DAsync(dst, sizeof(double) * h->geo.sy, src, sizeof(double) * h->n[0],
                                  sizeof(double) * h->n[0], (size_t)h->n[1] * h->n[2], k, h->stream));
    return ADS_OK;
}

int copy_out(ads_ctx *h, double *dst, const double *src, int mem) {
    cudaMemcpyKind k = mem == ADS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CUDA_TRY(h, cudaMemcpy2DAsync(dst, sizeof(double) * h->n[0], src, sizeof(double) * h->geo.sy,
                                  sizeof(double) * h->n[0], (size_t)h->n[1] * h->n[2], k, h->stream));
    return ADS_OK;
}

}  // namespace

extern "C" {

int ads_create(ads_handle *out, int nx, int ny, int nz, int p, double tau, int bc) {
    if (!out) return ADS_E_INVAL;
    *out = nullptr;
    if (p < 1 || p > 5 || nx < 1 || ny < 1 || nz < 1 || !(tau > 0.0) || !std::isfinite(tau) ||
        (bc != ADS_BC_NATURAL && bc != ADS_BC_DIRICHLET0))
        return ADS_E_INVAL;
    if (bc == ADS_BC_DIRICHLET0 && (nx + p < 3 || ny + p < 3 || nz + p < 3)) return ADS_E_INVAL;
    ads_ctx *h = new (std::nothrow) ads_ctx;
    if (!h) return ADS_E_NOMEM;
    h->p = p;
    h->bc = bc;
    h->tau = tau;
    h->nel[0] = nx;
    h->nel[1] = ny;
    h->nel[2] = nz;
    int rc = ADS_OK;
    cudaGetDevice(&h->device);
    for (int d = 0; d < 3 && rc == ADS_OK; ++d) {
        h->n[d] = h->nel[d] + p;
        rc = build_direction(h, d);
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
        size_t fb = sizeof(double) * h->Nalloc;
        if ((rc = dalloc(h, (void **)&h->U, fb)) == ADS_OK && (rc = dalloc(h, (void **)&h->U2, fb)) == ADS_OK &&
            (rc = dalloc(h, (void **)&h->V, fb)) == ADS_OK && (rc = dalloc(h, (void **)&h->A, fb)) == ADS_OK &&
            (rc = dalloc(h, (void **)&h->R, fb)) == ADS_OK && (rc = dalloc(h, (void **)&h->Wk, fb)) == ADS_OK &&
            (rc = dalloc(h, (void **)&h->dpartial, sizeof(double) * 1024)) == ADS_OK &&
            (rc = dalloc(h, (void **)&h->dres, sizeof(double) * 8)) == ADS_OK) {
            cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
            if (e != cudaSuccess) rc = fail(h, ADS_E_CUDA, "stream: %s", cudaGetErrorString(e));
            h->own_stream = true;
        }
        if (rc == ADS_OK) {
            for (double *f : {h->U, h->U2, h->V, h->A, h->R, h->Wk}) cudaMemsetAsync(f, 0, fb, h->stream);
            if (cudaStreamSynchronize(h->stream) != cudaSuccess) rc = fail(h, ADS_E_CUDA, "memset failed");
        }
    }
    if (rc != ADS_OK) {
        ads_destroy(h);
        return rc;
    }
    *out = h;
    return ADS_OK;
}

int ads_create_elastic(ads_handle *out, int, int, int, int, double, int, double, double, double) {
    if (out) *out = nullptr;
    return ADS_E_INVAL;  // implemented in a later milestone
}

int ads_set_stream(ads_handle h, void *stream) {
    int rc = guard(h);
    if (rc) return rc;
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    if (stream) {
        if (h->own_stream) cudaStreamDestroy(h->stream);
        h->stream = (cudaStream_t)stream;
        h->own_stream = false;
    } else if (!h->own_stream) {
        CUDA_TRY(h, cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
    }
    return ADS_OK;
}

int ads_load_vector(ads_handle h, int d, int func, double c, double sigma, double *out) {
    int rc = guard(h);
    if (rc) return rc;
    if (d < 0 || d > 2 || !out || (func != ADS_FUNC_SIN && func != ADS_FUNC_GAUSS) ||
        (func == ADS_FUNC_GAUSS && !(sigma > 0.0)))
        return fail(h, ADS_E_INVAL, "ads_load_vector: bad argument");
    load_vector(h->sp[d], func, c, sigma, out);
    return ADS_OK;
}

int ads_mass_solve_1d(ads_handle h, int d, double *x) {
    int rc = guard(h);
    if (rc) return rc;
    if (d < 0 || d > 2 || !x) return fail(h, ADS_E_INVAL, "ads_mass_solve_1d: bad argument");
    lu_solve_host(h->mass_lu[d], x);
    return ADS_OK;
}

int ads_set_source(ads_handle h, const double *bx, const double *by, const double *bz, int wavelet, double f0,
                   double t0, double amp) {
    int rc = guard(h);
    if (rc) return rc;
    if (!bx) {
        h->has_src = false;
        return ADS_OK;
    }
    if (!by || !bz || (wavelet != ADS_WAVELET_NONE && wavelet != ADS_WAVELET_RICKER))
        return fail(h, ADS_E_INVAL, "ads_set_source: bad argument");
    const double *b[3] = {bx, by, bz};
    for (int d = 0; d < 3; ++d) {
        std::vector<double> v(b[d], b[d] + h->n[d]);
        if (h->bc == ADS_BC_DIRICHLET0) v[0] = v[h->n[d] - 1] = 0.0;
        if (!h->src[d]) {
            if ((rc = dalloc(h, (void **)&h->src[d], sizeof(double) * h->n[d]))) return rc;
        }
        CUDA_TRY(h, cudaMemcpy(h->src[d], v.data(), sizeof(double) * h->n[d], cudaMemcpyHostToDevice));
    }
    h->has_src = true;
    h->wavelet = wavelet;
    h->f0 = f0;
    h->t0 = t0;
    h->amp = amp;
    return ADS_OK;
}

int ads_set_state(ads_handle h, const double *u, const double *udot, int mem) {
    int rc = guard(h);
    if (rc) return rc;
    if (!u || (mem != ADS_MEM_HOST && mem != ADS_MEM_DEVICE)) return fail(h, ADS_E_INVAL, "ads_set_state: bad argument");
    if ((rc = copy_in(h, h->U, u, mem))) return rc;
    if (udot) {
        if ((rc = copy_in(h, h->V, udot, mem))) return rc;
    } else {
        CUDA_TRY(h, cudaMemsetAsync(h->V, 0, sizeof(double) * h->Nalloc, h->stream));
    }
    if (h->bc == ADS_BC_DIRICHLET0) {
        launch_mask_boundary(h->U, h->geo, h->stream);
        if ((rc = check_launch(h, "mask"))) return rc;
        launch_mask_boundary(h->V, h->geo, h->stream);
        if ((rc = check_launch(h, "mask"))) return rc;
    }
    return init_state(h);
}

int ads_set_state_separable(ads_handle h, int nterms, const double *amp, const int *comp, const double *sx,
                            const double *sy, const double *sz) {
    int rc = guard(h);
    if (rc) return rc;
    if (nterms < 0 || (nterms > 0 && (!amp || !sx || !sy || !sz)))
        return fail(h, ADS_E_INVAL, "ads_set_state_separable: bad argument");
    CUDA_TRY(h, cudaMemsetAsync(h->U, 0, sizeof(double) * h->Nalloc, h->stream));
    CUDA_TRY(h, cudaMemsetAsync(h->V, 0, sizeof(double) * h->Nalloc, h->stream));
    if (nterms > 0) {
        const int n0 = h->n[0], n1 = h->n[1], n2 = h->n[2];
        std::vector<double> packed((size_t)nterms * (n0 + n1 + n2));
        double *d = nullptr;
        if ((rc = dalloc(h, (void **)&d, sizeof(double) * packed.size()))) return rc;
        for (int t = 0; t < nterms; ++t) {
            std::memcpy(&packed[(size_t)t * (n0 + n1 + n2)], sx + (size_t)t * n0, sizeof(double) * n0);
            std::memcpy(&packed[(size_t)t * (n0 + n1 + n2) + n0], sy + (size_t)t * n1, sizeof(double) * n1);
            std::memcpy(&packed[(size_t)t * (n0 + n1 + n2) + n0 + n1], sz + (size_t)t * n2, sizeof(double) * n2);
        }
        CUDA_TRY(h, cudaMemcpy(d, packed.data(), sizeof(double) * packed.size(), cudaMemcpyHostToDevice));
        for (int t = 0; t < nterms; ++t) {
            if (comp && comp[t] != 0) return fail(h, ADS_E_INVAL, "component %d on a scalar handle", comp[t]);
            const double *b = d + (size_t)t * (n0 + n1 + n2);
            launch_add_separable(h->U, amp[t], b, b + n0, b + n0 + n1, h->geo, h->stream);
            if ((rc = check_launch(h, "separable"))) return rc;
        }
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
        cudaFree(d);
        h->allocs.pop_back();
    }
    if (h->bc == ADS_BC_DIRICHLET0) {
        launch_mask_boundary(h->U, h->geo, h->stream);
        if ((rc = check_launch(h, "mask"))) return rc;
    }
    return init_state(h);
}

int ads_step(ads_handle h, int nsteps) {
    int rc = guard(h);
    if (rc) return rc;
    if (nsteps < 0) return fail(h, ADS_E_INVAL, "nsteps < 0");
    if (!h->have_state) return fail(h, ADS_E_STATE, "ads_step before ads_set_state");
    for (int s = 0; s < nsteps; ++s) {
        const double t1 = (double)(h->step + 1) * h->tau;  // F at t_{n+1} (C14)
        // drift + RHS: U2 = U + tau V, R = F(t_{n+1}) - K U2
        if ((rc = run_kop(h, h->U, h->V, h->tau, source_g(h, t1), -1.0, h->U2, h->R))) return rc;
        // a = D^-1 R; V += tau a; keep a only on the last step of the batch
        if ((rc = run_solve(h, h->R, h->Wk, h->R, s == nsteps - 1 ? h->A : nullptr, h->V, h->tau))) return rc;
        std::swap(h->U, h->U2);
        h->step += 1;
    }
    return ADS_OK;
}

int ads_energy(ads_handle h, double out[3]) {
    int rc = guard(h);
    if (rc) return rc;
    if (!out) return fail(h, ADS_E_INVAL, "ads_energy: out is NULL");
    const Geom &g = h->geo;
    const long N = h->Nalloc;  // padding entries are 0 in every field
    double res[3];
    // v = V - tau/2 a ; kinetic = 1/2 v' M v
    CUDA_TRY(h, cudaMemcpyAsync(h->R, h->V, sizeof(double) * N, cudaMemcpyDeviceToDevice, h->stream));
    launch_axpby(N, -0.5 * h->tau, h->A, 1.0, h->R, h->stream);
    if ((rc = check_launch(h, "axpby"))) return rc;
    launch_axis_apply(h->p, 0, h->dd[0].mband, h->R, h->Wk, g, h->stream);
    launch_axis_apply(h->p, 1, h->dd[1].mband, h->Wk, h->U2, g, h->stream);
    launch_axis_apply(h->p, 2, h->dd[2].mband, h->U2, h->Wk, g, h->stream);
    if ((rc = check_launch(h, "axis_apply"))) return rc;
    launch_dot(N, h->R, h->Wk, h->dpartial, h->dres + 0, h->stream);
    // potential = 1/2 U' K U
    if ((rc = run_kop(h, h->U, h->V, 0.0, 0.0, 1.0, nullptr, h->R))) return rc;
    launch_dot(N, h->U, h->R, h->dpartial, h->dres + 1, h->stream);
    // invariant = 1/2 V' D V + 1/2 U_n' K U_{n+1}
    launch_axis_apply(h->p, 0, h->dd[0].aband, h->V, h->Wk, g, h->stream);
    launch_axis_apply(h->p, 1, h->dd[1].aband, h->Wk, h->U2, g, h->stream);
    launch_axis_apply(h->p, 2, h->dd[2].aband, h->U2, h->Wk, g, h->stream);
    launch_dot(N, h->V, h->Wk, h->dpartial, h->dres + 2, h->stream);
    if ((rc = run_kop(h, h->U, h->V, h->tau, 0.0, 1.0, nullptr, h->R))) return rc;
    launch_dot(N, h->U, h->R, h->dpartial, h->dres + 3, h->stream);
    if ((rc = check_launch(h, "dot"))) return rc;
    double d4[4];
    CUDA_TRY(h, cudaMemcpyAsync(d4, h->dres, sizeof(double) * 4, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    res[0] = 0.5 * d4[0];
    res[1] = 0.5 * d4[1];
    res[2] = 0.5 * d4[2] + 0.5 * d4[3];
    for (int i = 0; i < 3; ++i) {
        if (!std::isfinite(res[i])) return fail(h, ADS_E_STATE, "non-finite energy (NaN/Inf in state)");
        out[i] = res[i];
    }
    return ADS_OK;
}

int ads_get_state(ads_handle h, double *u, double *udot, double *a, int mem) {
    int rc = guard(h);
    if (rc) return rc;
    if (mem != ADS_MEM_HOST && mem != ADS_MEM_DEVICE) return fail(h, ADS_E_INVAL, "bad mem");
    if (u && (rc = copy_out(h, u, h->U, mem))) return rc;
    if (udot) {
        CUDA_TRY(h, cudaMemcpyAsync(h->Wk, h->V, sizeof(double) * h->Nalloc, cudaMemcpyDeviceToDevice, h->stream));
        launch_axpby(h->Nalloc, -0.5 * h->tau, h->A, 1.0, h->Wk, h->stream);
        if ((rc = check_launch(h, "axpby"))) return rc;
        if ((rc = copy_out(h, udot, h->Wk, mem))) return rc;
    }
    if (a && (rc = copy_out(h, a, h->A, mem))) return rc;
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return ADS_OK;
}

double ads_time(ads_handle h) { return h ? (double)h->step * h->tau : NAN; }
long ads_step_count(ads_handle h) { return h ? h->step : -1; }

int ads_dims(ads_handle h, int *nx, int *ny, int *nz, int *ncomp) {
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
    int rc = guard(h);
    if (rc) return rc;
    if (!x || !out || x == out) return fail(h, ADS_E_INVAL, "ads_apply_k: bad pointers");
    if ((rc = copy_in(h, h->U2, x, ADS_MEM_DEVICE))) return rc;
    if ((rc = run_kop(h, h->U2, h->U2, 0.0, 0.0, 1.0, nullptr, h->R))) return rc;
    return copy_out(h, out, h->R, ADS_MEM_DEVICE);
}

int ads_solve_d(ads_handle h, const double *x, double *out) {
    int rc = guard(h);
    if (rc) return rc;
    if (!x || !out) return fail(h, ADS_E_INVAL, "ads_solve_d: bad pointers");
    if ((rc = copy_in(h, h->R, x, ADS_MEM_DEVICE))) return rc;
    if ((rc = run_sweep(h, 0, h->R, h->Wk, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 1, h->Wk, h->R, nullptr, 0.0))) return rc;
    if ((rc = run_sweep(h, 2, h->R, h->Wk, nullptr, 0.0))) return rc;
    return copy_out(h, out, h->Wk, ADS_MEM_DEVICE);
}

int ads_sweep(ads_handle h, int d, const double *x, double *out) {
    int rc = guard(h);
    if (rc) return rc;
    if (!x || !out || d < 0 || d > 2) return fail(h, ADS_E_INVAL, "ads_sweep: bad argument");
    if ((rc = copy_in(h, h->R, x, ADS_MEM_DEVICE))) return rc;
    if ((rc = run_sweep(h, d, h->R, h->Wk, nullptr, 0.0))) return rc;
    return copy_out(h, out, h->Wk, ADS_MEM_DEVICE);
}

long ads_launch_count(ads_handle h) { return h ? h->launches : -1; }

int ads_profile_enable(ads_handle h, int on) {
    int rc = guard(h);
    if (rc) return rc;
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    h->prof = on != 0;
    h->prof_rec.clear();
    h->ev_used = 0;
    return ADS_OK;
}

int ads_profile_read(ads_handle h, double *ms, long *count) {
    int rc = guard(h);
    if (rc) return rc;
    if (!ms || !count) return fail(h, ADS_E_INVAL, "ads_profile_read: NULL output");
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    for (int c = 0; c < ADS_NPROF; ++c) {
        ms[c] = 0.0;
        count[c] = 0;
    }
    for (auto &r : h->prof_rec) {
        float t = 0.f;
        CUDA_TRY(h, cudaEventElapsedTime(&t, r.second.first, r.second.second));
        ms[r.first] += t;
        count[r.first] += 1;
    }
    return ADS_OK;
}

const char *ads_last_error(ads_handle h) { return h ? h->err.c_str() : "null handle"; }

int ads_destroy(ads_handle h) {
    if (!h) return ADS_OK;
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (void *p : h->allocs) cudaFree(p);
    for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return ADS_OK;
}

}  // extern "C"
