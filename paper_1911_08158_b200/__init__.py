"""Thin Python binding of libads_b200.so (include/ads.h), argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
passes pointers and sizes.  There is no CPU fallback: if the shared library is
missing or cannot be loaded, import fails loudly (``AdsError``).

Host arrays are numpy float64; device arrays are torch float64 CUDA tensors
(PyTorch is used only for device memory and streams).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADS_B200_LIB") or os.path.join(_HERE, "libads_b200.so")  # env: experiment builds

ADS_BC_NATURAL, ADS_BC_DIRICHLET0 = 0, 1
ADS_MEM_HOST, ADS_MEM_DEVICE = 0, 1
ADS_FUNC_SIN, ADS_FUNC_GAUSS = 0, 1
ADS_WAVELET_NONE, ADS_WAVELET_RICKER = 0, 1
_ERRS = {-1: "ADS_E_INVAL", -2: "ADS_E_SINGULAR", -3: "ADS_E_CUDA", -4: "ADS_E_NCCL", -5: "ADS_E_NOMEM",
         -6: "ADS_E_STATE"}

# every symbol include/ads.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "ads_create", "ads_create_elastic", "ads_set_stream", "ads_load_vector", "ads_mass_solve_1d",
    "ads_set_source", "ads_set_state", "ads_set_state_separable", "ads_step", "ads_energy", "ads_get_state",
    "ads_time", "ads_step_count", "ads_dims", "ads_apply_k", "ads_solve_d", "ads_sweep", "ads_launch_count",
    "ads_last_error", "ads_destroy", "ads_profile_enable", "ads_profile_read", "ads_step_bytes",
    "ads_get_unique_id", "ads_slab_plan", "ads_create_dist", "ads_create_virtual", "ads_local_extent",
    "ads_modal_basis", "ads_modal_advance", "ads_set_scheme", "ads_set_tau", "ads_set_zsolve",
]


class AdsError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{_ERRS.get(code, code)}: {msg}")
        self.code = code


_lib = None
_H = ctypes.c_void_p
_I, _D, _L = ctypes.c_int, ctypes.c_double, ctypes.c_long
_VP = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise AdsError(-3, f"CUDA extension not built: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "ads_create": (_I, [ctypes.POINTER(_H), _I, _I, _I, _I, _D, _I]),
            "ads_create_elastic": (_I, [ctypes.POINTER(_H), _I, _I, _I, _I, _D, _I, _D, _D, _D]),
            "ads_set_stream": (_I, [_H, _VP]),
            "ads_load_vector": (_I, [_H, _I, _I, _D, _D, _VP]),
            "ads_mass_solve_1d": (_I, [_H, _I, _VP]),
            "ads_set_source": (_I, [_H, _VP, _VP, _VP, _I, _D, _D, _D]),
            "ads_set_state": (_I, [_H, _VP, _VP, _I]),
            "ads_set_state_separable": (_I, [_H, _I, _VP, _VP, _VP, _VP, _VP]),
            "ads_step": (_I, [_H, _I]),
            "ads_energy": (_I, [_H, _VP]),
            "ads_get_state": (_I, [_H, _VP, _VP, _VP, _I]),
            "ads_time": (_D, [_H]),
            "ads_step_count": (_L, [_H]),
            "ads_dims": (_I, [_H, _VP, _VP, _VP, _VP]),
            "ads_apply_k": (_I, [_H, _VP, _VP]),
            "ads_solve_d": (_I, [_H, _VP, _VP]),
            "ads_sweep": (_I, [_H, _I, _VP, _VP]),
            "ads_launch_count": (_L, [_H]),
            "ads_last_error": (ctypes.c_char_p, [_H]),
            "ads_destroy": (_I, [_H]),
            "ads_profile_enable": (_I, [_H, _I]),
            "ads_profile_read": (_I, [_H, _VP, _VP]),
            "ads_step_bytes": (_I, [_H, _VP]),
            "ads_get_unique_id": (_I, [_VP]),
            "ads_slab_plan": (_I, [_I, _I, _I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
            "ads_create_dist": (_I, [ctypes.POINTER(_H), _I, _I, _I, _I, _D, _I, _I, _I, _VP, _I]),
            "ads_create_virtual": (_I, [ctypes.POINTER(_H), _I, _I, _I, _I, _D, _I, _I]),
            "ads_local_extent": (_I, [_H, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
            "ads_modal_basis": (_I, [_I, _I, _I, _VP, _VP]),
            "ads_modal_advance": (_I, [_H, _L]),
            "ads_set_scheme": (_I, [_H, _I]),
            "ads_set_tau": (_I, [_H, _D]),
            "ads_set_zsolve": (_I, [_H, _I]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _host(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data


def _ptr_mem(x):
    """(keepalive, pointer, mem) for a numpy host array or a torch float64 tensor."""
    if x is None:
        return None, None, ADS_MEM_HOST
    if hasattr(x, "data_ptr"):  # torch tensor
        import torch
        assert x.dtype == torch.float64 and x.is_contiguous()
        if x.is_cuda:
            return x, x.data_ptr(), ADS_MEM_DEVICE
        return x, x.data_ptr(), ADS_MEM_HOST
    a, p = _host(x)
    return a, p, ADS_MEM_HOST


def get_unique_id() -> bytes:
    """NCCL unique id (128 bytes) for Solver(dist=...); host-only."""
    buf = (ctypes.c_ubyte * 128)()
    rc = lib().ads_get_unique_id(buf)
    if rc != 0:
        raise AdsError(rc, "ads_get_unique_id failed")
    return bytes(buf)


def modal_basis(nel, p, bc=1):
    """(lambda, phi): the 1D generalised eigenpairs K phi = lambda M phi, phi^T M phi = I, of one
    direction on its active DOFs (ads_modal_basis; host-only)."""
    na = nel + p - (2 if bc == ADS_BC_DIRICHLET0 else 0)
    lam = np.zeros(max(na, 0))
    phi = np.zeros((max(na, 0), max(na, 0)))
    rc = lib().ads_modal_basis(nel, p, bc, lam.ctypes.data, phi.ctypes.data)
    if rc != 0:
        raise AdsError(rc, "ads_modal_basis failed")
    return lam, phi


def slab_plan(nz, p, world, rank):
    """(z_begin, z_count): global planes owned by slab `rank` for nz elements (host-only)."""
    b, c = ctypes.c_int(), ctypes.c_int()
    rc = lib().ads_slab_plan(nz, p, world, rank, ctypes.byref(b), ctypes.byref(c))
    if rc != 0:
        raise AdsError(rc, "ads_slab_plan failed")
    return b.value, c.value


def broadcast_unique_id(rank, group=None) -> bytes:
    """Rank 0 creates the NCCL id, torch.distributed broadcasts it (any backend, CPU tensor)."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t = torch.tensor(list(get_unique_id()), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().tolist())


class Solver:
    """One ADS solver handle on the current CUDA device: P-wave or elasticity on one GPU,
    a z-slab of a multi-GPU grid (dist=(rank, world, uid)), or all slabs of a grid on this
    device exchanging by device copies (virtual_slabs=G)."""

    def __init__(self, nel, p, tau, bc=ADS_BC_DIRICHLET0, elastic=False, lam=1.0, mu=1.0, rho=1.0, dist=None,
                 virtual_slabs=0, device=None):
        if isinstance(nel, int):
            nel = (nel, nel, nel)
        h = _H()
        if elastic:
            rc = lib().ads_create_elastic(ctypes.byref(h), nel[0], nel[1], nel[2], p, tau, bc, lam, mu, rho)
        elif dist is not None:
            rank, world, uid = dist
            buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
            if device is None:
                import torch
                device = torch.cuda.current_device()
            rc = lib().ads_create_dist(ctypes.byref(h), nel[0], nel[1], nel[2], p, tau, bc, rank, world, buf, device)
        elif virtual_slabs:
            rc = lib().ads_create_virtual(ctypes.byref(h), nel[0], nel[1], nel[2], p, tau, bc, virtual_slabs)
        else:
            rc = lib().ads_create(ctypes.byref(h), nel[0], nel[1], nel[2], p, tau, bc)
        if rc != 0:
            raise AdsError(rc, "ads_create failed")
        self.h = h
        self.nel, self.p, self.tau, self.bc, self.elastic = tuple(nel), p, tau, bc, elastic
        n = (ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int())
        lib().ads_dims(h, *(ctypes.byref(x) for x in n))
        zb, zc = ctypes.c_int(), ctypes.c_int()
        lib().ads_local_extent(h, ctypes.byref(zb), ctypes.byref(zc))
        self.z_begin, self.z_count = zb.value, zc.value
        self.n = (n[0].value, n[1].value, n[2].value)  # z: owned planes for a dist slab
        self.ncomp = n[3].value
        self.N = self.n[0] * self.n[1] * self.n[2]
        self.shape = ((3,) if elastic else ()) + (self.n[2], self.n[1], self.n[0])

    def _check(self, rc):
        if rc != 0:
            raise AdsError(rc, lib().ads_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ads_destroy(self.h)
        self.h = None

    __del__ = close

    def set_stream(self, stream=None):
        """Attach a torch.cuda.Stream (or raw cudaStream_t int).  None, or PyTorch's default stream
        (cuda_stream 0), selects the library's own stream, which is ordered against the default
        stream (include/ads.h ads_set_stream)."""
        ptr = None if stream is None else getattr(stream, "cuda_stream", stream)
        self._check(lib().ads_set_stream(self.h, ptr))

    def load_vector(self, d, func):
        """1D load vector (global length n_d = nel_d + p, also for slabs)."""
        nd = self.nel[d] + self.p if 0 <= d < 3 else 1  # bad d: the library reports ADS_E_INVAL
        out = np.zeros(nd)
        if func[0] == "sin":
            self._check(lib().ads_load_vector(self.h, d, ADS_FUNC_SIN, 0.0, 1.0, out.ctypes.data))
        else:
            self._check(lib().ads_load_vector(self.h, d, ADS_FUNC_GAUSS, float(func[1]), float(func[2]),
                                              out.ctypes.data))
        return out

    def mass_solve_1d(self, d, x):
        x = np.array(x, dtype=np.float64, copy=True)
        self._check(lib().ads_mass_solve_1d(self.h, d, x.ctypes.data))
        return x

    def set_source(self, b=None, wavelet=ADS_WAVELET_RICKER, f0=25.0, t0=0.04, amp=1.0):
        if b is None:
            self._check(lib().ads_set_source(self.h, None, None, None, 0, 0.0, 0.0, 0.0))
            return
        bs = [_host(x)[0] for x in b]
        self._check(lib().ads_set_source(self.h, bs[0].ctypes.data, bs[1].ctypes.data, bs[2].ctypes.data,
                                         wavelet, f0, t0, amp))

    def set_state(self, u, udot=None):
        ku, pu, mem = _ptr_mem(u)
        kv, pv, memv = _ptr_mem(udot)
        if udot is not None and memv != mem:
            raise ValueError("u and udot must live in the same memory")
        self._check(lib().ads_set_state(self.h, pu, pv, mem))

    def set_state_separable(self, amps, sx, sy, sz, comps=None):
        amps = np.ascontiguousarray(amps, dtype=np.float64)
        sx, sy, sz = (np.ascontiguousarray(s, dtype=np.float64) for s in (sx, sy, sz))
        comp = None if comps is None else np.ascontiguousarray(comps, dtype=np.int32)
        self._check(lib().ads_set_state_separable(self.h, len(amps), amps.ctypes.data,
                                                  None if comp is None else comp.ctypes.data,
                                                  sx.ctypes.data, sy.ctypes.data, sz.ctypes.data))

    def step(self, nsteps=1):
        self._check(lib().ads_step(self.h, nsteps))

    def set_tau(self, tau):
        """Continue with step size tau from the current state and time (ads_set_tau)."""
        self._check(lib().ads_set_tau(self.h, tau))
        self.tau = tau

    def set_scheme(self, scheme):
        """1 = reading R1 (default), 0 = the literal Eq. 16 (ads_set_scheme); set the state again."""
        self._check(lib().ads_set_scheme(self.h, scheme))

    def set_zsolve(self, mode):
        """Slab handles: 0 = distributed SPIKE (default), 1 = all-to-all transpose (ads_set_zsolve)."""
        self._check(lib().ads_set_zsolve(self.h, mode))

    def modal_advance(self, nsteps):
        """Advance by nsteps R1 steps exactly in modal space (ads_modal_advance)."""
        self._check(lib().ads_modal_advance(self.h, nsteps))

    def energy(self):
        out = np.zeros(3)
        self._check(lib().ads_energy(self.h, out.ctypes.data))
        return out

    def get_state(self, u=None, udot=None, a=None):
        """Return host numpy (U_n, udot_n, a_n), or fill the given device tensors."""
        if u is None and udot is None and a is None:
            u, udot, a = (np.zeros(self.shape) for _ in range(3))
            self._check(lib().ads_get_state(self.h, u.ctypes.data, udot.ctypes.data, a.ctypes.data, ADS_MEM_HOST))
            return u, udot, a
        ks = [_ptr_mem(x) for x in (u, udot, a)]
        mems = {k[2] for k, x in zip(ks, (u, udot, a)) if x is not None}
        if len(mems) != 1:
            raise ValueError("outputs must live in the same memory")
        self._check(lib().ads_get_state(self.h, ks[0][1], ks[1][1], ks[2][1], mems.pop()))
        return u, udot, a

    def time(self):
        return lib().ads_time(self.h)

    def step_count(self):
        return lib().ads_step_count(self.h)

    def launch_count(self):
        return lib().ads_launch_count(self.h)

    def profile_enable(self, on=True):
        self._check(lib().ads_profile_enable(self.h, 1 if on else 0))

    def profile_read(self):
        """(ms[5], count[5]) per kernel class: kop, sweep x, sweep y, sweep z+kick, modal transform."""
        ms = np.zeros(5)
        cnt = np.zeros(5, dtype=np.int64)
        self._check(lib().ads_profile_read(self.h, ms.ctypes.data, cnt.ctypes.data))
        return ms, cnt

    def step_bytes(self):
        """Algorithmic HBM bytes per DOF of each step kernel class (kop, sweep x, y, z; ads_step_bytes)."""
        b = np.zeros(5)
        self._check(lib().ads_step_bytes(self.h, b.ctypes.data))
        return b[:4]

    # unit operations on torch device tensors
    def apply_k(self, x, out):
        self._check(lib().ads_apply_k(self.h, x.data_ptr(), out.data_ptr()))

    def solve_d(self, x, out):
        self._check(lib().ads_solve_d(self.h, x.data_ptr(), out.data_ptr()))

    def sweep(self, d, x, out):
        self._check(lib().ads_sweep(self.h, d, x.data_ptr(), out.data_ptr()))


def project_1d(solver, func, d):
    """s_d = M_d^-1 b_d: the 1D factor of a separable L2 projection."""
    return solver.mass_solve_1d(d, solver.load_vector(d, func))


def make_solver(wl, dist=None, virtual_slabs=0, u0=None, zsolve=0):
    """Solver for a workloads.Workload with its initial state and source set (library-side projection,
    or the given coefficients u0).  dist=(rank, world, uid): this process's z-slab;
    virtual_slabs=G: all G slabs on this device; zsolve: slab z solve (0 SPIKE, 1 all-to-all)."""
    s = Solver(wl.nel, wl.p, wl.tau, wl.bc, elastic=wl.elastic, lam=wl.lam, mu=wl.mu, rho=wl.rho, dist=dist,
               virtual_slabs=virtual_slabs)
    if zsolve:
        s.set_zsolve(zsolve)
    if wl.source is not None:
        src = wl.source
        b = [s.load_vector(d, src.f[d]) for d in range(3)]
        s.set_source(b, src.wavelet, src.f0, src.t0, src.amp)
    terms = wl.u0
    if u0 is not None:
        s.set_state(u0)
    elif terms:
        sx = np.concatenate([project_1d(s, t.f[0], 0) for t in terms])
        sy = np.concatenate([project_1d(s, t.f[1], 1) for t in terms])
        sz = np.concatenate([project_1d(s, t.f[2], 2) for t in terms])
        s.set_state_separable([t.amp for t in terms], sx, sy, sz, [t.comp for t in terms])
    else:
        s.set_state_separable([], np.zeros(0), np.zeros(0), np.zeros(0))
    return s
