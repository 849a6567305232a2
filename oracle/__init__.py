"""Python view of the CPU oracle (oracle/ads_oracle.c) plus the modal oracle.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg may import this package.
It shares no code with ``paper_1911_08158_b200`` (the CUDA product path) and
never imports it.

The C oracle is built by ``build()`` (also called from
``__graft_entry__.build()``) with ``gcc -O2 -ffp-contract=off``: plain,
single-threaded fp64.  The same source is also built with -DOR_LONG_DOUBLE
(x87 extended precision, ``libads_oracle_ld.so``): ``PWave(..., ext=True)`` and
``Elastic(..., ext=True)`` run it as the truth reference for the one-step fp64
bound (T1).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ads_oracle.c")
_LIB = os.path.join(_HERE, "libads_oracle.so")
_LIB_LD = os.path.join(_HERE, "libads_oracle_ld.so")
_lib = None
_lib_ld = None

_D = ctypes.c_double
_I = ctypes.c_int
_P = ctypes.c_void_p
_DP = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    for out, extra in ((_LIB, []), (_LIB_LD, ["-DOR_LONG_DOUBLE"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
            subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c99", *extra,
                                   "-o", out, _SRC, "-lm"])
    return _LIB


def lib(ext: bool = False):
    """The oracle library: fp64 (default) or, ext=True, the same code in x87 extended precision."""
    global _lib, _lib_ld
    if (_lib_ld if ext else _lib) is None:
        build()
        L = ctypes.CDLL(_LIB_LD if ext else _LIB)
        _D = ctypes.c_longdouble if ext else ctypes.c_double
        _DP = ctypes.POINTER(_D)
        sig = {
            "or_knots": (None, [_I, _I, _DP]),
            "or_bspline": (_D, [_DP, _I, _I, _D]),
            "or_bspline_d": (_D, [_DP, _I, _I, _D]),
            "or_gauss": (None, [_I, _DP, _DP]),
            "or_matrices_1d": (_I, [_I, _I, _I, _DP, _DP, _DP]),
            "or_load_1d": (_I, [_I, _I, _I, _I, _D, _D, _DP]),
            "or_banded_lu": (_I, [_I, _I, _DP]),
            "or_lu_solve": (None, [_I, _I, _DP, _DP]),
            "or_ricker": (_D, [_D, _D, _D]),
            "or_pw_create": (_I, [ctypes.POINTER(_P), _I, _I, _I, _I, _D, _I, _I]),
            "or_pw_destroy": (None, [_P]),
            "or_pw_set_source": (_I, [_P, _DP, _DP, _DP, _I, _D, _D, _D]),
            "or_pw_set_state": (_I, [_P, _DP, _DP]),
            "or_pw_step": (_I, [_P, _I]),
            "or_pw_get_state": (_I, [_P, _DP, _DP, _DP]),
            "or_pw_get_raw": (_I, [_P, _DP, _DP, _DP]),
            "or_pw_energy": (_I, [_P, _DP]),
            "or_pw_kapply": (_I, [_P, _DP, _DP]),
            "or_pw_dapply": (_I, [_P, _DP, _DP]),
            "or_pw_mapply": (_I, [_P, _DP, _DP]),
            "or_pw_dsolve": (_I, [_P, _DP]),
            "or_pw_msolve": (_I, [_P, _DP]),
            "or_pw_msolve_1d": (_I, [_P, _I, _DP]),
            "or_pw_matrix": (_I, [_P, _I, _I, _DP]),
            "or_pw_time": (_D, [_P]),
            "or_el_create": (_I, [ctypes.POINTER(_P), _I, _I, _I, _I, _D, _I, _D, _D, _D]),
            "or_el_destroy": (None, [_P]),
            "or_el_apply": (_I, [_P, _DP, _DP]),
            "or_el_dsolve": (_I, [_P, _DP]),
            "or_el_set_state": (_I, [_P, _DP, _DP]),
            "or_el_step": (_I, [_P, _I]),
            "or_el_get_state": (_I, [_P, _DP, _DP, _DP]),
            "or_el_energy": (_I, [_P, _DP]),
            "or_el_time": (_D, [_P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if ext:
            _lib_ld = L
        else:
            _lib = L
    return _lib_ld if ext else _lib


def _ptr(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    if a.dtype == np.longdouble and np.longdouble != np.float64:
        return a.ctypes.data_as(ctypes.POINTER(ctypes.c_longdouble))
    assert a.dtype == np.float64
    return a.ctypes.data_as(_DP)


class OracleError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise OracleError(f"oracle error {rc}")


# ---------------------------------------------------------------- 1D pieces
def knots(p, nel):
    t = np.zeros(nel + 2 * p + 1)
    lib().or_knots(p, nel, _ptr(t))
    return t


def matrices_1d(p, nel, bc=0):
    """Dense (M, K, B) of the 1D space; nel = 0: the 2D scheme's third
    axis (one function, M = 1, K = B = 0)."""
    n = 1 if nel == 0 else nel + p
    M, K, B = np.zeros((n, n)), np.zeros((n, n)), np.zeros((n, n))
    _check(lib().or_matrices_1d(p, nel, bc, _ptr(M), _ptr(K), _ptr(B)))
    return M, K, B


def load_1d(p, nel, bc, func, ext=False):
    """b_a = int f N_a for a workloads.Func1D descriptor (nel = 0: the 2D scheme's third axis, [1]);
    ext: computed by the extended-precision build (returned as np.longdouble)."""
    dt = np.longdouble if ext else np.float64
    if nel == 0:
        return np.ones(1, dt)
    n = nel + p
    b = np.zeros(n, dt)
    if func[0] == "sin":
        _check(lib(ext).or_load_1d(p, nel, bc, 0, 0.0, 1.0, _ptr(b)))
    elif func[0] == "gauss":
        _check(lib(ext).or_load_1d(p, nel, bc, 1, float(func[1]), float(func[2]), _ptr(b)))
    else:
        raise ValueError(func)
    return b


def banded_lu(A, p):
    LU = np.ascontiguousarray(A, dtype=np.float64).copy()
    _check(lib().or_banded_lu(LU.shape[0], p, _ptr(LU)))
    return LU


def lu_solve(LU, p, b):
    x = np.ascontiguousarray(b, dtype=np.float64).copy()
    lib().or_lu_solve(LU.shape[0], p, _ptr(LU), _ptr(x))
    return x


def ricker(t, f0=25.0, t0=0.04):
    return lib().or_ricker(t, f0, t0)


# ---------------------------------------------------------------- P-wave
class PWave:
    """Oracle P-wave solver; scheme 1 = reading R1 (default), 0 = literal Eq. 16."""

    def __init__(self, nel, p, tau, bc=1, scheme=1, ext=False):
        if isinstance(nel, int):
            nel = (nel, nel, nel)
        self._L, self.dtype = lib(ext), (np.longdouble if ext else np.float64)
        self.nel, self.p, self.tau, self.bc = tuple(nel), p, tau, bc
        self.n = tuple(1 if e == 0 else e + p for e in nel)  # nel_z = 0: the 2D scheme (one z function)
        self.shape = (self.n[2], self.n[1], self.n[0])  # numpy (z, y, x): x fastest
        self.N = int(np.prod(self.n))
        h = _P()
        _check(self._L.or_pw_create(ctypes.byref(h), nel[0], nel[1], nel[2], p, tau, bc, scheme))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self._L.or_pw_destroy(self.h)
            self.h = None

    def _f(self, a):
        return np.ascontiguousarray(np.asarray(a, dtype=self.dtype).reshape(self.shape))

    def set_source(self, b=None, wavelet=1, f0=25.0, t0=0.04, amp=1.0):
        if b is None:
            _check(self._L.or_pw_set_source(self.h, None, None, None, 0, 0.0, 0.0, 0.0))
            return
        bs = [np.ascontiguousarray(x, dtype=self.dtype) for x in b]
        self._src = bs
        _check(self._L.or_pw_set_source(self.h, _ptr(bs[0]), _ptr(bs[1]), _ptr(bs[2]), wavelet, f0, t0, amp))

    def set_state(self, u, udot=None):
        u = self._f(u)
        ud = None if udot is None else self._f(udot)
        _check(self._L.or_pw_set_state(self.h, _ptr(u), _ptr(ud)))

    def step(self, nsteps=1):
        _check(self._L.or_pw_step(self.h, nsteps))

    def get_state(self):
        u, ud, a = (np.zeros(self.shape, self.dtype) for _ in range(3))
        _check(self._L.or_pw_get_state(self.h, _ptr(u), _ptr(ud), _ptr(a)))
        return u, ud, a

    def get_raw(self):
        U, V, a = (np.zeros(self.shape, self.dtype) for _ in range(3))
        _check(self._L.or_pw_get_raw(self.h, _ptr(U), _ptr(V), _ptr(a)))
        return U, V, a

    def energy(self):
        e = np.zeros(3, self.dtype)
        _check(self._L.or_pw_energy(self.h, _ptr(e)))
        return e

    def time(self):
        return self._L.or_pw_time(self.h)

    def _op(self, fn, x):
        x = self._f(x)
        out = np.zeros(self.shape, self.dtype)
        _check(fn(self.h, _ptr(x), _ptr(out)))
        return out

    def kapply(self, x):
        return self._op(self._L.or_pw_kapply, x)

    def dapply(self, x):
        return self._op(self._L.or_pw_dapply, x)

    def mapply(self, x):
        return self._op(self._L.or_pw_mapply, x)

    def dsolve(self, x):
        x = self._f(x).copy()
        _check(self._L.or_pw_dsolve(self.h, _ptr(x)))
        return x

    def msolve(self, x):
        x = self._f(x).copy()
        _check(self._L.or_pw_msolve(self.h, _ptr(x)))
        return x

    def msolve_1d(self, d, x):
        x = np.ascontiguousarray(x, dtype=self.dtype).copy()
        _check(self._L.or_pw_msolve_1d(self.h, d, _ptr(x)))
        return x

    def matrix(self, d, which):
        """which: 0 = M_d, 1 = K_d, 2 = A_d, 3 = LU(A_d) (BC applied)."""
        n = self.n[d]
        out = np.zeros((n, n), self.dtype)
        _check(self._L.or_pw_matrix(self.h, d, which, _ptr(out)))
        return out


# ---------------------------------------------------------------- elasticity
class Elastic:
    """Oracle 3D elasticity solver (delta-form alternating-triangular split E1)."""

    def __init__(self, nel, p, tau, bc=1, lam=1.0, mu=1.0, rho=1.0, ext=False):
        if isinstance(nel, int):
            nel = (nel, nel, nel)
        self._L, self.dtype = lib(ext), (np.longdouble if ext else np.float64)
        self.nel, self.p, self.tau, self.bc = tuple(nel), p, tau, bc
        self.n = tuple(1 if e == 0 else e + p for e in nel)  # nel_z = 0: the 2D (plane-strain) problem
        self.shape = (3, self.n[2], self.n[1], self.n[0])
        self.N = int(np.prod(self.n))
        h = _P()
        _check(self._L.or_el_create(ctypes.byref(h), nel[0], nel[1], nel[2], p, tau, bc, lam, mu, rho))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self._L.or_el_destroy(self.h)
            self.h = None

    def _f(self, a):
        return np.ascontiguousarray(np.asarray(a, dtype=self.dtype).reshape(self.shape))

    def apply(self, x):
        x = self._f(x)
        out = np.zeros(self.shape, self.dtype)
        _check(self._L.or_el_apply(self.h, _ptr(x), _ptr(out)))
        return out

    def dsolve(self, x):
        x = self._f(x).copy()
        _check(self._L.or_el_dsolve(self.h, _ptr(x)))
        return x

    def set_state(self, u, udot=None):
        u = self._f(u)
        ud = None if udot is None else self._f(udot)
        _check(self._L.or_el_set_state(self.h, _ptr(u), _ptr(ud)))

    def step(self, nsteps=1):
        _check(self._L.or_el_step(self.h, nsteps))

    def get_state(self):
        u, ud, a = (np.zeros(self.shape, self.dtype) for _ in range(3))
        _check(self._L.or_el_get_state(self.h, _ptr(u), _ptr(ud), _ptr(a)))
        return u, ud, a

    def energy(self):
        e = np.zeros(3, self.dtype)
        _check(self._L.or_el_energy(self.h, _ptr(e)))
        return e

    def time(self):
        return self._L.or_el_time(self.h)


# ---------------------------------------------------------------- workloads
def project_separable(wl, terms=None):
    """Oracle-side coefficients of a workloads separable sum (L2 projection,
    PAPER.md:620): each 1D factor s_d = M_d^-1 b_d (Dirichlet-restricted)."""
    p, nel, bc = wl.p, wl.nel, wl.bc
    n = wl.n
    ncomp = 3 if wl.elastic else 1
    u = np.zeros((ncomp, n[2], n[1], n[0]))
    pw = PWave(nel, p, wl.tau, bc)
    for t in (wl.u0 if terms is None else terms):
        s = [pw.msolve_1d(d, load_1d(p, nel[d], bc, t.f[d])) for d in range(3)]
        u[t.comp] += t.amp * np.einsum("k,j,i->kji", s[2], s[1], s[0])
    return u if wl.elastic else u[0]


def source_vectors(wl, ext=False):
    if wl.source is None:
        return None
    return [load_1d(wl.p, wl.nel[d], wl.bc, wl.source.f[d], ext) for d in range(3)]


def make_solver(wl, scheme=1, ext=False, u0=None):
    """Oracle solver for a workloads.Workload with its initial state and source set (ext: the
    extended-precision build; u0: start from these coefficients instead of the projection)."""
    u0 = project_separable(wl) if u0 is None else u0
    if wl.elastic:
        s = Elastic(wl.nel, wl.p, wl.tau, wl.bc, wl.lam, wl.mu, wl.rho, ext=ext)
        s.set_state(u0)
        return s
    s = PWave(wl.nel, wl.p, wl.tau, wl.bc, scheme, ext=ext)
    if wl.source is not None:
        src = wl.source
        s.set_source(source_vectors(wl, ext), src.wavelet, src.f0, src.t0, src.amp)
    s.set_state(u0)
    return s


def one_step_truth(wl, u0=None):
    """(u, udot, a) after one step of the extended-precision oracle, as fp64 arrays: the truth
    the GPU's one-step bound is measured against (north_star 1e-12; T1)."""
    s = make_solver(wl, ext=True, u0=u0)
    s.step(1)
    out = tuple(np.asarray(x, dtype=np.float64) for x in s.get_state())
    del s
    return out
