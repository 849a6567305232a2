"""Independent reference computations used to PIN the oracle.

Nothing here imports oracle/ or the product package.  Everything is built from
library routines (scipy.interpolate.BSpline for basis functions,
numpy.polynomial.legendre.leggauss for quadrature, numpy dense linear algebra)
or from closed forms (truncated-power cardinal B-splines).
"""
from __future__ import annotations

from math import comb, factorial

import numpy as np
from scipy.interpolate import BSpline


def open_knots(p, nel):
    return np.concatenate([np.zeros(p), np.linspace(0.0, 1.0, nel + 1), np.ones(p)])


def basis_tables(p, nel, nq):
    """Quadrature points/weights over [0,1] and basis values/derivatives there (scipy BSpline)."""
    t = open_knots(p, nel)
    n = nel + p
    xg, wg = np.polynomial.legendre.leggauss(nq)
    xs, ws = [], []
    for e in range(nel):
        a, b = e / nel, (e + 1) / nel
        xs.append(0.5 * (a + b) + 0.5 * (b - a) * xg)
        ws.append(0.5 * (b - a) * wg)
    x = np.concatenate(xs)
    w = np.concatenate(ws)
    spl = BSpline(t, np.eye(n), p, extrapolate=False)
    N = np.nan_to_num(spl(x))                 # (nq_total, n)
    dN = np.nan_to_num(spl.derivative()(x))
    return x, w, N, dN


def gram_1d(p, nel):
    """(M, K, B) by scipy-BSpline brute force with p+3 Gauss points per element."""
    x, w, N, dN = basis_tables(p, nel, p + 3)
    M = (N * w[:, None]).T @ N
    K = (dN * w[:, None]).T @ dN
    B = (dN * w[:, None]).T @ N      # B(a,c) = int N'_a N_c
    return M, K, B


def restrict(Mat):
    """Zero-Dirichlet interior restriction padded with zero rows/cols."""
    R = Mat.copy()
    R[0, :] = R[-1, :] = 0.0
    R[:, 0] = R[:, -1] = 0.0
    return R


def cardinal(m, x, deriv=0):
    """Cardinal B-spline of order m (support [0, m]) by the truncated-power formula
    B_m(x) = 1/(m-1)! sum_k (-1)^k C(m,k) (x-k)_+^(m-1), and its derivatives."""
    deg = m - 1 - deriv
    s = 0.0
    for k in range(m + 1):
        z = x - k
        if z > 0:
            s += (-1) ** k * comb(m, k) * z ** deg
    return s / factorial(deg)


def kron3(Ax, Ay, Az):
    """Dense matrix of Ax (x) Ay (x) Az acting on x-fastest vectorised arrays."""
    return np.kron(Az, np.kron(Ay, Ax))


def brute_force_stiffness_3d(p, nel):
    """K3D(a, c) = int_cube grad phi_a . grad phi_c by tensor Gauss quadrature of the
    3D basis functions themselves (no Kronecker factorisation used)."""
    x, w, N, dN = basis_tables(p, nel, p + 2)
    n = nel + p
    # all 3D points: (z, y, x) ordering with x fastest
    W = np.einsum("k,j,i->kji", w, w, w).ravel()
    nq = len(x)
    # basis phi_(a=(ax,ay,az)) evaluated at point (qz,qy,qx), index a = (az*n + ay)*n + ax
    Phi = np.einsum("kc,jb,ia->kjicba", N, N, N).reshape(nq ** 3, n ** 3)
    Gx = np.einsum("kc,jb,ia->kjicba", N, N, dN).reshape(nq ** 3, n ** 3)
    Gy = np.einsum("kc,jb,ia->kjicba", N, dN, N).reshape(nq ** 3, n ** 3)
    Gz = np.einsum("kc,jb,ia->kjicba", dN, N, N).reshape(nq ** 3, n ** 3)
    K = sum((G * W[:, None]).T @ G for G in (Gx, Gy, Gz))
    M = (Phi * W[:, None]).T @ Phi
    return M, K, (Gx, Gy, Gz, W)


def brute_force_elastic_3d(p, nel, lam, mu):
    """Dense elasticity stiffness from the weak form:
    a(w,u) = int 2 mu eps(w):eps(u) + lam div w div u, vector basis phi_a e_i,
    assembled directly from strains at quadrature points.  Component-major."""
    M, _, (Gx, Gy, Gz, W) = brute_force_stiffness_3d(p, nel)
    G = (Gx, Gy, Gz)
    nd = Gx.shape[1]
    A = np.zeros((3 * nd, 3 * nd))
    for i in range(3):          # test component
        for k in range(3):      # trial component
            # eps(phi e_i)_{ab} = 1/2 (d_b phi delta_ai + d_a phi delta_bi)
            # 2 mu eps(w):eps(u) = mu sum_ab (d_b w_a d_b u_a + d_b w_a d_a u_b)
            blk = np.zeros((nd, nd))
            if i == k:
                for b in range(3):
                    blk += mu * (G[b] * W[:, None]).T @ G[b]
            blk += mu * (G[k] * W[:, None]).T @ G[i]     # d_b w_a d_a u_b with a=i, b=k
            blk += lam * (G[i] * W[:, None]).T @ G[k]    # div w div u
            A[i * nd:(i + 1) * nd, k * nd:(k + 1) * nd] = blk
    return M, A


def dirichlet_mask_3d(n):
    m = np.ones((n, n, n), dtype=bool)
    m[0, :, :] = m[-1, :, :] = m[:, 0, :] = m[:, -1, :] = m[:, :, 0] = m[:, :, -1] = False
    return m.ravel()


def rel_l2(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def brute_force_elastic_2d(p, nel, lam, mu):
    """Dense plane-strain elasticity stiffness (PAPER.md:307-361 in 2D; the blocks PAPER.md:362-387)
    from strains at quadrature points: a(w,u) = int 2 mu eps(w):eps(u) + lam div w div u over the
    unit square, vector basis phi_a e_i (i in {x, y}); plus the 2D mass and the scalar stiffness.
    Component-major, x fastest."""
    x, w, N, dN = basis_tables(p, nel, p + 2)
    n = nel + p
    W = np.einsum("j,i->ji", w, w).ravel()
    nq = len(x)
    Phi = np.einsum("jb,ia->jiba", N, N).reshape(nq ** 2, n ** 2)
    Gx = np.einsum("jb,ia->jiba", N, dN).reshape(nq ** 2, n ** 2)
    Gy = np.einsum("jb,ia->jiba", dN, N).reshape(nq ** 2, n ** 2)
    G = (Gx, Gy)
    nd = n * n
    A = np.zeros((2 * nd, 2 * nd))
    for i in range(2):
        for k in range(2):
            blk = np.zeros((nd, nd))
            if i == k:
                for b in range(2):
                    blk += mu * (G[b] * W[:, None]).T @ G[b]
            blk += mu * (G[k] * W[:, None]).T @ G[i]
            blk += lam * (G[i] * W[:, None]).T @ G[k]
            A[i * nd:(i + 1) * nd, k * nd:(k + 1) * nd] = blk
    M = (Phi * W[:, None]).T @ Phi
    K = sum((g * W[:, None]).T @ g for g in G)
    return M, K, A
