"""Modal (spectral) oracle for the split P-wave scheme.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows the paper's §3 decomposition: for each direction
the generalised eigenproblem K_xi v = lambda M_xi v gives K_xi = M_xi P D P^-1
with P^T M_xi P = I (Eq. 17-18).  The split operator
D = A_x (x) A_y (x) A_z, A_d = M_d + eta K_d, eta = tau^2/4, is then diagonal
in the tensor eigenbasis P3 = P_x (x) P_y (x) P_z with entries
delta = (1 + eta l_i)(1 + eta l_j)(1 + eta l_k) (the E_xi = (I + eta D_xi)^-1
of PAPER.md:173 inverted), and K has entries L = l_i + l_j + l_k.  Hence the
R1 step (DESIGN.md §3 R1; PAPER.md:426 with Upsilon -> K)

    cP = cU + tau cV;  ca = (cF(t_{n+1}) - L cP) / delta;  cV += tau ca;  cU = cP

advances every mode independently.  States map by c = P3^T M U (M-orthonormal
basis); load vectors are dual and map by c_F = P3^T F.  With F = 0 the
recurrence is the 2x2 linear map [[1, tau], [-tau L/delta, 1 - tau^2 L/delta]]
raised to the n-th power (computed by repeated squaring).

Because it never forms K P nor runs the three directional sweeps, this is an
implementation of the step independent of oracle/ads_oracle.c's step logic; it
shares only the oracle's 1D Gram matrices (pinned separately against
closed-form cardinal B-spline rows and scipy-BSpline brute-force quadrature).
Only zero Dirichlet (bc = 1) is supported: the eigenproblem is posed on the
interior-restricted 1D matrices (reading C3).  nel_z = 0 is the 2D scheme as printed
(PAPER.md:123-143): the third axis has one function, M = 1, K = 0, no boundary.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from . import matrices_1d, ricker


class ModalPWave:
    def __init__(self, nel, p, tau):
        if isinstance(nel, int):
            nel = (nel, nel, nel)
        self.nel, self.p, self.tau = tuple(nel), p, tau
        self.n = tuple(1 if e == 0 else e + p for e in nel)
        self.eta = tau * tau / 4.0
        self.P, self.lam, self.Q = [], [], []
        # active DOFs per direction: interior (Dirichlet) or the single function of the 2D axis
        self.sl = tuple(slice(None) if e == 0 else slice(1, -1) for e in nel)
        for d in range(3):
            M, K, _ = matrices_1d(p, nel[d], bc=1)
            Mi, Ki = M[self.sl[d], self.sl[d]], K[self.sl[d], self.sl[d]]
            lam, P = scipy.linalg.eigh(Ki, Mi)   # P^T Mi P = I, Ki P = Mi P diag(lam)
            self.P.append(P)
            self.lam.append(lam)
            self.Q.append(P.T @ Mi)              # c = Q u   (M-orthonormal coordinates)
        lx, ly, lz = self.lam
        self.L = lz[:, None, None] + ly[None, :, None] + lx[None, None, :]
        e = self.eta
        self.delta = (1 + e * lz)[:, None, None] * (1 + e * ly)[None, :, None] * (1 + e * lx)[None, None, :]

    # ---- transforms on interior arrays (z, y, x) ----
    @staticmethod
    def _modes(T, Ax, Ay, Az):
        T = np.tensordot(T, Ax.T, axes=([2], [0]))          # x
        T = np.tensordot(T, Ay.T, axes=([1], [0])).transpose(0, 2, 1)
        T = np.tensordot(Az, T, axes=([1], [0]))
        return np.ascontiguousarray(T)

    def to_modal(self, u):
        """c = P3^T M u for a full (nz, ny, nx) coefficient array (boundary ignored)."""
        ui = np.asarray(u)[self.sl[2], self.sl[1], self.sl[0]]
        return self._modes(ui, self.Q[0], self.Q[1], self.Q[2])

    def from_modal(self, c):
        ui = self._modes(c, self.P[0], self.P[1], self.P[2])
        u = np.zeros((self.n[2], self.n[1], self.n[0]))
        u[self.sl[2], self.sl[1], self.sl[0]] = ui
        return u

    def run(self, u0, udot0=None, nsteps=0, source=None, wavelet=1, f0=25.0, t0=0.04, amp=1.0):
        """Evolve (u0, udot0) by nsteps R1 steps with the half-kick start.

        source: None or the three 1D load vectors b_d (F(t) = amp g(t) b_x(x)b_y(x)b_z).
        Returns (U_n, udot_n, a_n) as full arrays."""
        tau = self.tau
        cU = self.to_modal(u0)
        cV = np.zeros_like(cU) if udot0 is None else self.to_modal(udot0)
        if source is not None:
            fs = [self.P[d].T @ np.asarray(source[d])[self.sl[d]] for d in range(3)]
            cFs = fs[2][:, None, None] * fs[1][None, :, None] * fs[0][None, None, :]

            def g(t):
                return amp * (ricker(t, f0, t0) if wavelet == 1 else 1.0)
        else:
            cFs = None
        Ld = self.L / self.delta

        def accel(cP, t):
            if cFs is None:
                return -Ld * cP
            return (g(t) * cFs - self.L * cP) / self.delta

        ca = accel(cU, 0.0)
        cV = cV + 0.5 * tau * ca
        if cFs is None and nsteps > 0:
            # [cU; cV] <- A^n [cU; cV], A = [[1, tau], [-tau Ld, 1 - tau^2 Ld]]
            a11 = np.ones_like(Ld); a12 = np.full_like(Ld, tau)
            a21 = -tau * Ld; a22 = 1.0 - tau * tau * Ld
            r11 = np.ones_like(Ld); r12 = np.zeros_like(Ld); r21 = np.zeros_like(Ld); r22 = np.ones_like(Ld)
            k = nsteps
            while k:
                if k & 1:
                    r11, r12, r21, r22 = (r11 * a11 + r12 * a21, r11 * a12 + r12 * a22,
                                          r21 * a11 + r22 * a21, r21 * a12 + r22 * a22)
                k >>= 1
                if k:
                    a11, a12, a21, a22 = (a11 * a11 + a12 * a21, a11 * a12 + a12 * a22,
                                          a21 * a11 + a22 * a21, a21 * a12 + a22 * a22)
            # the last kick's a_n = (V_n - V_{n-1})/tau; recompute from state n-1 -> n
            cU, cV = r11 * cU + r12 * cV, r21 * cU + r22 * cV
            ca = -Ld * cU  # a_n = -Ld U_n   (U_n = P of the last step)
        else:
            for s in range(nsteps):
                cP = cU + tau * cV
                ca = accel(cP, (s + 1) * tau)
                cV = cV + tau * ca
                cU = cP
        udot = cV - 0.5 * tau * ca
        return self.from_modal(cU), self.from_modal(udot), self.from_modal(ca)

    def exact_semidiscrete(self, u0, t):
        """Semi-discrete exact solution (no time error): c(t) = cos(sqrt(L) t) c(0), udot0 = 0, F = 0."""
        c0 = self.to_modal(u0)
        return self.from_modal(np.cos(np.sqrt(self.L) * t) * c0)
