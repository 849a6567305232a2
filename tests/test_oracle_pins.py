"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names what it pins and what plausible oracle mistake it would catch.
References: PAPER.md lines (the paper), SPEC.md lines (test ideas), SURVEY.md §8(c).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.modal import ModalPWave
import workloads
from pins_util import (brute_force_elastic_3d, brute_force_stiffness_3d, cardinal, gram_1d, kron3,
                       rel_l2, restrict, dirichlet_mask_3d)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- 1D assembly
def test_spec_p1_fixtures():
    """SPEC.md:102/111/120/179/265/336 exact p=1 one-element matrices (hand integrals)."""
    g = _gold("spec_p1_fixtures.json")
    M, K, B = oracle.matrices_1d(1, 1, bc=0)
    np.testing.assert_allclose(M, g["M"], atol=1e-15)
    np.testing.assert_allclose(K, g["K"], atol=1e-15)
    np.testing.assert_allclose(B, g["B"], atol=1e-15)   # catches a transposed B (test vs trial derivative)
    LU = oracle.banded_lu(M, 1)
    assert abs(LU[1, 1] - g["LU_U22"]) < 1e-15
    pw = oracle.PWave((1, 1, 1), 1, 2.0, bc=0)            # tau = 2 -> eta = 1
    np.testing.assert_allclose(pw.matrix(0, 2), g["A_tau2"], atol=1e-15)
    ev = np.sort(np.real(np.linalg.eigvals(np.linalg.solve(M, K))))
    np.testing.assert_allclose(ev, g["pencil_eigenvalues"], atol=1e-12)


@pytest.mark.parametrize("p", [2, 3])
def test_cardinal_interior_rows(p):
    """Interior rows equal cardinal B-spline values (closed form, truncated powers)
    and the golden integer fixtures: catches wrong knots, Gauss rule or basis recursion."""
    nel = 16
    h = 1.0 / nel
    M, K, _ = oracle.matrices_1d(p, nel, bc=0)
    g = _gold("cardinal_rows.json")[f"p{p}"]
    m = 2 * p + 2
    row = nel // 2
    for k in range(-p, p + 1):
        mc = h * cardinal(m, p + 1 + k)
        kc = -cardinal(m, p + 1 + k, deriv=2) / h
        assert abs(M[row, row + k] - mc) < 1e-15
        assert abs(K[row, row + k] - kc) < 1e-12
    scale = 120 if p == 2 else 5040
    kscale = 6 if p == 2 else 120
    np.testing.assert_allclose(M[row, row - p:row + p + 1] * scale / h, g[list(g)[0]], atol=1e-11)
    np.testing.assert_allclose(K[row, row - p:row + p + 1] * kscale * h, g[list(g)[1]], atol=1e-11)


@pytest.mark.parametrize("p,nel", [(1, 1), (1, 3), (2, 1), (2, 5), (3, 4), (3, 9), (4, 6)])
def test_gram_vs_scipy_bspline(p, nel):
    """Boundary and interior rows vs an independent scipy.interpolate.BSpline assembly."""
    M, K, B = oracle.matrices_1d(p, nel, bc=0)
    Mr, Kr, Br = gram_1d(p, nel)
    np.testing.assert_allclose(M, Mr, atol=1e-14)
    np.testing.assert_allclose(K, Kr, atol=1e-11 * max(1, nel ** 2))
    np.testing.assert_allclose(B, Br, atol=1e-13 * nel)
    # banded structure M_ij = 0 <=> |i-j| > p
    n = nel + p
    i, j = np.indices((n, n))
    assert np.all(M[np.abs(i - j) > p] == 0.0)
    assert np.all(M[np.abs(i - j) <= p] > 0.0)


@pytest.mark.parametrize("p,nel", [(2, 7), (3, 5)])
def test_gram_invariants(p, nel):
    """Partition of unity (sum M = 1), K 1 = 0, B + B^T = boundary terms."""
    M, K, B = oracle.matrices_1d(p, nel, bc=0)
    assert abs(M.sum() - 1.0) < 1e-14
    assert np.abs(K @ np.ones(nel + p)).max() < 1e-11
    S = B + B.T
    E = np.zeros_like(S)
    E[-1, -1] = 1.0
    E[0, 0] = -1.0                        # N_a(1)N_c(1) - N_a(0)N_c(0)
    np.testing.assert_allclose(S, E, atol=1e-12)
    np.testing.assert_allclose(M, M.T, atol=0)
    np.testing.assert_allclose(K, K.T, atol=0)


def test_dirichlet_pencil_first_eigenvalue():
    """lambda_1 of the restricted pencil -> pi^2 (SURVEY §8(c) basis pins: 8.3e-13 at c2)."""
    for p, nel, tol in [(2, 16, 3e-6), (3, 64, 1e-11)]:
        M, K, _ = oracle.matrices_1d(p, nel, bc=1)
        ev = np.sort(np.real(np.linalg.eigvals(np.linalg.solve(M[1:-1, 1:-1], K[1:-1, 1:-1]))))
        assert abs(ev[0] / math.pi ** 2 - 1) < tol


# ----------------------------------------------------------------- LU / sweeps
def test_banded_lu_vs_dense_solve():
    rng = np.random.default_rng(0)
    for p, nel in [(2, 9), (3, 12)]:
        M, K, _ = oracle.matrices_1d(p, nel, bc=0)
        A = M + 0.37 * K
        LU = oracle.banded_lu(A, p)
        b = rng.standard_normal(nel + p)
        np.testing.assert_allclose(oracle.lu_solve(LU, p, b), np.linalg.solve(A, b), rtol=1e-12, atol=1e-12)
    # pure stiffness (constant kernel) must be reported singular
    _, K, _ = oracle.matrices_1d(1, 4, bc=0)
    with pytest.raises(oracle.OracleError):
        oracle.banded_lu(K, 1)


def test_diag_kron_solve_fixture():
    """(2I)(x)(3I) b = ones -> 1/6; exercised through dense LU solves per axis."""
    g = _gold("spec_p1_fixtures.json")
    LU2 = oracle.banded_lu(2 * np.eye(4), 1)
    LU3 = oracle.banded_lu(3 * np.eye(4), 1)
    x = oracle.lu_solve(LU3, 1, oracle.lu_solve(LU2, 1, np.ones(4)))
    np.testing.assert_allclose(x, g["diag_kron_solve"], rtol=1e-15)


@pytest.mark.parametrize("bc", [0, 1])
def test_dsolve_dapply_vs_dense_kron(bc):
    """D^-1 by three sweeps == dense solve of A_x(x)A_y(x)A_z built
    from the independent scipy assembly; anisotropic grid catches swapped axes."""
    nel, p, tau = (3, 4, 2), 2, 0.3
    pw = oracle.PWave(nel, p, tau, bc=bc)
    eta = tau * tau / 4
    A = []
    for d in range(3):
        M, K, _ = gram_1d(p, nel[d])
        Ad = M + eta * K
        if bc == 1:
            Ad = restrict(Ad)
            Ad[0, 0] = Ad[-1, -1] = 1.0
        A.append(Ad)
    D = kron3(*A)
    r = workloads.random_field(11, pw.N)
    x = pw.dsolve(r)
    np.testing.assert_allclose(x.ravel(), np.linalg.solve(D, r), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(pw.dapply(r).ravel(), D @ r, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("p,nel", [(2, 2), (2, 3), (3, 2)])
def test_kapply_vs_bruteforce_3d_quadrature(p, nel):
    """K P == brute-force 3D stiffness int grad phi_a . grad phi_c (no Kronecker algebra),
    natural BC; and the Dirichlet restriction of it."""
    _, K3, _ = brute_force_stiffness_3d(p, nel)
    pw = oracle.PWave(nel, p, 0.1, bc=0)
    x = workloads.random_field(5, pw.N)
    np.testing.assert_allclose(pw.kapply(x).ravel(), K3 @ x, rtol=1e-12, atol=1e-12)
    pwd = oracle.PWave(nel, p, 0.1, bc=1)
    m = dirichlet_mask_3d(nel + p)
    Kd = K3 * m[:, None] * m[None, :]
    np.testing.assert_allclose(pwd.kapply(x).ravel(), Kd @ x, rtol=1e-12, atol=1e-12)


def test_kapply_discrete_eigenvector():
    """K (phi(x)phi(x)phi) = 3 lambda M (phi(x)phi(x)phi) for a 1D discrete eigenvector."""
    p, nel = 3, 6
    pw = oracle.PWave(nel, p, 0.1, bc=1)
    M = pw.matrix(0, 0)[1:-1, 1:-1]
    K = pw.matrix(0, 1)[1:-1, 1:-1]
    lam, V = np.linalg.eig(np.linalg.solve(M, K))
    k = int(np.argmin(np.real(lam)))
    phi = np.zeros(nel + p)
    phi[1:-1] = np.real(V[:, k])
    u = np.einsum("k,j,i->kji", phi, phi, phi)
    np.testing.assert_allclose(pw.kapply(u), 3 * np.real(lam[k]) * pw.mapply(u), rtol=1e-10, atol=1e-13)


def test_splitting_defect_order_tau4():
    """D - (M + eta K) = eta^2(...) + eta^3 K(x)K(x)K: defect ratio 16 per tau halving
    (Eq. 15, 'dropping' the tau^4/16 term).  Catches eta != tau^2/4."""
    p, nel = 2, 3
    ratios = []
    prev = None
    for tau in [0.05, 0.025, 0.0125]:
        pw = oracle.PWave(nel, p, tau, bc=0)
        Ms = [pw.matrix(d, 0) for d in range(3)]
        Ks = [pw.matrix(d, 1) for d in range(3)]
        As = [pw.matrix(d, 2) for d in range(3)]
        eta = tau * tau / 4
        Mf = kron3(*Ms)
        Kf = kron3(Ks[0], Ms[1], Ms[2]) + kron3(Ms[0], Ks[1], Ms[2]) + kron3(Ms[0], Ms[1], Ks[2])
        defect = np.linalg.norm(kron3(*As) - (Mf + eta * Kf)) / np.linalg.norm(Mf)
        if prev is not None:
            ratios.append(prev / defect)
        prev = defect
    assert all(abs(r - 16) < 0.25 for r in ratios), ratios


# ----------------------------------------------------------------- whole step
def _one_step_dense(nel, p, tau, u0, F=None):
    """One R1 step by dense linear algebra on the independent scipy matrices."""
    eta = tau * tau / 4
    Ms, Ks, As = [], [], []
    for d in range(3):
        M, K, _ = gram_1d(p, nel[d])
        M, K = restrict(M), restrict(K)
        A = M + eta * K
        A[0, 0] = A[-1, -1] = 1.0
        Ms.append(M); Ks.append(K); As.append(A)
    D = kron3(*As)
    Kf = kron3(Ks[0], Ms[1], Ms[2]) + kron3(Ms[0], Ks[1], Ms[2]) + kron3(Ms[0], Ms[1], Ks[2])
    F = np.zeros_like(u0) if F is None else F
    a0 = np.linalg.solve(D, F - Kf @ u0)
    V = 0.5 * tau * a0                     # half-kick, udot0 = 0
    P = u0 + tau * V
    a1 = np.linalg.solve(D, F - Kf @ P)
    return P, V + tau * a1, a1


def test_one_step_vs_dense():
    nel, p, tau = (3, 2, 4), 2, 0.07
    pw = oracle.PWave(nel, p, tau, bc=1)
    u0 = workloads.random_field(3, pw.N).reshape(pw.shape)
    m = np.zeros(pw.shape, bool)
    m[1:-1, 1:-1, 1:-1] = True
    u0 = np.where(m, u0, 0.0)
    pw.set_state(u0)
    pw.step(1)
    U, V, a = pw.get_raw()
    Ud, Vd, ad = _one_step_dense(nel, p, tau, u0.ravel())
    assert rel_l2(U, Ud) < 1e-13 and rel_l2(V, Vd) < 1e-13 and rel_l2(a, ad) < 1e-13


@pytest.mark.parametrize("cfg,nsteps", [("c1", 20), ("c2", 10)])
def test_modal_closed_form_matches_stepping(cfg, nsteps):
    """Mode-by-mode exact evolution == oracle stepping (~1e-13)."""
    wl = workloads.get(cfg)
    if cfg == "c2":
        wl = wl.scaled(16, nsteps)
    s = oracle.make_solver(wl)
    u0 = oracle.project_separable(wl)
    s.step(nsteps)
    u, ud, a = s.get_state()
    mu, mud, ma = ModalPWave(wl.nel, wl.p, wl.tau).run(u0, nsteps=nsteps)
    assert rel_l2(u, mu) < 1e-13
    assert rel_l2(ud, mud) < 1e-12
    assert rel_l2(a, ma) < 1e-12


def test_modal_forced_matches_stepping():
    """Forced (Ricker x Gaussian, c3 recipe on a 12^3 mesh): dual load vectors map by P^T."""
    wl = workloads.get("c3").scaled(12, 60)
    s = oracle.make_solver(wl)
    s.step(60)
    u, ud, a = s.get_state()
    src = wl.source
    mu, mud, ma = ModalPWave(wl.nel, wl.p, wl.tau).run(np.zeros(s.shape), nsteps=60,
                                                        source=oracle.source_vectors(wl),
                                                        wavelet=src.wavelet, f0=src.f0, t0=src.t0)
    assert np.linalg.norm(u) > 0
    assert rel_l2(u, mu) < 1e-12 and rel_l2(ud, mud) < 1e-12 and rel_l2(a, ma) < 1e-12


def test_c1_standing_mode_accuracy_and_literal_garble():
    """c1 vs the PDE closed form cos(sqrt(3) pi t) sin sin sin (BASELINE config 1).
    R1 error 2.2e-4-ish at t = 0.2 (accept <= 3e-4); the literal Eq. 16 (R0) is
    inconsistent (wave speed 1/sqrt 2) and misses by > 10% (SURVEY §0 finding 1)."""
    wl = workloads.get("c1")
    u0 = oracle.project_separable(wl)
    errs = {}
    for scheme in (1, 0):
        s = oracle.make_solver(wl, scheme=scheme)
        s.step(wl.steps)
        u, _, _ = s.get_state()
        t = s.time()
        ex = math.cos(math.sqrt(3) * math.pi * t) * u0
        d = u - ex
        errs[scheme] = math.sqrt(np.sum(d * s.mapply(d)) / np.sum(u0 * s.mapply(u0)))
    assert errs[1] < 3e-4, errs
    assert errs[0] > 0.1, errs


def test_second_order_in_time():
    """PAPER.md:256 'second order in time': tau-halving vs the semi-discrete exact solution."""
    nel, p = 8, 2
    wl = workloads.get("c1").scaled(nel)
    u0 = oracle.project_separable(wl)
    T = 1.0
    errs = []
    for tau in [0.02, 0.01, 0.005, 0.0025]:
        s = oracle.PWave(nel, p, tau, bc=1)
        s.set_state(u0)
        s.step(int(round(T / tau)))
        u, _, _ = s.get_state()
        ex = ModalPWave(nel, p, tau).exact_semidiscrete(u0, T)
        errs.append(np.linalg.norm(u - ex))
    ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
    assert all(3.8 < r < 4.2 for r in ratios), ratios


@pytest.mark.parametrize("tau", [0.05, 1.0, 10.0, 1000.0])
def test_energy_invariant_unconditional(tau):
    """Exact discrete invariant 1/2 V'DV + 1/2 U_n'K U_{n+1} (PAPER.md:440-443 energy identity
    with Upsilon -> K) conserved for any tau: unconditional stability pin."""
    wl = workloads.get("c2").scaled(6)
    s = oracle.PWave(6, 3, tau, bc=1)
    u0 = oracle.project_separable(wl) + 0.1 * np.where(dirichlet_mask_3d(9).reshape(9, 9, 9),
                                                       workloads.random_field(2, 729).reshape(9, 9, 9), 0)
    s.set_state(u0)
    e0 = s.energy()
    for _ in range(4):
        s.step(50)
        e = s.energy()
        assert abs(e[2] - e0[2]) <= 1e-13 * abs(e0[2])


def test_work_identity_forced():
    """E_{n+3/2} - E_{n+1/2} = 1/2 F_{n+1}'(U_{n+2} - U_n) (multiply the three-level form by
    U_{n+2} - U_n): pins the time level of the source and the invariant together."""
    wl = workloads.get("c3").scaled(8, 0)
    s = oracle.make_solver(wl)
    b = oracle.source_vectors(wl)
    Fs = np.einsum("k,j,i->kji", b[2], b[1], b[0])
    tau = wl.tau
    s.step(35)
    U_n, _, _ = s.get_raw()
    E_a = s.energy()[2]
    s.step(1)
    U_n1, V_n1, _ = s.get_raw()
    E_b = s.energy()[2]
    g = oracle.ricker(36 * tau)
    U_n2 = U_n1 + tau * V_n1
    work = 0.5 * g * np.sum(Fs * (U_n2 - U_n))
    assert abs(work) > 1e-12
    assert abs((E_b - E_a) - work) <= 1e-12 * abs(work) + 1e-17


def test_set_get_roundtrip():
    """Half-kick start: get_state right after set_state returns udot0 exactly (to rounding)."""
    pw = oracle.PWave(5, 2, 0.05, bc=1)
    u0 = np.where(dirichlet_mask_3d(7).reshape(7, 7, 7), workloads.random_field(8, 343).reshape(7, 7, 7), 0)
    v0 = np.where(dirichlet_mask_3d(7).reshape(7, 7, 7), workloads.random_field(9, 343).reshape(7, 7, 7), 0)
    pw.set_state(u0, v0)
    u, ud, _ = pw.get_state()
    assert rel_l2(u, u0) == 0.0
    assert rel_l2(ud, v0) < 1e-15


# ----------------------------------------------------------------- elasticity
def test_elastic_operator_vs_bruteforce():
    """Upsilon blocks (C10/C11) == dense weak-form elasticity stiffness from strains at quadrature
    points (natural BC, lam != mu to separate the two coefficients)."""
    p, nel, lam, mu = 2, 2, 1.7, 0.6
    _, A = brute_force_elastic_3d(p, nel, lam, mu)
    el = oracle.Elastic(nel, p, 0.1, bc=0, lam=lam, mu=mu)
    x = workloads.random_field(21, 3 * el.N)
    np.testing.assert_allclose(el.apply(x).ravel(), A @ x, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(A, A.T, atol=1e-13)


def test_elastic_rigid_body_kernel():
    """Natural BC: the 6 rigid motions are in the kernel of Upsilon (PAPER.md:297 traction-free)."""
    p, nel = 2, 3
    el = oracle.Elastic(nel, p, 0.1, bc=0, lam=1.3, mu=0.7)
    n = nel + p
    # Greville abscissae reproduce linear functions exactly
    t = oracle.knots(p, nel)
    g = np.array([t[a + 1:a + p + 1].mean() for a in range(n)])
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    one, zero = np.ones_like(X), np.zeros_like(X)
    modes = [(one, zero, zero), (zero, one, zero), (zero, zero, one),
             (-Y, X, zero), (zero, -Z, Y), (Z, zero, -X)]
    for m in modes:
        u = np.stack(m)
        assert np.abs(el.apply(u)).max() < 1e-12 * max(1.0, np.abs(u).max()) * n * n


def test_elastic_dsolve_vs_dense():
    """Delta-form predictor/corrector == dense solve with D~ = L~ (rho M)^-1 L~^T, where
    L~ has S_i = rho (x)(M_d + c_{i,d}K_d) on the diagonal and tau^2/2 Ups_ij below."""
    p, nel, tau, lam, mu, rho = 2, 2, 0.2, 1.4, 0.8, 1.3
    el = oracle.Elastic(nel, p, tau, bc=0, lam=lam, mu=mu, rho=rho)
    M3, A = brute_force_elastic_3d(p, nel, lam, mu)
    nd = M3.shape[0]
    Ms, Ks = [], []
    for d in range(3):
        M, K, _ = gram_1d(p, nel)
        Ms.append(M); Ks.append(K)
    L = np.zeros((3 * nd, 3 * nd))
    for i in range(3):
        cs = [tau * tau / (4 * rho) * ((2 * mu + lam) if d == i else mu) for d in range(3)]
        S = rho * kron3(*[Ms[d] + cs[d] * Ks[d] for d in range(3)])
        L[i * nd:(i + 1) * nd, i * nd:(i + 1) * nd] = S
        for j in range(i):
            L[i * nd:(i + 1) * nd, j * nd:(j + 1) * nd] = 0.5 * tau * tau * A[i * nd:(i + 1) * nd, j * nd:(j + 1) * nd]
    RM = np.kron(np.eye(3), rho * M3)
    Dt = L @ np.linalg.solve(RM, L.T)
    r = workloads.random_field(31, 3 * nd)
    np.testing.assert_allclose(el.dsolve(r).ravel(), np.linalg.solve(Dt, r), rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("tau", [0.01, 0.5, 10.0])
def test_elastic_invariant(tau):
    """E1 conserves 1/2 V'D~V + 1/2 U_n' Ups U_{n+1} (Theorem PAPER.md:435-465, sigma = 1/2)."""
    wl = workloads.get("c5").scaled(4)
    el = oracle.Elastic(4, 2, tau, bc=1)
    el.set_state(oracle.project_separable(wl))
    e0 = el.energy()
    assert e0[2] > 0
    el.step(30)
    e = el.energy()
    assert abs(e[2] - e0[2]) <= 1e-12 * e0[2]


def test_elastic_second_order():
    """PAPER.md:483 second order: tau-halving vs the semi-discrete exact solution of
    rho M u'' + Ups u = 0 (dense generalised eigensolve, tiny Dirichlet grid)."""
    import scipy.linalg
    p, nel, lam, mu, rho = 2, 3, 1.0, 1.0, 1.0
    wl = workloads.get("c5").scaled(nel)
    u0 = oracle.project_separable(wl)
    M3, A = brute_force_elastic_3d(p, nel, lam, mu)
    m = np.tile(dirichlet_mask_3d(nel + p), 3)
    RM = np.kron(np.eye(3), rho * M3)[np.ix_(m, m)]
    Ai = A[np.ix_(m, m)]
    lamv, Q = scipy.linalg.eigh(Ai, RM)
    T = 0.5
    c0 = Q.T @ RM @ u0.ravel()[m]
    ex = np.zeros(u0.size)
    ex[m] = Q @ (np.cos(np.sqrt(lamv) * T) * c0)
    errs = []
    for tau in [0.02, 0.01, 0.005]:
        el = oracle.Elastic(nel, p, tau, bc=1, lam=lam, mu=mu, rho=rho)
        el.set_state(u0)
        el.step(int(round(T / tau)))
        u, _, _ = el.get_state()
        errs.append(np.linalg.norm(u.ravel() - ex))
    ratios = [errs[0] / errs[1], errs[1] / errs[2]]
    assert all(3.7 < r < 4.3 for r in ratios), ratios


# ---- the 2D scheme as printed: nel_z = 0 (row f2) ----

def _wl2d(nel, p, tau, steps, source=None):
    sin = ("sin",)
    return workloads.Workload(name="2d", p=p, nel=nel, tau=tau, steps=steps, source=source,
                              u0=[] if source else [workloads.SeparableTerm(1.0, 0, (sin, sin, sin))])


def test_2d_equals_z_constant_3d_natural_bc():
    """With natural BC the constant is in the kernel of K_z and A_z 1 = M_z 1, so a 3D state that
    is constant in z evolves exactly as the 2D scheme (x) 1: K(u2 (x) 1) = (K2D u2) (x) M_z 1 and
    D^-1 (v (x) M_z 1) = (D2D^-1 v) (x) 1.  Pins the 2D path on the (separately pinned) 3D one."""
    p, tau, steps = 2, 1e-2, 12
    o2 = oracle.PWave((9, 7, 0), p, tau, bc=0)
    o3 = oracle.PWave((9, 7, 5), p, tau, bc=0)
    rng = np.random.default_rng(3)
    u2, v2 = rng.standard_normal(o2.shape), rng.standard_normal(o2.shape)
    o2.set_state(u2, v2)
    o3.set_state(np.repeat(u2, o3.shape[0], axis=0), np.repeat(v2, o3.shape[0], axis=0))
    o2.step(steps)
    o3.step(steps)
    for a2, a3 in zip(o2.get_state(), o3.get_state()):
        for k in range(o3.shape[0]):
            assert np.abs(a3[k] - a2[0]).max() <= 1e-12 * np.abs(a2).max()


def test_2d_standing_mode_closed_form():
    """u0 = L2 projection of sin(pi x) sin(pi y), zero Dirichlet, udot0 = 0: the PDE solution is
    cos(sqrt(2) pi t) u0; the discrete solution after 20 steps (tau = 0.01, p = 2, 16^2 elements)
    must match it to the spatial/temporal discretisation error (~1e-4, like c1's 2.19e-4 in 3D).
    A dropped or doubled stiffness term (wrong wave speed) misses by > 1e-2."""
    wl = _wl2d((16, 16, 0), 2, 1e-2, 20)
    o = oracle.make_solver(wl)
    u0 = o.get_state()[0].copy()
    o.step(wl.steps)
    u = o.get_state()[0]
    exact = math.cos(math.sqrt(2.0) * math.pi * wl.steps * wl.tau) * u0
    err = np.linalg.norm(u - exact) / np.linalg.norm(exact)
    assert err < 5e-4, err
    # the same for a 1.5x wave speed (K scaled) is far off: the check has teeth
    exact_wrong = math.cos(1.5 * math.sqrt(2.0) * math.pi * wl.steps * wl.tau) * u0
    assert np.linalg.norm(u - exact_wrong) / np.linalg.norm(exact_wrong) > 1e-2


@pytest.mark.parametrize("forced", [False, True])
def test_2d_stepping_vs_modal_closed_form(forced):
    src = workloads.Source(f=(("gauss", 0.4, 0.1), ("gauss", 0.55, 0.1), ("sin",))) if forced else None
    wl = _wl2d((13, 10, 0), 3, 5e-3, 30, src)
    o = oracle.make_solver(wl)
    u0 = o.get_state()[0].copy()
    o.step(wl.steps)
    m = ModalPWave(wl.nel, wl.p, wl.tau)
    if forced:
        mu, mud, ma = m.run(u0, nsteps=wl.steps, source=oracle.source_vectors(wl), wavelet=src.wavelet,
                            f0=src.f0, t0=src.t0)
    else:
        mu, mud, ma = m.run(u0, nsteps=wl.steps)
    for a, b in zip(o.get_state(), (mu, mud, ma)):
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)


# ----------------------------------------------------------------- source pieces (C14)
def test_ricker_closed_form_properties():
    """or_ricker (the source of BASELINE configs[2]; reading C14) against properties of the Ricker
    ("Mexican hat") wavelet that do not depend on how its formula is typed: peak 1 at t0, symmetric
    about t0, zeros at t0 +- 1/(sqrt(2) pi f0), troughs -2 exp(-3/2) at t0 +- sqrt(3/2)/(pi f0),
    zero mean; and c3's start value R(0) with f0 t0 = 1, i.e. (1 - 2 pi^2) exp(-pi^2) = -9.69e-4
    (SURVEY.md §8(d)).  Catches a wrong constant (pi vs 2 pi, sigma convention), sign or centre."""
    from scipy.integrate import quad
    for f0, t0 in [(25.0, 0.04), (10.0, 0.02), (3.0, 0.7)]:
        assert oracle.ricker(t0, f0, t0) == 1.0
        z = 1.0 / (math.sqrt(2.0) * math.pi * f0)
        tr = math.sqrt(1.5) / (math.pi * f0)
        for s in (-1.0, 1.0):
            assert abs(oracle.ricker(t0 + s * z, f0, t0)) < 1e-15
            assert abs(oracle.ricker(t0 + s * tr, f0, t0) + 2.0 * math.exp(-1.5)) < 1e-15
        for dt in (0.1 * z, 0.7 * z, 2.3 * z):
            assert oracle.ricker(t0 + dt, f0, t0) == pytest.approx(oracle.ricker(t0 - dt, f0, t0), rel=1e-14)
        # minimum over a fine grid is the trough (no lower value anywhere)
        ts = t0 + np.linspace(-5 * z, 5 * z, 4001)
        assert min(oracle.ricker(t, f0, t0) for t in ts) >= -2.0 * math.exp(-1.5) - 1e-15
        span = 12.0 / f0
        area, _ = quad(lambda t: oracle.ricker(t, f0, t0), t0 - span, t0 + span, points=[t0], limit=200)
        assert abs(area) < 1e-10 / f0
    g = _gold("ricker_c3.json")
    r0 = (1.0 - 2.0 * math.pi ** 2) * math.exp(-math.pi ** 2)
    assert abs(r0 - g["R0"]) < 5e-8          # the survey's printed value, 4 digits
    assert abs(oracle.ricker(0.0, 25.0, 0.04) - r0) < 1e-17
    # the peak of the c3 source falls on step t0 / tau = 40
    assert oracle.ricker(40 * 1e-3, 25.0, 0.04) == 1.0


@pytest.mark.parametrize("p,nel,bc", [(1, 24, 0), (2, 64, 1), (3, 40, 1), (3, 13, 0), (5, 30, 0)])
def test_load_vector_vs_adaptive_quadrature(p, nel, bc):
    """or_load_1d, b_a = int f N_a (the L2-projection right-hand side; reading C4: 8
    Gauss points per element) against scipy's adaptive quad of f times the scipy BSpline basis
    function over its support, for the Gaussian of c2-c5 (several centres and widths, incl. c3's
    sigma = 0.02) and sin(pi x) of c1.  Catches a wrong normalisation (2 sigma^2 vs sigma^2), a
    shifted centre, a wrong basis index or element map, and the Dirichlet end handling."""
    from scipy.integrate import quad
    from scipy.interpolate import BSpline
    from pins_util import open_knots
    t = open_knots(p, nel)
    n = nel + p
    brk = np.linspace(0.0, 1.0, nel + 1)
    funcs = [("sin",), ("gauss", 0.5, 0.05), ("gauss", 0.3, 0.02), ("gauss", 0.71, 0.13)]
    # the 8-point rule (C4) integrates f N_a to rounding only where f is resolved, h <= sigma
    funcs = [fn for fn in funcs if fn[0] == "sin" or fn[2] * nel >= 1.0]
    for fn in funcs:
        f = (lambda x: math.sin(math.pi * x)) if fn[0] == "sin" else \
            (lambda x, c=fn[1], s=fn[2]: math.exp(-(x - c) ** 2 / (2.0 * s * s)))
        b = oracle.load_1d(p, nel, bc, fn)
        ref = np.zeros(n)
        for a in range(n):
            Na = BSpline(t, np.eye(n)[a], p, extrapolate=False)
            lo, hi = t[a], t[a + p + 1]
            pts = [x for x in brk if lo < x < hi]
            ref[a] = quad(lambda x: f(x) * float(np.nan_to_num(Na(x))), lo, hi, points=pts or None,
                          limit=400, epsabs=1e-16, epsrel=1e-14)[0]
        if bc == 1:
            ref[0] = ref[-1] = 0.0
        scale = np.abs(ref).max()
        # 8-point Gauss on a degree-p polynomial times an analytic f: error ~ (h/sigma)^16
        assert np.abs(b - ref).max() <= 2e-12 * scale, (fn, np.abs(b - ref).max() / scale)


def test_extended_precision_oracle_rows_and_agreement():
    """The extended-precision build (libads_oracle_ld.so, the truth reference of DESIGN.md T1) is
    the same algorithm: its interior Gram rows equal the exact rational cardinal values to
    long-double accuracy (the fp64 build only to ~1e-13 relative), and one step of c2's recipe
    agrees with the fp64 build to fp64 rounding."""
    from fractions import Fraction
    if np.finfo(np.longdouble).eps >= 1e-17:
        pytest.skip("long double is not extended precision on this platform")
    g = _gold("cardinal_rows.json")
    for p, nel in [(2, 16), (3, 32)]:
        s = oracle.PWave((nel, 4, 4), p, 1e-3, bc=0, ext=True)
        M, K = s.matrix(0, 0), s.matrix(0, 1)
        row = nel // 2
        (_, mv), (_, kv) = list(g[f"p{p}"].items())
        msc, ksc = (120, 6) if p == 2 else (5040, 120)
        for k in range(-p, p + 1):
            exm = Fraction(mv[k + p], msc * nel)                 # h [..] / scale
            exk = Fraction(kv[k + p] * nel, ksc)                 # [..] / (scale h)
            # np.longdouble -> exact rational through its decimal repr (21 significant digits)
            gm = Fraction(np.format_float_scientific(M[row, row + k], unique=True))
            gk = Fraction(np.format_float_scientific(K[row, row + k], unique=True))
            assert abs(gm - exm) <= abs(exm) * Fraction(1, 10 ** 17)
            assert abs(gk - exk) <= abs(exk) * Fraction(1, 10 ** 17)
    wl = workloads.get("c2").scaled(20, 1)
    u0 = oracle.project_separable(wl)
    a = oracle.PWave(wl.nel, wl.p, wl.tau, wl.bc)
    b = oracle.PWave(wl.nel, wl.p, wl.tau, wl.bc, ext=True)
    for s in (a, b):
        s.set_state(u0)
        s.step(1)
    for x, y in zip(a.get_state(), b.get_state()):
        assert rel_l2(x, np.asarray(y, dtype=np.float64)) < 1e-13


# ---- 2D elasticity (row f2): nel_z = 0, PAPER.md:362-387 ----
def test_elastic_2d_operator_vs_bruteforce():
    """2D Upsilon (nel_z = 0: one z function, M_z = 1, K_z = B_z = 0) == the dense plane-strain
    stiffness assembled from strains (PAPER.md:362-387 blocks, readings C10/C11): the in-plane
    blocks match it, the antiplane component u_z only sees mu (Kx My + Mx Ky) and nothing couples
    it to (u_x, u_y)."""
    from pins_util import brute_force_elastic_2d
    p, nel, lam, mu = 2, 3, 1.7, 0.6
    _, K2, A2 = brute_force_elastic_2d(p, nel, lam, mu)
    el = oracle.Elastic((nel, nel, 0), p, 0.1, bc=0, lam=lam, mu=mu)
    nd = (nel + p) ** 2
    x = workloads.random_field(41, 3 * nd)
    y = el.apply(x).ravel()
    np.testing.assert_allclose(y[:2 * nd], A2 @ x[:2 * nd], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(y[2 * nd:], mu * (K2 @ x[2 * nd:]), rtol=1e-12, atol=1e-12)
    xz = x.copy()
    xz[:2 * nd] = 0.0
    assert np.abs(el.apply(xz).ravel()[:2 * nd]).max() == 0.0


def test_elastic_2d_rigid_body_kernel():
    """Natural (traction-free) 2D BC: the three in-plane rigid motions -- two
    translations and the rotation (-y, x) -- and the antiplane translation are in the kernel."""
    p, nel = 3, 4
    el = oracle.Elastic((nel, nel, 0), p, 0.1, bc=0, lam=1.3, mu=0.7)
    n = nel + p
    t = oracle.knots(p, nel)
    g = np.array([t[a + 1:a + p + 1].mean() for a in range(n)])  # Greville: linear reproduction
    Y, X = np.meshgrid(g, g, indexing="ij")
    one, zero = np.ones_like(X), np.zeros_like(X)
    for m in [(one, zero, zero), (zero, one, zero), (-Y, X, zero), (zero, zero, one)]:
        u = np.stack(m)[:, None]
        assert np.abs(el.apply(u)).max() < 1e-12 * n * n
    # a non-rigid in-plane motion (shear) is not
    assert np.abs(el.apply(np.stack((Y, zero, zero))[:, None])).max() > 1e-3


@pytest.mark.parametrize("tau", [0.01, 0.5, 10.0])
def test_elastic_2d_invariant_and_decoupling(tau):
    """The 2D E1 scheme conserves its invariant at any tau and a state with
    u_z = 0 keeps u_z = 0 (the 2D problem of the paper is the (u_x, u_y) part)."""
    wl = workloads.get("c5").scaled(6)
    wl.nel = (6, 5, 0)
    el = oracle.Elastic(wl.nel, 2, tau, bc=1)
    u0 = workloads_2d_elastic(wl)
    el.set_state(u0)
    e0 = el.energy()
    assert e0[2] > 0
    el.step(25)
    e = el.energy()
    assert abs(e[2] - e0[2]) <= 1e-12 * e0[2]
    u, ud, a = el.get_state()
    assert np.abs(u[2]).max() == 0.0 and np.abs(ud[2]).max() == 0.0


def test_elastic_2d_second_order():
    """Second order in time for the 2D problem: tau-halving against the
    semi-discrete exact solution from a dense generalised eigensolve of the brute-force plane-strain
    operator (Dirichlet, interior DOFs)."""
    import scipy.linalg
    from pins_util import brute_force_elastic_2d
    p, nel, lam, mu, rho = 2, 4, 1.0, 1.0, 1.0
    wl = workloads.get("c5").scaled(nel)
    wl.nel = (nel, nel, 0)
    u0 = workloads_2d_elastic(wl)
    M2, _, A2 = brute_force_elastic_2d(p, nel, lam, mu)
    n = nel + p
    m2 = np.ones((n, n), dtype=bool)
    m2[0, :] = m2[-1, :] = m2[:, 0] = m2[:, -1] = False
    m = np.tile(m2.ravel(), 2)
    RM = np.kron(np.eye(2), rho * M2)[np.ix_(m, m)]
    lamv, Q = scipy.linalg.eigh(A2[np.ix_(m, m)], RM)
    T = 0.5
    uin = u0[:2].reshape(-1)[m]
    ex = Q @ (np.cos(np.sqrt(lamv) * T) * (Q.T @ RM @ uin))
    errs = []
    for tau in [0.02, 0.01, 0.005]:
        el = oracle.Elastic(wl.nel, p, tau, bc=1, lam=lam, mu=mu, rho=rho)
        el.set_state(u0)
        el.step(int(round(T / tau)))
        u, _, _ = el.get_state()
        errs.append(np.linalg.norm(u[:2].reshape(-1)[m] - ex))
    ratios = [errs[0] / errs[1], errs[1] / errs[2]]
    assert all(3.7 < r < 4.3 for r in ratios), ratios


def workloads_2d_elastic(wl):
    """A smooth 2D elastic start: the c5 recipe's bumps in (x, y), u_z = 0 (projected by the oracle)."""
    w = workloads.Workload(name="2d-el", p=wl.p, nel=wl.nel, tau=wl.tau, steps=wl.steps, bc=wl.bc, elastic=True,
                           u0=[t for t in wl.u0 if t.comp < 2])  # along the 2D axis every load is [1]
    return oracle.project_separable(w)
