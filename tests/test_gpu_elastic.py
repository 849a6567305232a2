"""GPU parity of the 3D elasticity path (E1)
through the C ABI against the CPU oracle (-m gpu).

Same tolerances as the P-wave path: relative L2 <= 1e-12 after one step and <= 1e-9 after the
run, on U, the returned udot and a (all three components); unit operators (Upsilon apply and the
delta-form predictor/corrector D~^-1) at 1e-13.
"""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

STEP1_TOL = 1e-12
RUN_TOL = 1e-9
OP_TOL = 1e-13


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def ads():
    import torch
    import paper_1911_08158_b200 as ads
    from paper_1911_08158_b200 import build
    build.build()
    assert torch.cuda.is_available()
    return ads


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# (nel, p, bc, lam, mu, rho, tau): several tiles / chunk layouts, ragged tails, both BCs
OP_CASES = [
    ((9, 7, 11), 2, 1, 1.0, 1.0, 1.0, 1e-2),
    ((6, 13, 5), 3, 0, 1.3, 0.7, 1.2, 0.05),
    ((40, 5, 6), 1, 1, 0.0, 2.0, 0.5, 0.3),
    ((3, 3, 3), 2, 0, 2.0, 0.5, 1.0, 1.0),
    # grids with Kronecker tiles inside the Toeplitz interior of every F_y (the coefficient-from-
    # parameters path of kron3_kernel) next to boundary tiles, and z pieces with staged F_z rows
    ((40, 40, 12), 2, 1, 1.0, 1.0, 1.0, 1e-3),
    ((20, 52, 33), 3, 0, 0.8, 1.1, 1.3, 2e-2),
]


@pytest.mark.parametrize("nel,p,bc,lam,mu,rho,tau", OP_CASES)
def test_elastic_unit_operators(ads, nel, p, bc, lam, mu, rho, tau):
    """Upsilon x (diagonal blocks in the fused operator kernel, couplings as banded Kronecker
    triples) and D~^-1 x (predictor/corrector over six partitioned ADS solves) vs the oracle."""
    import torch
    s = ads.Solver(nel, p, tau, bc, elastic=True, lam=lam, mu=mu, rho=rho)
    o = oracle.Elastic(nel, p, tau, bc, lam, mu, rho)
    x = workloads.random_field(7 + p, 3 * s.N).reshape(s.shape)
    if bc == 1:  # Dirichlet: the operators act on the interior-restricted spaces
        x[:, 0], x[:, -1], x[:, :, 0], x[:, :, -1], x[:, :, :, 0], x[:, :, :, -1] = 0, 0, 0, 0, 0, 0
    xd = _dev(x)
    out = torch.empty_like(xd)
    s.apply_k(xd, out)
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), o.apply(x)) < OP_TOL
    s.solve_d(xd, out)
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), o.dsolve(x)) < OP_TOL


def _compare_run(ads, wl, checkpoints):
    """One step against the extended-precision oracle (T1), later checkpoints against
    the fp64 oracle stepped alongside; both sides start from the oracle's projection."""
    u0 = oracle.project_separable(wl)
    g = ads.make_solver(wl, u0=u0)
    o = oracle.make_solver(wl, u0=u0)
    done = 0
    for nsteps in checkpoints:
        g.step(nsteps - done)
        o.step(nsteps - done)
        done = nsteps
        ref = oracle.one_step_truth(wl, u0) if nsteps == 1 else o.get_state()
        tol = STEP1_TOL if nsteps == 1 else RUN_TOL
        errs = tuple(rel(x, y) for x, y in zip(g.get_state(), ref))
        assert max(errs) < tol, (wl.name, nsteps, errs)
    return g, o


def test_c5_recipe_scaled(ads):
    """Config 5 recipe (lambda = mu = rho = 1, p = 2, one seeded bump per component) on 20^3
    elements, full 100 steps; energies agree and the invariant is conserved."""
    wl = workloads.get("c5").scaled(20)
    g, o = _compare_run(ads, wl, [1, 40, wl.steps])
    ge, oe = g.energy(), o.energy()
    assert np.allclose(ge, oe, rtol=1e-11, atol=1e-15), (ge, oe)


def test_elastic_anisotropic_natural(ads):
    wl = workloads.get("c5").scaled(8, 25)
    wl.nel = (11, 8, 13)
    wl.bc = 0
    wl.lam, wl.mu, wl.rho = 1.7, 0.6, 1.1
    _compare_run(ads, wl, [1, 25])


def test_elastic_invariant_large_tau(ads):
    """Unconditional stability: the invariant stays constant at tau = 10."""
    wl = workloads.get("c5").scaled(10, 0)
    wl.tau = 10.0
    g = ads.make_solver(wl)
    e0 = g.energy()
    g.step(40)
    e1 = g.energy()
    assert e0[2] > 0 and abs(e1[2] - e0[2]) < 1e-11 * e0[2], (e0, e1)


def test_elastic_errors(ads):
    with pytest.raises(ads.AdsError):
        ads.Solver(4, 2, 0.1, elastic=True, mu=0.0)
    g = ads.Solver(4, 2, 0.1, elastic=True)
    with pytest.raises(ads.AdsError):
        g.sweep(0, _dev(np.zeros(g.shape)), _dev(np.zeros(g.shape)))


@pytest.mark.slow
def test_c5_full_size(ads):
    """Full config 5 (BASELINE configs[4]: 130^3 x 3 components, 100 steps): one step against the
    extended-precision oracle at 1e-12 and the whole run against the fp64 C oracle stepped
    alongside at 1e-9, element by element on U, udot and a; the invariant is conserved."""
    wl = workloads.get("c5")
    g, o = _compare_run(ads, wl, [1, wl.steps])
    e1 = g.energy()
    assert np.allclose(e1, o.energy(), rtol=1e-10, atol=1e-15)
    g0 = ads.make_solver(wl, u0=oracle.project_separable(wl))
    e0 = g0.energy()
    assert abs(e1[2] - e0[2]) < 1e-12 * wl.steps * e0[2], (e0, e1)


def _wl2d_elastic(nel, p, bc, tau=2e-3, steps=30, lam=1.0, mu=1.0):
    """The c5 recipe's (u_x, u_y) bumps on a 2D grid (nel_z = 0), u_z = 0: the plane-strain problem
    PAPER.md:362-387 (row f2)."""
    wl = workloads.get("c5").scaled(8, steps)
    wl.nel, wl.p, wl.bc, wl.tau, wl.lam, wl.mu = nel, p, bc, tau, lam, mu
    wl.u0 = [t for t in wl.u0 if t.comp < 2]
    return wl


@pytest.mark.parametrize("nel,p,bc", [((37, 21, 0), 2, 1), ((20, 33, 0), 3, 0), ((64, 48, 0), 2, 1)])
def test_elastic_2d_vs_oracle(ads, nel, p, bc):
    """Row f2: 2D (plane-strain) elasticity, ads_create_elastic with nz = 0, against the oracle's 2D
    path: one step vs the extended-precision oracle at 1e-12, a 30-step run at 1e-9, energies; u_z
    stays zero."""
    wl = _wl2d_elastic(nel, p, bc, lam=1.3, mu=0.8)
    g, o = _compare_run(ads, wl, [1, wl.steps])
    assert g.shape == (3, 1, nel[1] + p, nel[0] + p)
    assert np.allclose(g.energy(), o.energy(), rtol=1e-11, atol=1e-15)
    u, ud, a = g.get_state()
    assert np.abs(u[2]).max() == 0.0 and np.abs(ud[2]).max() == 0.0


def test_elastic_2d_unit_operators(ads):
    """2D Upsilon and D~^-1 on the GPU vs the oracle (random fields, natural BC)."""
    import torch
    nel, p = (23, 17, 0), 3
    s = ads.Solver(nel, p, 0.05, 0, elastic=True, lam=1.1, mu=0.9)
    o = oracle.Elastic(nel, p, 0.05, 0, 1.1, 0.9, 1.0)
    x = workloads.random_field(17, 3 * s.N).reshape(s.shape)
    xd = _dev(x)
    out = torch.empty_like(xd)
    s.apply_k(xd, out)
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), o.apply(x)) < OP_TOL
    s.solve_d(xd, out)
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), o.dsolve(x)) < OP_TOL
