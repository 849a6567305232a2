"""GPU parity of the exact-in-time modal propagator (ads_modal_advance; SURVEY.md §8 row f3,
PAPER.md:157-176) against the modal oracle (oracle/modal.py) and against the library's own
stepping (ads_step).  Tolerances: the oracle and the GPU use independent bases (scipy eigh vs
the library's Householder/QL) and independent transforms, so agreement is bounded by the
basis error amplified by the operator (T1): 1e-11 relative L2 on (U, udot, a)."""
import numpy as np
import pytest

import oracle
from oracle.modal import ModalPWave
import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-11


def rel(a, b):
    a, b = np.ravel(a), np.ravel(b)
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


def _state(shape, seed, bc=1):
    u = workloads.random_field(seed, int(np.prod(shape))).reshape(shape)
    v = workloads.random_field(seed + 1, int(np.prod(shape))).reshape(shape)
    # smooth the fields (a few low modes dominate, like the paper's bumps) and zero Dirichlet DOFs
    z, y, x = np.meshgrid(*(np.linspace(0, 1, n) for n in shape), indexing="ij")
    env = np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
    u, v = env * (1 + 0.1 * u), env * 0.5 * (1 + 0.1 * v)
    if bc == 1:
        for f in (u, v):
            f[0], f[-1], f[:, 0], f[:, -1], f[:, :, 0], f[:, :, -1] = 0, 0, 0, 0, 0, 0
    return u, v


@pytest.mark.parametrize("nel,p,tau,nsteps", [((16, 16, 16), 2, 1e-2, 20), ((21, 13, 30), 3, 5e-3, 37),
                                              ((131, 70, 150), 3, 2e-3, 9), ((200, 129, 67), 2, 1e-3, 5),
                                              ((9, 11, 7), 1, 2e-2, 64), ((12, 10, 8), 5, 4e-3, 5)])
def test_free_run_vs_modal_oracle_and_stepping(ads, nel, p, tau, nsteps):
    g = ads.Solver(nel, p, tau)
    u0, v0 = _state(g.shape, 11)
    g.set_state(u0, v0)
    g.modal_advance(nsteps)
    gu, gud, ga = g.get_state()
    assert g.step_count() == nsteps
    mu, mud, ma = ModalPWave(nel, p, tau).run(u0, v0, nsteps=nsteps)
    assert rel(gu, mu) < TOL and rel(gud, mud) < TOL and rel(ga, ma) < TOL, (rel(gu, mu), rel(gud, mud), rel(ga, ma))
    s = ads.Solver(nel, p, tau)
    s.set_state(u0, v0)
    s.step(nsteps)
    su, sud, sa = s.get_state()
    assert rel(gu, su) < TOL and rel(gud, sud) < TOL and rel(ga, sa) < TOL


def test_forced_run_vs_modal_oracle_and_stepping(ads):
    wl = workloads.get("c3").scaled(20, 60)
    g = ads.make_solver(wl)           # zero state, Ricker-forced separable source (t up to 0.06)
    g.modal_advance(wl.steps)
    gu, gud, ga = g.get_state()
    src = wl.source
    mu, mud, ma = ModalPWave(wl.nel, wl.p, wl.tau).run(np.zeros(g.shape), nsteps=wl.steps,
                                                        source=oracle.source_vectors(wl), wavelet=src.wavelet,
                                                        f0=src.f0, t0=src.t0)
    assert rel(gu, mu) < TOL and rel(gud, mud) < TOL and rel(ga, ma) < TOL, (rel(gu, mu), rel(gud, mud), rel(ga, ma))
    s = ads.make_solver(wl)
    s.step(wl.steps)
    su, sud, sa = s.get_state()
    assert rel(gu, su) < TOL and rel(gud, sud) < TOL and rel(ga, sa) < TOL


def test_mixed_stepping_and_modal(ads):
    """step(7) + modal_advance(20) + step(6) == step(33): the device step counter (source time of
    graph replays) follows the modal jump."""
    wl = workloads.get("c3").scaled(16, 33)
    g = ads.make_solver(wl)
    g.step(7)
    g.modal_advance(20)
    g.step(6)
    s = ads.make_solver(wl)
    s.step(33)
    for a, b in zip(g.get_state(), s.get_state()):
        assert rel(a, b) < TOL


def test_natural_bc_vs_stepping(ads):
    nel, p, tau = (14, 9, 11), 2, 1e-2
    g = ads.Solver(nel, p, tau, 0)
    u0, v0 = _state(g.shape, 5, bc=0)
    g.set_state(u0, v0)
    g.modal_advance(40)
    s = ads.Solver(nel, p, tau, 0)
    s.set_state(u0, v0)
    s.step(40)
    for a, b in zip(g.get_state(), s.get_state()):
        assert rel(a, b) < TOL


def test_long_run_invariant_and_oracle(ads):
    """10^6 steps in one call (time independent of nsteps): the conserved invariant (C6)
    is unchanged and the state matches the modal oracle's repeated squaring."""
    nel, p, tau = (12, 12, 12), 2, 1e-2
    g = ads.Solver(nel, p, tau)
    u0, v0 = _state(g.shape, 3)
    g.set_state(u0, v0)
    e0 = g.energy()
    g.modal_advance(10 ** 6)
    e1 = g.energy()
    assert abs(e1[2] - e0[2]) <= 1e-10 * abs(e0[2])
    mu, mud, ma = ModalPWave(nel, p, tau).run(u0, v0, nsteps=10 ** 6)
    gu, gud, ga = g.get_state()
    assert rel(gu, mu) < 1e-9 and rel(gud, mud) < 1e-9


def test_errors(ads):
    e = ads.Solver((4, 4, 4), 2, 1e-2, elastic=True)
    e.set_state(np.zeros(e.shape))
    with pytest.raises(ads.AdsError):
        e.modal_advance(3)
    g = ads.Solver((4, 4, 4), 2, 1e-2)
    with pytest.raises(ads.AdsError):
        g.modal_advance(3)  # no state yet
    g.set_state(np.zeros(g.shape))
    with pytest.raises(ads.AdsError):
        g.modal_advance(-1)
