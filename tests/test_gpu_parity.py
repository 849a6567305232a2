"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle (-m gpu).

Tolerances (BASELINE.json north_star): relative L2 <= 1e-12 after one step and
<= 1e-9 after the full run, on U, the returned udot and a.  Unit operators are
held to 1e-13 (a single application; cond(A_d) <= ~30).
"""
import numpy as np
import pytest

import oracle
from oracle.modal import ModalPWave
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


# grids spanning several kop tiles (32 x 8) / sweep chunk layouts with ragged tails
OP_CASES = [
    ((37, 21, 13), 3, 1),
    ((40, 9, 70), 2, 0),
    ((5, 6, 7), 1, 1),
    ((11, 12, 13), 4, 0),
    ((9, 8, 10), 5, 1),
    ((1, 1, 1), 2, 0),
    ((1, 1, 1), 1, 0),
    ((1, 2, 1), 2, 1),
    ((100, 3, 5), 3, 1),
]


@pytest.mark.parametrize("nel,p,bc", OP_CASES)
def test_unit_operators(ads, nel, p, bc):
    """K-apply (fused kernel), each directional sweep and the full D^-1 vs the oracle."""
    import torch
    tau = 0.013 * (1 + p)
    s = ads.Solver(nel, p, tau, bc)
    o = oracle.PWave(nel, p, tau, bc)
    x = workloads.random_field(100 + p, s.N).reshape(s.shape)
    xd = _dev(x)
    out = torch.empty_like(xd)
    s.apply_k(xd, out)
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), o.kapply(x)) < OP_TOL
    s.solve_d(xd, out)
    torch.cuda.synchronize()
    assert rel(out.cpu().numpy(), o.dsolve(x)) < OP_TOL
    # single-direction sweeps vs dense 1D solves along that axis
    for d in range(3):
        s.sweep(d, xd, out)
        torch.cuda.synchronize()
        A = o.matrix(d, 2)
        axis = 2 - d  # numpy (z, y, x)
        ref = np.moveaxis(np.linalg.solve(A, np.moveaxis(x, axis, 0).reshape(A.shape[0], -1)).reshape(
            np.moveaxis(x, axis, 0).shape), 0, axis)
        assert rel(out.cpu().numpy(), ref) < OP_TOL, d


def _compare_run(ads, wl, nsteps_list, tol_first=STEP1_TOL, tol_run=RUN_TOL):
    """One step against the extended-precision oracle (the truth of the one-step bound, DESIGN.md
    T1), later checkpoints against the fp64 oracle stepped alongside.  Both sides start from the
    oracle's projection of the workload."""
    u0 = oracle.project_separable(wl)
    g = ads.make_solver(wl, u0=u0)
    o = oracle.make_solver(wl, u0=u0)
    done = 0
    for k, nsteps in enumerate(nsteps_list):
        g.step(nsteps - done)
        o.step(nsteps - done)
        done = nsteps
        gu, gud, ga = g.get_state()
        ref = oracle.one_step_truth(wl, u0) if nsteps == 1 else o.get_state()
        tol = tol_first if nsteps == 1 else tol_run
        errs = tuple(rel(x, y) for x, y in zip((gu, gud, ga), ref))
        assert max(errs) < tol, (wl.name, nsteps, errs)
    return g, o


def test_c1_full_run(ads):
    """BASELINE config 1 exactly (p=2, 16^3 el, tau 1e-2, 20 steps)."""
    wl = workloads.get("c1")
    g, o = _compare_run(ads, wl, [1, wl.steps])
    ge, oe = g.energy(), o.energy()
    assert np.allclose(ge, oe, rtol=1e-12, atol=1e-15)


def test_c2_full_run(ads):
    """BASELINE config 2 exactly (p=3, 64^3 el, tau 5e-3, 100 steps)."""
    wl = workloads.get("c2")
    _compare_run(ads, wl, [1, wl.steps])


def test_c3_recipe_scaled(ads):
    """Config 3 recipe (Ricker x Gaussian source, zero state) on 40^3 elements, full 200 steps."""
    wl = workloads.get("c3").scaled(40)
    g, o = _compare_run(ads, wl, [1, 60, wl.steps])
    ge, oe = g.energy(), o.energy()
    assert np.allclose(ge, oe, rtol=1e-11)


def test_c4_recipe_scaled(ads):
    """Config 4 recipe (8 seeded bumps, p=3) on 48^3 elements, full 100 steps."""
    wl = workloads.get("c4").scaled(48)
    _compare_run(ads, wl, [1, wl.steps])


def test_anisotropic_natural_bc(ads):
    wl = workloads.get("c2").scaled(10, 30)
    wl.nel = (23, 10, 17)
    wl.bc = 0
    _compare_run(ads, wl, [1, 30])


def test_set_get_roundtrip_and_energy_invariant(ads):
    wl = workloads.get("c2").scaled(12, 0)
    g = ads.make_solver(wl)
    u0 = oracle.project_separable(wl)
    u, ud, a = g.get_state()
    assert rel(u, u0) < 1e-14
    assert np.abs(ud).max() < 1e-14 * np.abs(u0).max() + 1e-300
    e0 = g.energy()
    g.step(50)
    e1 = g.energy()
    assert abs(e1[2] - e0[2]) < 1e-12 * e0[2]


def test_device_state_io_and_stream(ads):
    """set_state/get_state with device (torch) tensors and a caller stream."""
    import torch
    wl = workloads.get("c1")
    g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
    st = torch.cuda.Stream()
    g.set_stream(st)
    u0 = oracle.project_separable(wl)
    v0 = 0.3 * u0
    g.set_state(_dev(u0), _dev(v0))
    g.step(5)
    u = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    ud = torch.empty_like(u)
    a = torch.empty_like(u)
    g.get_state(u, ud, a)
    o = oracle.PWave(wl.nel, wl.p, wl.tau, wl.bc)
    o.set_state(u0, v0)
    o.step(5)
    ou, oud, oa = o.get_state()
    assert rel(u.cpu().numpy(), ou) < 1e-12 and rel(ud.cpu().numpy(), oud) < 1e-12 and rel(a.cpu().numpy(), oa) < 1e-12


def test_errors(ads):
    g = ads.Solver(4, 2, 0.1)
    with pytest.raises(ads.AdsError) as e:
        g.step(1)  # before set_state
    assert e.value.code == -6
    with pytest.raises(ads.AdsError):
        g.load_vector(3, ("sin",))
    g.set_state(np.zeros(g.shape))
    with pytest.raises(ads.AdsError):
        g.step(-1)
    g.step(0)
    assert g.step_count() == 0


# ------------------------------------------------------------------ full-size cases (slow)
@pytest.mark.slow
def test_c3_full_size_vs_modal(ads):
    """Full config 3 (258^3, 200 steps, forced) vs the modal oracle (exact mode-by-mode)."""
    wl = workloads.get("c3")
    g = ads.make_solver(wl)
    g.step(wl.steps)
    gu, gud, ga = g.get_state()
    src = wl.source
    mu, mud, ma = ModalPWave(wl.nel, wl.p, wl.tau).run(np.zeros(g.shape), nsteps=wl.steps,
                                                        source=oracle.source_vectors(wl), wavelet=src.wavelet,
                                                        f0=src.f0, t0=src.t0)
    assert rel(gu, mu) < RUN_TOL and rel(gud, mud) < RUN_TOL and rel(ga, ma) < RUN_TOL


@pytest.mark.slow
def test_c4_full_size_one_step_and_run(ads):
    """Full config 4 (515^3): one step vs the C oracle element by element, full 100-step run vs
    the modal oracle."""
    wl = workloads.get("c4")
    # both sides start from the SAME coefficients (the oracle's L2 projection); the one-step
    # reference is the extended-precision oracle (north_star's 1e-12 on U, udot and a against
    # the truth; T1)
    u0 = oracle.project_separable(wl)
    g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
    g.set_state(u0)
    g.step(1)
    gu, gud, ga = g.get_state()
    tu, tud, ta = oracle.one_step_truth(wl, u0)
    errs = (rel(gu, tu), rel(gud, tud), rel(ga, ta))
    del tu, tud, ta
    assert max(errs) < STEP1_TOL, errs
    g.step(wl.steps - 1)
    gu, gud, ga = g.get_state()
    mu, mud, ma = ModalPWave(wl.nel, wl.p, wl.tau).run(u0, nsteps=wl.steps)
    assert rel(gu, mu) < RUN_TOL and rel(gud, mud) < RUN_TOL and rel(ga, ma) < RUN_TOL


@pytest.mark.parametrize("p,nel", [(1, (30, 9, 17)), (4, (13, 11, 9)), (5, (12, 7, 10))])
def test_full_run_other_degrees(ads, p, nel):
    """Degrees 1, 4, 5 (specialised kernels for every p in [1, 5]) through a 25-step forced run."""
    wl = workloads.get("c3").scaled(8, 25)
    wl.p, wl.nel, wl.tau = p, nel, 2e-3
    wl.source = workloads.Source(f=(("gauss", 0.4, 0.1), ("gauss", 0.5, 0.1), ("gauss", 0.6, 0.1)), f0=10.0, t0=0.02)
    # a = D^-1 F: the solve's rounding error is bounded by eps cond(D), cond(D) = prod_d cond(A_d)
    # (Kronecker product); B-spline mass matrices grow ill-conditioned with p (T1)
    o = oracle.PWave(nel, p, wl.tau, 1)
    kappa = float(np.prod([np.linalg.cond(o.matrix(d, 2)[1:-1, 1:-1]) for d in range(3)]))
    _compare_run(ads, wl, [1, 25], tol_first=max(STEP1_TOL, 2.2e-16 * kappa))


def test_largest_line_length(ads):
    """n_d = 1056 (the largest supported line: 32 chunks of 33 rows) in x, y and z separately."""
    import torch
    for nel in [(1053, 4, 5), (4, 1053, 5), (5, 4, 1053)]:
        s = ads.Solver(nel, 3, 1e-3, 1)
        o = oracle.PWave(nel, 3, 1e-3, 1)
        x = workloads.random_field(5, s.N).reshape(s.shape)
        xd = _dev(x)
        out = torch.empty_like(xd)
        s.solve_d(xd, out)
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), o.dsolve(x)) < OP_TOL, nel
    with pytest.raises(ads.AdsError):
        ads.Solver((1054, 4, 4), 3, 1e-3, 1)


_SPLIT_CHILD = r'''
import sys, numpy as np
sys.path.insert(0, sys.argv[3])
import paper_1911_08158_b200 as ads, workloads
s = ads.Solver((40, 37, 45), 3, 2e-3)
u0 = workloads.random_field(7, s.N).reshape(s.shape)
v0 = workloads.random_field(8, s.N).reshape(s.shape)
for f in (u0, v0):  # zero Dirichlet DOFs
    f[0], f[-1], f[:, 0], f[:, -1], f[:, :, 0], f[:, :, -1] = 0, 0, 0, 0, 0, 0
s.set_state(u0, v0)
s.step(5)
np.save(sys.argv[2], np.stack(s.get_state()))
'''


@pytest.mark.parametrize("nz", [1, 3, 7])
def test_kop_z_split_is_bitwise_invariant(ads, tmp_path, nz):
    """The fused operator kernel's z split (launch configuration, kernels.cu kop_launch) must not
    change a single bit: every output plane receives its 2p+1 contributions in the same order."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag, env_nz in (("auto", None), ("forced", str(nz))):
        env = dict(os.environ)
        env.pop("ADS_KOP_NZ", None)
        if env_nz:
            env["ADS_KOP_NZ"] = env_nz
        f = str(tmp_path / f"{tag}.npy")
        r = subprocess.run([sys.executable, "-c", _SPLIT_CHILD, tag, f, root], env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[tag] = np.load(f)
    assert np.array_equal(out["auto"], out["forced"])


def test_literal_scheme_r0_vs_oracle(ads):
    """ads_set_scheme(0): the literal Eq. 16 (reading R0) against the oracle's scheme=0, c1 recipe
    and a forced case; under R0 the c1 standing mode is visibly wrong (the garble, R1)."""
    for wl in (workloads.get("c1"), workloads.get("c3").scaled(12, 30)):
        g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
        g.set_scheme(0)
        o = oracle.PWave(wl.nel, wl.p, wl.tau, wl.bc, scheme=0)
        if wl.source is not None:
            bs = oracle.source_vectors(wl)
            g.set_source(bs, wl.source.wavelet, wl.source.f0, wl.source.t0, wl.source.amp)
            o.set_source(bs, wl.source.wavelet, wl.source.f0, wl.source.t0, wl.source.amp)
        u0 = oracle.project_separable(wl) if wl.u0 else np.zeros(g.shape)
        g.set_state(u0)
        o.set_state(u0)
        for n in (1, wl.steps - 1):
            g.step(n)
            o.step(n)
            gs, os_ = g.get_state(), o.get_state()
            # the literal update U + tau V' - tau^2/2 a equals U + tau V only up to rounding: from a
            # zero state the oracle's U after one step is ~1e-26, the GPU's exactly 0, so each
            # field is compared against the state's scale (u, tau udot, tau^2 a)
            scale = max(np.linalg.norm(os_[0]), wl.tau * np.linalg.norm(os_[1]), wl.tau ** 2 * np.linalg.norm(os_[2]))
            for k, (a, b) in enumerate(zip(gs, os_)):
                f = (1.0, wl.tau, wl.tau ** 2)[k]
                tol = STEP1_TOL if n == 1 else RUN_TOL
                assert np.linalg.norm(a - b) <= tol * max(np.linalg.norm(b), scale / f), (n, k, rel(a, b))
        ge, oe = g.energy(), o.energy()
        assert abs(ge[0] - oe[0]) <= 1e-10 * abs(oe[0]) and abs(ge[1] - oe[1]) <= 1e-10 * abs(oe[1])
    with pytest.raises(ads.AdsError):
        g.modal_advance(2)  # the modal propagator implements R1 only
    e = ads.Solver((4, 4, 4), 2, 1e-2, elastic=True)
    with pytest.raises(ads.AdsError):
        e.set_scheme(0)


@pytest.mark.parametrize("forced", [False, True])
def test_set_tau_restart_vs_oracle(ads, forced):
    """ads_set_tau (row f4): n1 steps at tau1, then n2 steps at tau2 from the same physical state
    and time, against the oracle restarted from (u, udot) with tau2 and, when forced, the wavelet
    centre shifted by t_n1 (the oracle's clock restarts at 0)."""
    wl = workloads.get("c3").scaled(12, 0) if forced else workloads.get("c1")
    tau1, tau2, n1, n2 = wl.tau, 0.6 * wl.tau, 9, 14
    g = ads.Solver(wl.nel, wl.p, tau1, wl.bc)
    o1 = oracle.PWave(wl.nel, wl.p, tau1, wl.bc)
    bs = oracle.source_vectors(wl) if forced else None
    if forced:
        g.set_source(bs, wl.source.wavelet, wl.source.f0, wl.source.t0, wl.source.amp)
        o1.set_source(bs, wl.source.wavelet, wl.source.f0, wl.source.t0, wl.source.amp)
    u0 = oracle.project_separable(wl) if wl.u0 else np.zeros(g.shape)
    g.set_state(u0)
    o1.set_state(u0)
    g.step(n1)
    o1.step(n1)
    ou, oud, _ = o1.get_state()
    del o1
    g.set_tau(tau2)
    g.step(n2)
    assert abs(g.time() - (n1 * tau1 + n2 * tau2)) <= 1e-15
    o2 = oracle.PWave(wl.nel, wl.p, tau2, wl.bc)
    if forced:
        o2.set_source(bs, wl.source.wavelet, wl.source.f0, wl.source.t0 - n1 * tau1, wl.source.amp)
    o2.set_state(ou, oud)
    o2.step(n2)
    for a, b in zip(g.get_state(), o2.get_state()):
        assert rel(a, b) < RUN_TOL, rel(a, b)


def test_set_tau_same_step_is_transparent(ads):
    """set_tau with the current tau (forced, graph-replayed steps after it) reproduces the
    uninterrupted run: the restart's a_n equals the stored one and the source clock is kept."""
    wl = workloads.get("c3").scaled(14, 40)
    g = ads.make_solver(wl)
    g.step(17)
    g.set_tau(wl.tau)
    g.step(23)
    s = ads.make_solver(wl)
    s.step(40)
    for a, b in zip(g.get_state(), s.get_state()):
        assert rel(a, b) < 1e-12


def _wl2d(nel, p, tau, steps, bc=1, source=None):
    sin = ("sin",)
    g = ("gauss", 0.45, 0.12)
    return workloads.Workload(name=f"2d{nel}", p=p, nel=nel, tau=tau, steps=steps, bc=bc, source=source,
                              u0=[] if source else [workloads.SeparableTerm(1.0, 0, (sin, g, sin))])


@pytest.mark.parametrize("nel,p,bc,forced", [((37, 21, 0), 3, 1, False), ((20, 33, 0), 2, 0, False),
                                             ((64, 40, 0), 3, 1, True), ((150, 7, 0), 1, 1, False)])
def test_2d_scheme_vs_oracle(ads, nel, p, bc, forced):
    """Row f2: the 2D scheme as printed (ads_create with nz = 0) against the oracle's 2D path,
    one step and a 40-step run, Dirichlet and natural BC, free and Ricker-forced."""
    src = workloads.Source(f=(("gauss", 0.4, 0.1), ("gauss", 0.55, 0.1), ("sin",))) if forced else None
    wl = _wl2d(nel, p, 4e-3, 40, bc, src)
    # both sides start from the oracle's projection; one step is held to 1e-12 against the
    # extended-precision oracle (T1), the run to 1e-9 against the fp64 oracle
    g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
    o = oracle.PWave(wl.nel, wl.p, wl.tau, wl.bc)
    if forced:
        bs = oracle.source_vectors(wl)
        g.set_source(bs, src.wavelet, src.f0, src.t0, src.amp)
        o.set_source(bs, src.wavelet, src.f0, src.t0, src.amp)
    u0 = oracle.project_separable(wl) if wl.u0 else np.zeros(o.shape)
    g.set_state(u0)
    o.set_state(u0)
    done = 0
    for n in (1, wl.steps):
        g.step(n - done)
        o.step(n - done)
        done = n
        ref = oracle.one_step_truth(wl, u0) if n == 1 else o.get_state()
        errs = [rel(x, y) for x, y in zip(g.get_state(), ref)]
        assert max(errs) < (STEP1_TOL if n == 1 else RUN_TOL), (n, errs)
    assert g.shape == (1, nel[1] + p, nel[0] + p)
    ge, oe = g.energy(), o.energy()
    assert np.allclose(ge, oe, rtol=1e-11, atol=1e-15)


def test_2d_modal_and_set_tau(ads):
    """The f3 / f4 entry points on a 2D handle: modal advance vs stepping, and a step-size change."""
    wl = _wl2d((30, 26, 0), 2, 5e-3, 50)
    a, b = ads.make_solver(wl), ads.make_solver(wl)
    a.modal_advance(50)
    b.step(50)
    for x, y in zip(a.get_state(), b.get_state()):
        assert rel(x, y) < 1e-11
    b.set_tau(2.5e-3)
    b.step(10)
    o = oracle.PWave(wl.nel, wl.p, 2.5e-3, wl.bc)
    u, ud, _ = a.get_state()
    o.set_state(u, ud)
    o.step(10)
    for x, y in zip(b.get_state(), o.get_state()):
        assert rel(x, y) < 1e-10


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_bitwise_deterministic(ads, cfg):
    """The path has no atomics or order-dependent reductions: two runs of the same seeded
    workload (graph replays, z-split launches, energies) agree bit for bit."""
    wl = workloads.get(cfg).scaled(24, 12)
    runs = []
    for _ in range(2):
        s = ads.make_solver(wl)
        s.step(wl.steps)
        runs.append((s.get_state(), s.energy()))
    (st0, e0), (st1, e1) = runs
    for a, b in zip(st0, st1):
        assert np.array_equal(a, b)
    assert np.array_equal(e0, e1)


def test_next_row_argument_errors(ads):
    """f2/f4 entry points reject what they do not support: 2D slabs, tau <= 0, scheme outside
    {0, 1}, tau changes on elasticity."""
    with pytest.raises(ads.AdsError):
        ads.Solver((8, 8, 0), 2, 1e-2, virtual_slabs=2)
    g = ads.Solver((8, 8, 8), 2, 1e-2)
    for bad in (0.0, -1e-3, float("nan")):
        with pytest.raises(ads.AdsError):
            g.set_tau(bad)
    with pytest.raises(ads.AdsError):
        g.set_scheme(2)
    e = ads.Solver((4, 4, 4), 2, 1e-2, elastic=True)
    with pytest.raises(ads.AdsError):
        e.set_tau(5e-3)


@pytest.mark.slow
def test_maximum_grid_properties(ads):
    """The largest supported grid (n_d = 1051 <= 1056 per direction, 1.16e9 DOFs, ~66 GB of
    fields): a few steps from a projected bump stay finite and keep the conserved invariant
    (C6) -- the oracle cannot run at this size, so parity here is a property."""
    import torch
    wl = workloads.get("c4")
    wl.nel = (1048, 1048, 1048)
    wl.u0 = wl.u0[:2]
    s = ads.make_solver(wl)
    e0 = s.energy()
    s.step(3)
    e1 = s.energy()
    assert np.all(np.isfinite(e1)) and e1[1] > 0
    assert abs(e1[2] - e0[2]) <= 1e-12 * abs(e0[2])
    u = torch.empty(s.shape, dtype=torch.float64, device="cuda")
    s.get_state(u, None, None)
    assert bool(torch.isfinite(u).all())
    s.close()
    del u
    torch.cuda.empty_cache()


@pytest.mark.parametrize("p,n", [(4, 600), (5, 600), (5, 865), (4, 590)])
def test_long_lines_high_degree_fit_shared_memory(ads, p, n):
    """p = 4, 5 lines of 577..865 rows (the 64 x 17 chunking's tables overflowed a CTA's
    shared memory there): the handle picks a chunking that fits and the sweeps along that axis
    match a dense solve, in x, y and z."""
    import torch
    for axis in range(3):
        nel = [3, 4, 5]
        nel[axis] = n - p
        s = ads.Solver(tuple(nel), p, 1e-3, 1)
        o = oracle.PWave(tuple(nel), p, 1e-3, 1)
        x = workloads.random_field(11 + axis, s.N).reshape(s.shape)
        xd = _dev(x)
        out = torch.empty_like(xd)
        s.solve_d(xd, out)
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), o.dsolve(x)) < OP_TOL, (p, n, axis)


def test_default_stream_ordering(ads):
    """With PyTorch's default stream (set_stream() / current_stream().cuda_stream == 0) the library
    works on its own blocking stream, ordered against the legacy default stream: device tensors
    written by PyTorch right before a call are seen, and outputs are complete for PyTorch right
    after it, with no explicit synchronisation."""
    import torch
    wl = workloads.get("c1")
    g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
    g.set_stream(torch.cuda.current_stream())
    u0 = oracle.project_separable(wl)
    big = torch.empty(1 << 26, dtype=torch.float64, device="cuda")
    for rep in range(3):
        ud = torch.zeros(g.shape, dtype=torch.float64, device="cuda")
        big.normal_()  # queue a long kernel on the default stream first
        ud.copy_(torch.from_numpy(u0).cuda(non_blocking=False) * (rep + 1))
        out = torch.empty_like(ud)
        g.apply_k(ud, out)
        out2 = out * 1.0  # consumed on the default stream immediately
        ref = oracle.PWave(wl.nel, wl.p, wl.tau, wl.bc).kapply(u0 * (rep + 1))
        assert rel(out2.cpu().numpy(), ref) < OP_TOL


def test_elastic_unit_ops_keep_state(ads):
    """Unit operators on a stepped elasticity handle leave its state alone (they used A,
    which holds a_n, as scratch): get_state and the energies are unchanged by them."""
    import torch
    wl = workloads.get("c5").scaled(8, 3)
    g = ads.make_solver(wl)
    g.step(3)
    st0, e0 = g.get_state(), g.energy()
    x = _dev(workloads.random_field(3, 3 * g.N).reshape(g.shape))
    out = torch.empty_like(x)
    g.apply_k(x, out)
    g.solve_d(x, out)
    torch.cuda.synchronize()
    st1, e1 = g.get_state(), g.energy()
    for a, b in zip(st0, st1):
        assert np.array_equal(a, b)
    assert np.array_equal(e0, e1)


def test_set_tau_releases_tables(ads):
    """Repeated ads_set_tau calls reuse device memory (each call leaked the old factor
    tables until destroy)."""
    import torch
    wl = workloads.get("c2").scaled(40, 0)
    g = ads.make_solver(wl)
    g.set_tau(wl.tau * 0.9)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for k in range(30):
        g.set_tau(wl.tau * (0.5 + 0.01 * k))
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 4 << 20, (free0 - free1)
