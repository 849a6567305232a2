"""GPU parity of the z-slab (multi-GPU) algorithm, run on one GPU as a virtual group
(SURVEY.md §8 row e): every slab of the grid on this device, halos and SPIKE
tips exchanged by device copies, the same kernels the NCCL path launches per rank.

Compared with the CPU oracle (the sequential split scheme) on U, udot and a: relative L2
<= 1e-12 after one step and <= 1e-9 after the run.  Slabs must be thick enough for the
certified SPIKE truncation (the spike coupling across a slab < 2^-64).
"""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def ads():
    import torch
    import paper_1911_08158_b200 as ads
    from paper_1911_08158_b200 import build
    build.build()
    assert torch.cuda.is_available()
    return ads


def _run(ads, wl, nslabs, checkpoints, zsolve=0):
    # both sides start from the same coefficients (the oracle's projection); the source load
    # vectors are formed independently.  One step is held to 1e-12 against the extended-precision
    # oracle (T1), later checkpoints to 1e-9 against the fp64 oracle.
    u0 = oracle.project_separable(wl)
    g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc, virtual_slabs=nslabs)
    if zsolve:
        g.set_zsolve(zsolve)
    if wl.source is not None:
        src = wl.source
        g.set_source([g.load_vector(d, src.f[d]) for d in range(3)], src.wavelet, src.f0, src.t0, src.amp)
    g.set_state(u0)
    o = oracle.make_solver(wl, u0=u0)
    done = 0
    for nsteps in checkpoints:
        g.step(nsteps - done)
        o.step(nsteps - done)
        done = nsteps
        ref = oracle.one_step_truth(wl, u0) if nsteps == 1 else o.get_state()
        tol = 1e-12 if nsteps == 1 else 1e-9
        errs = tuple(rel(x, y) for x, y in zip(g.get_state(), ref))
        assert max(errs) < tol, (wl.name, nslabs, nsteps, errs)
    return g, o


@pytest.mark.parametrize("nslabs", [2, 3])
def test_virtual_slabs_c4_recipe(ads, nslabs):
    """c4 recipe (p = 3, 8 bumps) on a grid long in z (slabs >= 70 planes), 30 steps."""
    wl = workloads.get("c4").scaled(16, 30)
    wl.nel = (19, 16, 75 * nslabs)
    g, o = _run(ads, wl, nslabs, [1, 30])
    ge, oe = g.energy(), o.energy()
    assert np.allclose(ge, oe, rtol=1e-11), (ge, oe)


@pytest.mark.parametrize("nslabs,nz", [(4, 256), (8, 513)])
def test_virtual_slabs_thin_refined(ads, nslabs, nz):
    """Slabs of ~64 planes (c4 at 8 GPUs): the interface systems need their one-step
    refinement with the neighbours' stage-1 values (certified (|Q| p d)^2 < 2^-64)."""
    wl = workloads.get("c4").scaled(8, 12)
    wl.nel = (9, 8, nz)
    _run(ads, wl, nslabs, [1, 12])


def test_virtual_slabs_forced_p2(ads):
    """c3 recipe (p = 2, Ricker x Gaussian source, zero state): 4 slabs of 58 planes and
    8 slabs of 32 planes (c3 at 8 GPUs)."""
    wl = workloads.get("c3").scaled(12, 60)
    wl.nel = (12, 14, 230)
    _run(ads, wl, 4, [1, 60])
    wl.nel = (10, 9, 254)
    _run(ads, wl, 8, [1, 60])


def test_virtual_slabs_natural_bc(ads):
    wl = workloads.get("c2").scaled(10, 20)
    wl.nel = (10, 9, 160)
    wl.bc = 0
    _run(ads, wl, 2, [1, 20])


def test_virtual_slabs_match_single_gpu(ads):
    """The slab algorithm reproduces the single-GPU path (same kernels, exact SPIKE) to rounding
    (amplified like T1 by the K P cancellation in a, udot: bound 1e-11 after 10 steps)."""
    wl = workloads.get("c4").scaled(16, 10)
    wl.nel = (21, 18, 150)
    u0 = oracle.project_separable(wl)
    ref = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
    ref.set_state(u0)
    ref.step(10)
    for G in (1, 2):
        g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc, virtual_slabs=G)
        g.set_state(u0)
        g.step(10)
        for x, y in zip(g.get_state(), ref.get_state()):
            assert rel(x, y) < 1e-11, G
        assert np.allclose(g.energy(), ref.energy(), rtol=1e-12)


def test_thin_slabs_rejected(ads):
    """Slabs too thin for the certified truncation are refused (ADS_E_INVAL), not approximated."""
    with pytest.raises(ads.AdsError) as e:
        ads.Solver((8, 8, 40), 3, 5e-4, virtual_slabs=4)
    assert e.value.code == -1


def test_nccl_slab_world1(ads):
    """The NCCL slab handle (ads_create_dist, communicator of one rank) runs the slab path with
    an NCCL all-reduce for the energies and matches the single-GPU handle (one GPU in this
    harness: multi-rank NCCL runs need one GPU per rank)."""
    wl = workloads.get("c2").scaled(12, 8)
    u0 = oracle.project_separable(wl)
    ref = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
    ref.set_state(u0)
    ref.step(8)
    g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc, dist=(0, 1, ads.get_unique_id()))
    assert (g.z_begin, g.z_count) == (0, wl.nel[2] + wl.p)
    g.set_state(u0)
    g.step(8)
    for x, y in zip(g.get_state(), ref.get_state()):
        assert rel(x, y) < 1e-13
    assert np.allclose(g.energy(), ref.energy(), rtol=1e-13)


def test_virtual_group_set_stream(ads):
    """A virtual slab group moves all its slabs to a caller stream (and back to its own) and
    keeps stepping: results match the same run on the default stream."""
    import torch
    wl = workloads.get("c3").scaled(40, 8)
    g = ads.make_solver(wl, virtual_slabs=2)
    st = torch.cuda.Stream()
    g.set_stream(st)
    g.step(4)
    g.set_stream(None)
    g.step(4)
    r = ads.make_solver(wl, virtual_slabs=2)
    r.step(8)
    for a, b in zip(g.get_state(), r.get_state()):
        assert np.array_equal(a, b)


# ---- all-to-all z solve (ads_set_zsolve(h, ADS_ZSOLVE_ALLTOALL), north_star's alternative) ----

@pytest.mark.parametrize("nslabs,nz", [(2, 150), (3, 225), (8, 513)])
def test_alltoall_virtual_vs_oracle(ads, nslabs, nz):
    """The transpose path (y blocks gathered into full-z pencils, single-GPU A_z factors, returned
    for the kick) against the oracle: 1e-12 after one step (extended-precision truth), 1e-9 after
    the run; y extents that split unevenly (19 / 3, 21 / 8)."""
    wl = workloads.get("c4").scaled(12, 12)
    wl.nel = (17, 16 if nslabs == 3 else 18, nz)
    _run(ads, wl, nslabs, [1, 12], zsolve=1)


def test_alltoall_forced_p2_and_natural(ads):
    wl = workloads.get("c3").scaled(12, 40)
    wl.nel = (12, 14, 230)
    _run(ads, wl, 4, [1, 40], zsolve=1)
    wl = workloads.get("c2").scaled(10, 20)
    wl.nel = (10, 9, 160)
    wl.bc = 0
    _run(ads, wl, 2, [1, 20], zsolve=1)


def test_alltoall_matches_spike_and_switches(ads):
    """Both z solves give the same state to rounding; a run may switch between them."""
    wl = workloads.get("c4").scaled(16, 10)
    wl.nel = (21, 18, 300)
    a = ads.make_solver(wl, virtual_slabs=4, zsolve=1)
    b = ads.make_solver(wl, virtual_slabs=4)
    a.step(6)
    b.step(6)
    for x, y in zip(a.get_state(), b.get_state()):
        assert rel(x, y) < 1e-12
    a.set_zsolve(0)
    b.set_zsolve(1)
    a.step(4)
    b.step(4)
    for x, y in zip(a.get_state(), b.get_state()):
        assert rel(x, y) < 1e-12
    assert np.allclose(a.energy(), b.energy(), rtol=1e-12)


def test_alltoall_nccl_world1(ads):
    """NCCL slab handle (one rank) on the all-to-all path: local transposes only."""
    wl = workloads.get("c2").scaled(12, 8)
    u0 = oracle.project_separable(wl)
    ref = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
    ref.set_state(u0)
    ref.step(8)
    g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc, dist=(0, 1, ads.get_unique_id()))
    g.set_zsolve(1)
    g.set_state(u0)
    g.step(8)
    for x, y in zip(g.get_state(), ref.get_state()):
        assert rel(x, y) < 1e-13
    assert np.allclose(g.energy(), ref.energy(), rtol=1e-13)


def test_alltoall_errors(ads):
    s = ads.Solver((8, 8, 8), 2, 1e-3)
    with pytest.raises(ads.AdsError):
        s.set_zsolve(1)  # not a slab handle
    g = ads.Solver((8, 8, 100), 2, 1e-3, virtual_slabs=2)
    with pytest.raises(ads.AdsError):
        g.set_zsolve(2)
    g2 = ads.Solver((3, 2, 254), 2, 1e-3, virtual_slabs=8)  # 4 y rows < 8 slabs
    with pytest.raises(ads.AdsError):
        g2.set_zsolve(1)
