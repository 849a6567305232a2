"""Config c5's recipe (3D elasticity, lambda = mu = rho = 1, p = 2, one seeded Gaussian bump per
component, zero Dirichlet, tau = 1e-3) scaled to 256^3 and 512^3 elements (SURVEY.md §8(f) f1:
"c5 scaled to 256^3/512^3").  Per grid: ms/step over graph-replayed steps (library CUDA events),
DOF-steps/s, the step's fraction of HBM on SURVEY §8(d)'s 176 B per vector DOF, launches per
step, and the E1 invariant over the run.  At 256^3 one step is also compared element by element
with the extended-precision oracle (T1; north_star 1e-12).
usage: python scripts/time_elastic_scaled.py [nel ...]   (default 128 256 512)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6533.5
BYTES = 176.0
PLAN = 264.0  # the step as built


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


for nel in [int(v) for v in sys.argv[1:]] or [128, 256, 512]:
    wl = workloads.get("c5").scaled(nel, 100)
    t0 = time.time()
    s = ads.make_solver(wl)
    t_setup = time.time() - t0
    st = torch.cuda.Stream()
    s.set_stream(st)
    e_start = s.energy()
    s.step(3)
    torch.cuda.synchronize()
    K = 20 if nel <= 256 else 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for rep in range(3):
        n0 = s.launch_count()
        e0.record(st)
        s.step(K)
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / K)
        lps = (s.launch_count() - n0) / K
    e_end = s.energy()
    nsteps = 3 + 3 * K
    dof = wl.ndof
    frac = BYTES * dof / (best * 1e-3) / 1e9 / PEAK
    pfrac = PLAN * dof / (best * 1e-3) / 1e9 / PEAK
    drift = abs(e_end[2] - e_start[2]) / e_start[2]
    print(f"c5@{nel}: {dof} DOFs ({dof // 3} per component), setup {t_setup:.1f} s, {best:.3f} ms/step, "
          f"{dof / (best * 1e-3):.3e} DOF-steps/s, {frac:.3f} of HBM on {BYTES:.0f} B/DOF ({PEAK} GB/s), "
          f"{pfrac:.3f} on the {PLAN:.0f} B/DOF the step moves, "
          f"{lps:.0f} launches/step; invariant over {nsteps} steps: {e_start[2]:.12e} -> {e_end[2]:.12e} "
          f"(rel {drift:.2e})", flush=True)
    del s
    torch.cuda.empty_cache()
    if nel == 256:
        import oracle
        u0 = oracle.project_separable(wl)
        g = ads.make_solver(wl, u0=u0)
        g.step(1)
        gs = g.get_state()
        del g
        torch.cuda.empty_cache()
        t0 = time.time()
        ref = oracle.one_step_truth(wl, u0)
        errs = tuple(rel(x, y) for x, y in zip(gs, ref))
        print(f"c5@{nel}: one step vs the extended-precision oracle ({time.time() - t0:.0f} s): rel L2 "
              f"u {errs[0]:.2e}, udot {errs[1]:.2e}, a {errs[2]:.2e} (north_star 1e-12)", flush=True)
