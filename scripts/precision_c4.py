"""One step of config c4 (515^3) on the GPU against the extended-precision oracle (the truth of
north_star's one-step 1e-12 bound, T1), with the fp64 C oracle's own distance to that
truth for scale.  Relative L2 on U, udot and a."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl = workloads.get(cfg)
t0 = time.time()
u0 = oracle.project_separable(wl)
g = ads.make_solver(wl, u0=u0)
g.step(1)
gs = g.get_state()
g.close()
t1 = time.time()
truth = oracle.one_step_truth(wl, u0)
t2 = time.time()
print(f"{cfg}: GPU vs extended-precision oracle after one step: u {rel(gs[0], truth[0]):.2e}  "
      f"udot {rel(gs[1], truth[1]):.2e}  a {rel(gs[2], truth[2]):.2e}  (LD oracle {t2 - t1:.0f} s)", flush=True)
o = oracle.make_solver(wl, u0=u0)
o.step(1)
os_ = o.get_state()
del o
print(f"{cfg}: fp64 C oracle vs extended-precision oracle:      u {rel(os_[0], truth[0]):.2e}  "
      f"udot {rel(os_[1], truth[1]):.2e}  a {rel(os_[2], truth[2]):.2e}", flush=True)
