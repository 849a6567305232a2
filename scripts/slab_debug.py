"""Compare single-GPU, virtual-slab (G = 1, 2, 3) and oracle results on one grid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


wl = workloads.get("c4").scaled(16, 1)
wl.nel = (19, 16, 150)
u0 = oracle.project_separable(wl)
o = oracle.make_solver(wl)
ou0, oud0, oa0 = o.get_state()
o.step(1)
ou, oud, oa = o.get_state()
for G in [0, 1, 2, 3]:
    s = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc, virtual_slabs=G)
    s.set_state(u0)
    gu0, gud0, ga0 = s.get_state()
    s.step(1)
    gu, gud, ga = s.get_state()
    print(G, "init a0 %.2e" % rel(ga0, oa0), "step: u %.2e udot %.2e a %.2e" % (rel(gu, ou), rel(gud, oud), rel(ga, oa)))
    if G:
        d = np.abs(ga0 - oa0).max(axis=(1, 2))
        print("   per-plane max |a0 err| (z):", " ".join("%.1e" % x for x in d[::6]))
