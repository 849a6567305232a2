"""Long run at full size: config c4 (F = 0) for K steps by stepping, the conserved invariant
(C6) before/after, and the state against the modal propagator (an independent path:
eigenbasis transforms instead of K P and sweeps) after the same K steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
wl = workloads.get("c4")
s = ads.make_solver(wl)
e0 = s.energy()
t = time.perf_counter()
s.step(K)
torch.cuda.synchronize()
dt = time.perf_counter() - t
e1 = s.energy()
print(f"c4 {K} steps in {dt:.2f} s ({K / dt:.0f} steps/s); energies before {e0}, after {e1}")
print(f"invariant relative change {abs(e1[2] - e0[2]) / abs(e0[2]):.2e}; kinetic + potential change "
      f"{abs(e1[0] + e1[1] - e0[0] - e0[1]) / abs(e0[0] + e0[1]):.2e}")
m = ads.make_solver(wl)
m.modal_advance(K)
for name, x, y in zip(("u", "udot", "a"), s.get_state(), m.get_state()):
    print(f"stepping vs modal after {K} steps: rel L2 {name} {np.linalg.norm(x - y) / np.linalg.norm(y):.2e}")
