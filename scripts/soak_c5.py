"""Long run of the elasticity config c5: the E1 scheme's conserved invariant (C12)
before and after K steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
s = ads.make_solver(workloads.get("c5"))
e0 = s.energy()
t = time.perf_counter()
s.step(K)
torch.cuda.synchronize()
dt = time.perf_counter() - t
e1 = s.energy()
print(f"c5 {K} steps in {dt:.2f} s; energies before {e0}, after {e1}")
print(f"invariant relative change {abs(e1[2] - e0[2]) / abs(e0[2]):.2e}; kinetic + potential change "
      f"{abs(e1[0] + e1[1] - e0[0] - e0[1]) / abs(e0[0] + e0[1]):.2e}")
