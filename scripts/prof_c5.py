"""ncu driver: config c5 (elasticity), warm-up, then 2 steps with direct launches (profiling on)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

s = ads.make_solver(workloads.get("c5"))
s.step(2)
torch.cuda.synchronize()
s.profile_enable(True)  # direct launches: one ncu record per kernel
s.step(1)
torch.cuda.synchronize()
print("ok")
