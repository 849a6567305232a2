"""ncu driver: c4 on G virtual slabs, 2 warm-up steps, then 1 step with direct launches (profiling on).
usage: python scripts/prof_slab_step.py G"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = ads.make_solver(workloads.get("c4"), virtual_slabs=G)
s.step(2)
torch.cuda.synchronize()
s.profile_enable(True)
s.step(2)
torch.cuda.synchronize()
print("ok")
