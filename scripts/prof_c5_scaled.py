"""ncu driver: the c5 recipe at nel^3 elements (default 512), 2 warm-up steps, then one step with
direct launches (profiling on).  usage: python scripts/prof_c5_scaled.py [nel]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

nel = int(sys.argv[1]) if len(sys.argv) > 1 else 512
s = ads.make_solver(workloads.get("c5").scaled(nel))
s.step(2)
torch.cuda.synchronize()
s.profile_enable(True)
s.step(1)
torch.cuda.synchronize()
print("ok")
