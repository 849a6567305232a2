"""ncu driver: config c4 as G virtual slabs (default 2), warm-up, then 1 profiled step."""
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
s.step(1)
torch.cuda.synchronize()
print("ok")
