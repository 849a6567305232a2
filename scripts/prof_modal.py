"""ncu driver: one modal_advance(100) at config c4 after a warm-up call (bases built)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

s = ads.make_solver(workloads.get(sys.argv[1] if len(sys.argv) > 1 else "c4"))
s.modal_advance(1)
torch.cuda.synchronize()
s.modal_advance(100)
torch.cuda.synchronize()
print("ok")
