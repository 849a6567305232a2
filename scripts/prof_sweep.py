"""One sweep launch per direction on an n^3 grid (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402

nel = int(sys.argv[1]) if len(sys.argv) > 1 else 127
p = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = ads.Solver(nel, p, 5e-4)
x = torch.rand(s.shape, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for d in range(3):
    s.sweep(d, x, y)
s.apply_k(x, y)
torch.cuda.synchronize()
print("ok")
