"""Minimal driver for ncu: build config `cfg`, set_state, run `steps` steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = workloads.get(cfg)
s = ads.make_solver(wl)
s.step(steps)
torch.cuda.synchronize()
print("ok", cfg, steps, s.energy())
