"""Probe of the modal transforms on grids with one long axis (isolates a direction / size)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

for nel in [(512, 16, 16), (16, 512, 16), (16, 16, 512), (254, 40, 40), (256, 40, 40), (300, 20, 20)]:
    s = ads.Solver(nel, 3, 5e-4)
    u = workloads.random_field(3, s.N).reshape(s.shape)
    u[0], u[-1], u[:, 0], u[:, -1], u[:, :, 0], u[:, :, -1] = 0, 0, 0, 0, 0, 0
    s.set_state(u)
    try:
        s.modal_advance(3)
        torch.cuda.synchronize()
        b = ads.Solver(nel, 3, 5e-4)
        b.set_state(u)
        b.step(3)
        x, y = s.get_state()[0], b.get_state()[0]
        print(nel, "ok", np.linalg.norm(x - y) / np.linalg.norm(y), flush=True)
    except Exception as e:
        print(nel, "FAIL", str(e)[:200], flush=True)
        break
