"""Step time of config c5 (3D elasticity, 130^3 x 3 DOFs) with the library's CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

wl = workloads.get("c5")
s = ads.make_solver(wl)
st = torch.cuda.Stream()
s.set_stream(st)
s.step(3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n0 = s.launch_count()
e0.record(st)
s.step(20)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"c5: {ms:.3f} ms/step, {wl.ndof / (ms / 1e3):.3e} DOF-steps/s, {(s.launch_count() - n0) / 20:.0f} launches/step")
print("energy", s.energy())
