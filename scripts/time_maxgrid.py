"""Step time at the largest supported grid (1048^3 elements, p = 3: 1051^3 = 1.16e9 DOFs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

wl = workloads.get("c4")
wl.nel = (1048, 1048, 1048)
wl.u0 = wl.u0[:2]
s = ads.make_solver(wl)
st = torch.cuda.Stream()
s.set_stream(st)
s.step(3)
torch.cuda.synchronize()
K = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
s.step(K)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
N = 1051 ** 3
print(f"1048^3 elements, p=3: {N} DOFs, {ms:.2f} ms/step, {N / (ms * 1e-3):.3e} DOF-steps/s, "
      f"{88.0 * N / (ms * 1e-3) / 1e12:.2f} TB/s at 88 B/DOF")
s.profile_enable(True)
s.step(5)
kms, cnt = s.profile_read()
s.profile_enable(False)
per = kms / cnt.clip(min=1)
B = [32.0, 16.0, 16.0, 24.0]
print({k: f"{m:.2f} ms ({b * N / (m * 1e-3) / 1e12:.2f} TB/s)" for k, m, b in zip(["kop", "sx", "sy", "sz+kick"], per, B)})
