"""Modal propagator (ads_modal_advance) vs stepping at config c4 (515^3):
wall time of one advance by K steps for several K, the transforms' FP64 rate, and agreement with
stepping after 100 steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl = workloads.get(cfg)
s = ads.make_solver(wl)
st = torch.cuda.Stream()
s.set_stream(st)
t0 = time.perf_counter()
s.modal_advance(1)  # builds the bases (host) and the cuBLAS handle
torch.cuda.synchronize()
print(f"{cfg}: first advance (bases + transforms) {time.perf_counter() - t0:.2f} s", flush=True)
n0, n1, n2 = s.n
g = s.geo if hasattr(s, "geo") else None
sy = (n0 + 7) // 8 * 8
flops_transform = 2.0 * (n0 * n0 * n1 * n2 + n1 * n1 * n0 * n2 + n2 * n2 * sy * n1)
for K in [1, 100, 10000]:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.modal_advance(K)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # 4 transforms (U, V in; U, V out) + the operator kernel and three sweeps for a
    print(f"modal_advance({K}): {ms:.2f} ms, {4 * flops_transform / (ms * 1e-3) / 1e12:.1f} TFLOP/s dense-equivalent "
          f"(4 x {flops_transform / 1e9:.0f} GFLOP unfolded; the folded products do half)", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
s.step(100)
e1.record(st)
torch.cuda.synchronize()
print(f"step(100): {e0.elapsed_time(e1):.2f} ms", flush=True)
# agreement after 100 steps from the workload's initial state
a = ads.make_solver(wl)
a.modal_advance(100)
b = ads.make_solver(wl)
b.step(100)
for name, x, y in zip(("u", "udot", "a"), a.get_state(), b.get_state()):
    print(f"modal vs stepping after 100 steps: rel L2 {name} {np.linalg.norm(x - y) / np.linalg.norm(y):.2e}")
