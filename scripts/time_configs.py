"""Step time and throughput of every BASELINE.json config (c1..c5) on one GPU through the public
API (make_solver + step, graph replay), CUDA events on the library stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

for name in ["c1", "c2", "c3", "c4", "c5"]:
    wl = workloads.get(name)
    s = ads.make_solver(wl)
    st = torch.cuda.Stream()
    s.set_stream(st)
    s.step(5)
    torch.cuda.synchronize()
    K = wl.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.step(K)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"{name}: {wl.ndof:>11d} DOFs, {K} steps: {ms * 1e3:8.1f} us/step, {wl.ndof / (ms * 1e-3):.3e} DOF-steps/s, "
          f"run {ms * K:.1f} ms", flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
