"""Step time of small configs with and without CUDA-graph replays (ads_step pairs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

for cfg in ["c1", "c2"]:
    wl = workloads.get(cfg)
    s = ads.make_solver(wl)
    for mode in ["graph", "direct"]:
        s.profile_enable(mode == "direct")  # profiling forces direct launches
        s.step(4)
        torch.cuda.synchronize()
        t = time.perf_counter()
        s.step(201)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 201
        print(cfg, mode, f"{dt * 1e6:.1f} us/step", s.launch_count(), flush=True)
    s.profile_enable(False)
