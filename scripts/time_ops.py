"""Per-kernel times of the step (library CUDA events, ads_profile_*) at several grid sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402

torch.cuda.set_device(0)
BYTES = np.array([32.0, 16.0, 16.0, 24.0])
for nel, p in [(127, 3), (255, 3), (512, 3), (256, 2)]:
    s = ads.Solver(nel, p, 5e-4)
    u = np.zeros(s.shape)
    u[1:-1, 1:-1, 1:-1] = np.random.default_rng(0).standard_normal(tuple(x - 2 for x in s.shape))
    s.set_state(u)
    s.step(3)
    s.profile_enable(True)
    s.step(10)
    ms, cnt = s.profile_read()
    s.profile_enable(False)
    per = ms / np.maximum(cnt, 1)
    gbs = BYTES * s.N / (per * 1e-3) / 1e9
    print(f"n={s.n[0]} p={p} N={s.N}", {k: f"{m:.3f}ms {g:.0f}GB/s" for k, m, g in
                                          zip(["kop", "sx", "sy", "sz+kick"], per, gbs)}, flush=True)
    s.close()
