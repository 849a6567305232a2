"""Step time of a large 2D problem (ads_create nz = 0) with the library's per-kernel events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402

torch.cuda.set_device(0)
for nel, p in [((1024, 1024, 0), 3), ((1048, 1048, 0), 2)]:
    s = ads.Solver(nel, p, 1e-3)
    u = np.zeros(s.shape)
    u[:, 1:-1, 1:-1] = np.random.default_rng(0).standard_normal((1, s.shape[1] - 2, s.shape[2] - 2))
    s.set_state(u)
    s.step(3)
    s.profile_enable(True)
    s.step(20)
    ms, cnt = s.profile_read()
    s.profile_enable(False)
    per = ms / np.maximum(cnt, 1)
    print(nel, p, s.N, {k: f"{m * 1e3:.1f}us" for k, m in zip(["kop", "sx", "sy", "sz+kick"], per)}, flush=True)
