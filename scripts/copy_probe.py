"""Host<->device copy rates on this box: contiguous pinned copies vs the pitched 2D copies the
state I/O uses (1.09 GB field of config c4)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402

n = 515
N = n ** 3
h = torch.empty(N, dtype=torch.float64, pin_memory=True).uniform_()
d = torch.empty(N, dtype=torch.float64, device="cuda")
for name, fn in [("H2D contiguous", lambda: d.copy_(h, non_blocking=True)),
                 ("D2H contiguous", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {N * 8 / dt / 1e9:.1f} GB/s", flush=True)
s = ads.Solver(512, 3, 5e-4)
u = h.view(n, n, n)
for name, fn in [("set_state(u) 2D copy + init", lambda: s.set_state(u)),
                 ("get_state(u) 2D copy", lambda: s.get_state(u, None, None))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"{name}: {dt * 1e3:.1f} ms ({N * 8 / dt / 1e9:.1f} GB/s per field)", flush=True)
