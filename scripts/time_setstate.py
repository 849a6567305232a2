"""ads_set_state_separable time at a config (the library-side projection of the workload's terms)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

wl = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "c4")
s = ads.make_solver(wl)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    ads.make_solver.__wrapped__ if False else None
    terms = wl.u0
    sx = __import__("numpy").concatenate([ads.project_1d(s, t.f[0], 0) for t in terms])
    sy = __import__("numpy").concatenate([ads.project_1d(s, t.f[1], 1) for t in terms])
    sz = __import__("numpy").concatenate([ads.project_1d(s, t.f[2], 2) for t in terms])
    t1 = time.perf_counter()
    s.set_state_separable([t.amp for t in terms], sx, sy, sz, [t.comp for t in terms])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    # the start procedure alone: set_state from a device copy of the field (one D2D copy + start)
    print(f"{wl.name}: {len(terms)} terms: 1D projections {1e3 * (t1 - t0):.2f} ms, set_state_separable "
          f"(one pass + half-kick start) {1e3 * (t2 - t1):.2f} ms", flush=True)
ud = torch.zeros(tuple(reversed(s.n)), dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.set_state(ud)
    torch.cuda.synchronize()
    print(f"{wl.name}: set_state(device field) (D2D copy + half-kick start) {1e3 * (time.perf_counter() - t0):.2f} ms",
          flush=True)
