"""Cost of the z-slab algorithm (row e) on one GPU: config c4 as G virtual slabs (all slabs on this
device, exchanges by device copies, the distributed kernels: halo exchange, slab sweeps, SPIKE
stage 1/2 with tip exchanges).  Total ms/step of all slabs vs the single-GPU step; per-kernel
times from an ncu-free CUDA-event loop over ads_step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

wl = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "c4")
for G, zs in [(0, 0), (2, 0), (4, 0), (8, 0), (2, 1), (4, 1), (8, 1)]:
    s = ads.make_solver(wl, virtual_slabs=G, zsolve=zs)
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
    print(f"{wl.name} slabs={G or 1}{' (single-GPU path)' if not G else ''}{' all-to-all' if zs else ''}: {ms:.3f} ms/step "
          f"(all slabs on one GPU), {(s.launch_count() - n0) / 20:.0f} launches/step", flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
