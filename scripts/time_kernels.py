"""Per-kernel and per-step times of a config on one GPU (CUDA events): graph-replayed steps, then
a profiled run (ads_profile_enable: events around every launch, direct launches).
usage: python scripts/time_kernels.py [cfg ...]   (default c4)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

NAMES = ["kop", "sweep x", "sweep y", "sweep z+kick", "modal transform"]
for cfg in (sys.argv[1:] or ["c4"]):
    wl = workloads.get(cfg)
    s = ads.make_solver(wl)
    st = torch.cuda.Stream()
    s.set_stream(st)
    s.step(4)
    torch.cuda.synchronize()
    K = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for rep in range(3):
        e0.record(st)
        s.step(K)
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / K)
    s.profile_enable(True)
    s.step(K)
    torch.cuda.synchronize()
    ms, cnt = s.profile_read()
    s.profile_enable(False)
    N = wl.ndof
    line = f"{cfg}: step {best * 1e3:.1f} us ({N / (best * 1e-3):.3e} DOF-steps/s)"
    for i, nm in enumerate(NAMES):
        if cnt[i]:
            avg = ms[i] / cnt[i]
            line += f" | {nm} {avg * 1e3:.1f} us"
    print(line, flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
