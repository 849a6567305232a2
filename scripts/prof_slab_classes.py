"""Per kernel class ms/step of c4 on G virtual slabs (library events around every launch, summed
over the slabs): kop, sweep x, sweep y, z (slab z blocks + SPIKE stage 1/2 + kick).
usage: python scripts/prof_slab_classes.py [G ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

wl = workloads.get("c4")
for G in [int(v) for v in sys.argv[1:]] or [2, 8]:
    s = ads.make_solver(wl, virtual_slabs=G)
    s.step(2)
    torch.cuda.synchronize()
    s.profile_enable(True)
    s.step(4)
    torch.cuda.synchronize()
    ms, cnt = s.profile_read()
    print(f"c4 slabs={G}: per step kop {ms[0] / 4:.3f} ms, sweep x {ms[1] / 4:.3f}, sweep y {ms[2] / 4:.3f}, "
          f"z blocks + SPIKE + kick {ms[3] / 4:.3f} (launches per step {list(cnt[:4] // 4)})", flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
