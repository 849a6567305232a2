"""z sweep + kick time with and without a kept (the last step of every ads_step batch stores a)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

wl = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "c4")
s = ads.make_solver(wl)
st = torch.cuda.Stream()
s.set_stream(st)
s.step(3)
for batch in (1, 20):
    s.profile_enable(True)
    for _ in range(20 // batch):
        s.step(batch)
    ms, cnt = s.profile_read()
    s.profile_enable(False)
    print(f"batches of {batch}: z sweep + kick {1e3 * ms[3] / cnt[3]:.1f} us per launch over {cnt[3]} launches "
          f"({20 // batch} with a kept)", flush=True)
