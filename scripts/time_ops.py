"""Time the unit operators (kop via apply_k, each sweep) at several grid sizes with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402

torch.cuda.set_device(0)
for nel, p in [(127, 3), (255, 3), (512, 3), (256, 2)]:
    s = ads.Solver(nel, p, 5e-4)
    st = torch.cuda.Stream()
    s.set_stream(st)
    x = torch.rand(s.shape, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    N = s.N
    res = {}
    with torch.cuda.stream(st):
        for name, fn in [("kop", lambda: s.apply_k(x, y)), ("sx", lambda: s.sweep(0, x, y)),
                         ("sy", lambda: s.sweep(1, x, y)), ("sz", lambda: s.sweep(2, x, y))]:
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10):
                fn()
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            byt = (32 if name == "kop" else 16) * N  # kop via apply_k: reads x twice (U=V=x), writes r
            res[name] = f"{ms:.3f}ms {ms * 1e6 / N * 1e3:.2f}ps/dof {(24 if name == 'kop' else 16) * N / ms / 1e6:.0f}GB/s"
    print(f"n={s.n[0]} p={p} N={N}", res, flush=True)
    s.close()
