"""kop time per launch vs the z split (ADS_KOP_NZ) for library variants (experiment driver).

    python scripts/kop_nz.py lib1.so lib2.so ...
"""
import os
import subprocess
import sys

CHILD = r'''
import numpy as np, torch, paper_1911_08158_b200 as ads
torch.cuda.set_device(0)
s = ads.Solver(512, 3, 5e-4)
u = np.zeros(s.shape)
u[1:-1, 1:-1, 1:-1] = np.random.default_rng(0).standard_normal(tuple(x - 2 for x in s.shape))
s.set_state(u); s.step(3); s.profile_enable(True); s.step(20)
ms, cnt = s.profile_read()
per = ms / np.maximum(cnt, 1)
print("%.3f %.3f %.3f %.3f" % tuple(per))
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for lib in sys.argv[1:]:
    for nz in [0, 1, 2, 3, 4, 6, 8, 12]:
        env = dict(os.environ, ADS_B200_LIB=os.path.abspath(lib), ADS_KOP_NZ=str(nz))
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, cwd=root, capture_output=True, text=True)
        print(os.path.basename(lib), "nz", nz, r.stdout.strip() or r.stderr[-300:], flush=True)
