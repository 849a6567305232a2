"""Run one P-wave step per (p, shape) in a fresh process and report CUDA errors (debug aid)."""
import subprocess
import sys

CHILD = r'''
import sys, numpy as np, torch, paper_1911_08158_b200 as ads
p = int(sys.argv[1]); nel = tuple(int(x) for x in sys.argv[2].split(","))
s = ads.Solver(nel, p, 1e-3)
u = np.zeros(s.shape); u[1:-1, 1:-1, 1:-1] = 1.0
s.set_state(u); s.step(2); print("ok", s.energy())
'''
for p in [1, 2, 3, 4, 5]:
    for nel in ["6,13,5", "32,32,32", "64,64,64"]:
        r = subprocess.run([sys.executable, "-c", CHILD, str(p), nel], capture_output=True, text=True,
                           env=dict(__import__("os").environ, CUDA_LAUNCH_BLOCKING="1"))
        print(p, nel, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:160], flush=True)
