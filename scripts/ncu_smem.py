"""Shared-memory wavefronts (and the excess over ideal, i.e. bank conflicts) per source line of a
kernel in an ncu report: python scripts/ncu_smem.py report.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if "Source" in r and "L1 Wavefronts Shared" in r)
ix = {h: i for i, h in enumerate(hdr)}
tot = collections.Counter()
exc = collections.Counter()
allw = 0.0
for r in rows:
    if len(r) != len(hdr) or r is hdr:
        continue
    try:
        wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
        ex = float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
    except ValueError:
        continue
    key = r[ix["Source"]].strip()[:90]
    tot[key] += wf
    exc[key] += ex
    allw += wf
print(f"total shared wavefronts {allw:.4g}, excessive {sum(exc.values()):.4g}")
for k, v in tot.most_common(n):
    print(f"{v / allw * 100:5.1f}%  excess {exc[k] / max(v, 1) * 100:5.1f}%  {k}")
