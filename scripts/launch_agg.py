"""Aggregate the last N launches of an ncu launch list (gpu__time_duration.sum, dram bytes) by kernel:
python scripts/launch_agg.py launches.csv [N]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
d = collections.defaultdict(dict)
for r in rows[1:]:
    i = int(r[ix["ID"]])
    d[i][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]])
    d[i]["name"] = r[ix["Kernel Name"]].split("(")[0]
ids = sorted(d)[-n:] if n else sorted(d)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i in ids:
    m = d[i]
    a = agg[m["name"]]
    a[0] += 1
    a[1] += m["gpu__time_duration.sum"]
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"total {tot / 1e6:.3f} ms over {len(ids)} launches")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    gbs = a[2] / a[1] if a[1] else 0.0  # bytes / ns = GB/s
    print(f"{a[1] / 1e3:10.1f} us {a[1] / tot * 100:5.1f}%  x{a[0]:<3d} {a[1] / a[0] / 1e3:8.1f} us/launch  "
          f"DRAM {a[2] / a[0] / 1e9:.3f} GB/launch  {gbs:7.1f} GB/s  {k}")
