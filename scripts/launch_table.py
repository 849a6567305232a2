"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name:
python scripts/launch_table.py launches.csv [skip_first_n]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot, cnt = collections.Counter(), collections.Counter()
seen = set()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    key = (r[ix["ID"]])
    if key in seen:
        continue
    seen.add(key)
    if int(r[ix["ID"]]) < skip:
        continue
    name = r[ix["Kernel Name"]].split("(")[0][:60]
    v = float(r[ix["Metric Value"]])
    unit = r[ix["Metric Unit"]]
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
for k, v in tot.most_common():
    print(f"{v:9.1f} us {v / T * 100:5.1f}%  x{cnt[k]:<4d} {k}")
