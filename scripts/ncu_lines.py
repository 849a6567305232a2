"""Per-source-line instruction and stall shares of one kernel in an ncu report.

    python scripts/ncu_lines.py report.ncu-rep kop4_kernelILi3 [N]

Joins ncu's SASS source page (instructions executed, stall samples per address) with the line table
of `nvdisasm -g` on the library's cubin (the report must come from the library built in-tree now).
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, sym, n=45):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1911_08158_b200", "libads_b200.so")],
                   cwd=tmp, capture_output=True)
    sass = ""
    for f in glob.glob(os.path.join(tmp, "*.cubin")):
        out = subprocess.run(["nvdisasm", "-g", "-c", f], capture_output=True, text=True).stdout
        if sym in out:
            sass = out
            break
    lines = sass.split("\n")
    st = [i for i, l in enumerate(lines) if l.startswith("//---") and sym in l][0]
    en = next((i for i, l in enumerate(lines[st + 1:], st + 1) if l.startswith("//---")), len(lines))
    cur, off2line = None, {}
    for l in lines[st:en]:
        m = re.search(r"## File .*line (\d+)", l)
        if m:
            cur = int(m.group(1))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    cnt, stall = collections.Counter(), collections.Counter()
    for r in data:
        ln = off2line.get(int(r[0], 16) - base)
        cnt[ln] += int(r[ix["Instructions Executed"]] or 0)
        stall[ln] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot, sst = sum(cnt.values()), max(1, sum(stall.values()))
    src = open(os.path.join(ROOT, "paper_1911_08158_b200", "csrc", "kernels.cu")).read().split("\n")
    print(f"{tot} warp instructions")
    for ln, v in sorted(cnt.items(), key=lambda x: -x[1])[:n]:
        print(f"{ln} {v / tot * 100:5.1f}% instr {stall[ln] / sst * 100:5.1f}% stall | "
              f"{src[ln - 1].strip()[:90] if ln else ''}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 45)
