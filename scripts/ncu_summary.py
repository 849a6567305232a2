"""Summarise an ncu report (or a launch-list CSV) into the tables kept under profiles/.

    python scripts/ncu_summary.py report.ncu-rep      # --set full capture: per-kernel table
    python scripts/ncu_summary.py launches.csv        # gpu__time_duration launch list
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print("| kernel | " + " | ".join(w[1] for w in WANT) + " | top stalls |")
    print("|---" * (len(WANT) + 2) + "|")
    for r in rows[2:]:
        cells = []
        for k, _ in WANT:
            i = hdr.index(k)
            cells.append(f"{r[i]} {units[i]}".strip())
        st = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), k[34:-23]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        name = r[hdr.index("Kernel Name")].split("(")[0]
        print(f"| {name} | " + " | ".join(cells) + " | " + ", ".join(f"{n} {v:.2f}" for v, n in st[:4]) + " |")


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(lines[start:]))
    print("id\tkernel\tgrid\tblock\tus")
    for r in rows:
        print(f"{r['ID']}\t{r['Kernel Name'].split('(')[0]}\t{r['Grid Size']}\t{r['Block Size']}\t"
              f"{float(r['Metric Value']) / 1e3:.1f}")


if __name__ == "__main__":
    p = sys.argv[1]
    rep(p) if p.endswith(".ncu-rep") else launches(p)
