"""Per-launch DRAM traffic of the step kernels from one `ncu --set full` capture.

    python scripts/ncu_traffic.py report.ncu-rep out.json

Writes {"source": report, "kernels": {name: {"dram_bytes": read + write, "duration_ms": ...}}}
with name in kop / sweep_x / sweep_y / sweep_z_kick (capture order of one step); bench.py copies
the dominant kernel's figure into roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TUNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(hdr)}
    res, sweeps = {}, 0
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        rd = float(r[col["dram__bytes_read.sum"]]) * UNIT[units[col["dram__bytes_read.sum"]]]
        wr = float(r[col["dram__bytes_write.sum"]]) * UNIT[units[col["dram__bytes_write.sum"]]]
        t = float(r[col["gpu__time_duration.sum"]]) * TUNIT[units[col["gpu__time_duration.sum"]]]
        if "kop_kernel" in name or "kop4_kernel" in name:
            key = "kop"
        elif "sweep_kernel" in name:
            key = ["sweep_x", "sweep_y", "sweep_z_kick"][min(sweeps, 2)]
            sweeps += 1
        else:
            continue
        res[key] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "duration_ms": t,
                    "kernel": name}
    json.dump({"source": rep.split("/")[-1], "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
