"""bench.py contract checks that need no GPU: the reference arm (the oracle)
prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--ref-nel", "12"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ["impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"]:
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_roofline_traffic_comes_from_the_committed_capture():
    """roofline.traffic = ncu dram read + write of the dominant kernel from the latest committed
    profiles/r*_traffic.json, only for the workload it was captured on (c4, 515^3 DOFs)."""
    import glob
    import importlib.util
    import json
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")),
                   key=lambda f: tuple(int(x) for x in re.findall(r"\d+", os.path.basename(f))))
    assert files, "no committed traffic capture"
    ref = json.load(open(files[-1]))["kernels"]["kop"]["dram_bytes"] / 1e9
    got, src = bench.ncu_traffic("kop", 515 ** 3)
    assert got == ref and src == os.path.basename(files[-1])
    assert 4.37 <= got <= 1.5 * 4.37  # at least the algorithmic bytes of one launch
    assert bench.ncu_traffic("kop", 1000) == (None, None)
