#!/usr/bin/env python
"""Benchmark of the ADS wave step (arXiv:1911.08158 hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Workload: BASELINE.json configs[3] (c4: p=3, 512^3 elements, 515^3 = 136.6M DOFs,
tau 5e-4, 8 seeded Gaussian bumps) -- the 512^3 case the north_star's targets
name.  One "step" = one full time step of the hot path (drift+source+K apply,
x/y/z partitioned banded sweeps, fused kick).  Metric: DOF-steps/s (fp64).

Timing: W untimed warm-up steps; then 5 repeats, each restarting from the initial state and
timing exactly K steps bracketed by a barrier + torch.cuda.synchronize() on both sides, CUDA
events on the library's stream, max over ranks; the median repeat is reported (graph-replayed
steps: the production launch path).  A separate profiled run gives the per-kernel times.  Every field (1.09 GB) is larger than L2 (126 MB), so no L2
flush is needed.  Per-kernel CUDA-event timing inside the library
(ads_profile_*) gives the roofline of the dominant kernel.

N > 1 (torchrun): the c4 grid is cut into N z-slabs, one per GPU (ads_create_dist: NCCL
halo and SPIKE-tip exchanges over NVLink), reported as strong scaling: `value` is the
whole-grid DOF-steps/s over the max-over-ranks time.

--impl reference: the CPU oracle (oracle/, single thread) on a bounded sample
of the same workload recipe; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import re
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "P-wave DOF-steps/sec (fp64)"
UNIT = "DOF-steps/s"
FALLBACK_HBM_GBS = 6650.0
# algorithmic HBM bytes per DOF for one launch of each kernel class:
#   reported by the library (ads_step_bytes): kop 32 (U, V -> P, r), sweeps x, y 16 each,
#   sweep z + kick 24 (+8 B for a on the last step of a batch)
KERNELS = ["kop", "sweep_x", "sweep_y", "sweep_z_kick"]
C4_DOFS = 515 ** 3  # the committed traffic captures are of config c4 on one GPU
ELASTIC_STEP_BYTES = 176.0  # elasticity bytes per vector DOF and step (estimate)
# the elastic step as built, per DOF: diagonal blocks 32, coupling pairs 2 x 24,
# six ADS solves 2 x 3 x 16, predictor/corrector couplings 2 x 24, rho M 16, kick 24
ELASTIC_PLAN_BYTES = 264.0


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return FALLBACK_HBM_GBS, "fallback", {}


def ncu_traffic(kernel, n_dof):
    """DRAM bytes per launch of `kernel` from the latest committed `--set full` capture
    (profiles/r*_traffic.json, written by scripts/ncu_traffic.py for config c4), or None."""
    import glob
    def version(path):  # r<round>_v<version>_traffic.json, compared numerically (v10 after v9)
        return tuple(int(x) for x in re.findall(r"\d+", os.path.basename(path)))
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), key=version)
    if not files or n_dof != C4_DOFS:
        return None, None
    with open(files[-1]) as f:
        d = json.load(f)
    k = d.get("kernels", {}).get(kernel)
    return (k["dram_bytes"] / 1e9, os.path.basename(files[-1])) if k else (None, None)


class ClockSampler:
    """Samples SM clock / throttle reasons with NVML during the timed region."""

    def __init__(self, device_index=0, period=0.02):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_init():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def host_info():
    """CPU model and core count of the host."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "oracle_threads": 1}




def config_table(ads, torch, hbm):
    """Step time of every BASELINE.json config through the public API (graph replays, CUDA events
    on a caller stream): the per-config view of the same build (c1/c2 are launch-bound, c5 is the
    elasticity step, 3 components)."""
    out = {}
    for name in ["c1", "c2", "c3", "c4", "c5"]:
        wl = workloads.get(name)
        s = ads.make_solver(wl)
        st = torch.cuda.Stream()
        s.set_stream(st)
        s.step(4)
        K = min(wl.steps, 50)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            e0.record(st)
            s.step(K)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / K)
        ms = statistics.median(ts)
        d = {"us_per_step": 1e3 * ms, "dof": wl.ndof, "dof_steps_per_s": wl.ndof / (ms / 1e3), "steps_timed": K}
        if not wl.elastic:  # the handle's own step plan (ads_step_bytes), and the 64 B/DOF floor
            plan = float(sum(s.step_bytes()))
            d["plan_bytes_per_dof"] = plan
            d["plan_hbm_frac"] = plan * wl.ndof / (ms / 1e3) / 1e9 / hbm
            d["floor_hbm_frac"] = 64.0 * wl.ndof / (ms / 1e3) / 1e9 / hbm
        out[name] = d
        s.close()
        del s
        torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------------ CPU oracle
def oracle_sample(wl, nel_sample, steps, warmup=0):
    """Time the oracle (as it stands, 1 thread) on `steps` steps of the workload recipe
    scaled to nel_sample^3 elements.  Returns (DOF-steps/s, seconds, sample description)."""
    import oracle
    w = wl.scaled(nel_sample, steps) if nel_sample != wl.nel[0] else wl
    o = oracle.make_solver(w)
    if warmup:
        o.step(warmup)
    t0 = time.perf_counter()
    o.step(steps)
    dt = time.perf_counter() - t0
    n = w.ndof
    desc = (f"oracle (oracle/ads_oracle.c, gcc -O2, 1 thread) on {steps} step(s) of the {wl.name} recipe at "
            f"{w.nel[0]}^3 elements ({n} DOFs), after set_state and {warmup} warm-up step(s); wall clock")
    return n * steps / dt, dt, desc


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    wl = workloads.get(args.config)
    nel = args.ref_nel
    val, dt, desc = oracle_sample(wl, nel, args.steps, warmup=args.warmup)
    n = wl.scaled(nel).ndof
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, workloads/)",
        "config": {"workload": f"{wl.name} recipe at {nel}^3 elements (bounded CPU sample)", "p": wl.p,
                   "n_dof": n, "tau": wl.tau},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc, **host_info()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU arm
def run_ours(args, rank, world, local):
    import torch
    import paper_1911_08158_b200 as ads
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    wl = workloads.get(args.config)
    N = wl.ndof  # global DOFs
    if world > 1:
        # strong scaling: the grid is cut into `world` z-slabs, one per GPU (NCCL over NVLink)
        uid = ads.broadcast_unique_id(rank)
        s = ads.make_solver(wl, dist=(rank, world, uid))
    else:
        s = ads.make_solver(wl)
    stream = torch.cuda.Stream()
    s.set_stream(stream)
    # the initial state (device copies), so every timed repeat restarts from it
    u_init = torch.empty(s.shape, dtype=torch.float64, device="cuda")
    ud_init = torch.empty_like(u_init)
    s.get_state(u_init, ud_init, None)
    s.step(args.warmup)
    torch.cuda.synchronize()

    # timed repeats (production launch path: graph replays): restart, barrier + sync, exactly K
    # steps between CUDA events on the library's stream, barrier + sync; median over the repeats
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = s.launch_count()
    reps = []
    with ClockSampler(local) as clk:
        for _ in range(args.repeats):
            s.set_state(u_init, ud_init)
            barrier(world)
            torch.cuda.synchronize()
            ev0.record(stream)
            s.step(args.steps)
            ev1.record(stream)
            torch.cuda.synchronize()
            barrier(world)
            reps.append(max_over_ranks(ev0.elapsed_time(ev1), world))
    launches = (s.launch_count() - launches0) // args.repeats
    ms = statistics.median(reps)
    value = N * args.steps / (ms / 1e3)  # whole-job DOF-steps/s (every rank's slab together)
    # per-kernel times: a separate profiled run (events around every launch, direct launches)
    s.set_state(u_init, ud_init)
    s.profile_enable(True)
    s.step(args.steps)
    kms, kcnt = s.profile_read()
    kms, kcnt = kms[:4], kcnt[:4]  # the step's kernel classes
    s.profile_enable(False)
    torch.cuda.synchronize()

    # ---- roofline of the dominant kernel (algorithmic bytes / its average launch time)
    hbm, peak_kind, _ = peaks()
    Nloc = s.N  # this rank's DOFs per component (the per-kernel rooflines are per GPU)
    if wl.elastic:
        # elasticity (c5): ~40 launches per step; the roofline is that of the
        # whole step against its estimated 176 B per vector DOF (3 components) and step
        step_bytes = ELASTIC_STEP_BYTES * N
        achieved = step_bytes / (ms / args.steps / 1e3) / 1e9
        kernels = {}
        roofline = {"bound": "hbm", "kernel": "elastic step (all launches)", "achieved": achieved, "peak": hbm,
                    "unit": "GB/s", "frac": achieved / hbm, "peak_kind": peak_kind, "traffic": None,
                    "algorithmic_bytes": step_bytes / 1e9, "step_bytes_per_dof": ELASTIC_STEP_BYTES,
                    "plan_bytes_per_dof": ELASTIC_PLAN_BYTES,
                    "plan_frac": ELASTIC_PLAN_BYTES * N / (ms / args.steps / 1e3) / 1e9 / hbm,
                    "note": "SURVEY.md §8(d) estimate: 170-180 B per vector DOF and step (6 ADS solves, "
                            "Kronecker triples); the step as built moves 264 B per DOF (DESIGN.md §7); "
                            "c5 fields (17.6 MB per component) are L2-resident"}
    else:
        shares = kms / kms.sum() if kms.sum() > 0 else kms
        dom = int(np.argmax(kms))
        per_launch_ms = kms / np.maximum(kcnt, 1)
        plan = s.step_bytes()  # algorithmic bytes per DOF of each kernel class of this handle's step
        kick = 3  # the z sweep carries the kick
        kernels = {}
        for i, name in enumerate(KERNELS):
            bpd = plan[i]
            if i == kick:  # a is stored on the last step of a batch only
                bpd = plan[i] + 8.0 / max(kcnt[i], 1)
            gbs = Nloc * bpd / (per_launch_ms[i] / 1e3) / 1e9 if per_launch_ms[i] > 0 else 0.0
            kernels[name] = {"ms_per_launch": per_launch_ms[i], "launches": int(kcnt[i]), "share": float(shares[i]),
                             "bytes_per_dof": bpd, "achieved_gbs": gbs, "frac": gbs / hbm}
        achieved = kernels[KERNELS[dom]]["achieved_gbs"]
        step_bytes = Nloc * (sum(plan) + 8.0 / args.steps)
        traffic, traffic_src = ncu_traffic(KERNELS[dom], Nloc)
        roofline = {"bound": "hbm", "kernel": KERNELS[dom], "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "peak_kind": peak_kind,
                    "traffic": traffic, "traffic_unit": "GB per launch (ncu dram read + write)",
                    "traffic_source": traffic_src,
                    "algorithmic_bytes": Nloc * kernels[KERNELS[dom]]["bytes_per_dof"] / 1e9,
                    "step_achieved": step_bytes / (ms / args.steps / 1e3) / 1e9,
                    "step_frac": step_bytes / (ms / args.steps / 1e3) / 1e9 / hbm,
                    "step_bytes_per_dof": step_bytes / N, "floor_bytes_per_dof": 64.0}

    # ---- end-to-end through the C ABI with host buffers (pinned), copies inside the timed region
    u_host = torch.empty(s.shape, dtype=torch.float64, pin_memory=True)
    ud_host = torch.empty_like(u_host, pin_memory=True)
    a_host = torch.empty_like(u_host, pin_memory=True)
    s.get_state(u_host, ud_host, a_host)  # the state the run starts from (also warms the copy path)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    s.set_state(u_host, ud_host)          # H2D u, udot + half-kick init
    s.step(args.steps)
    e = s.energy()                        # D2H 3 doubles
    s.get_state(u_host, ud_host, None)    # D2H the state reached: u, udot
    torch.cuda.synchronize()
    t_e2e = max_over_ranks(time.perf_counter() - t0, world)
    e2e = {"value": N * args.steps / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": 2 * 8 * N / args.steps, "d2h_bytes_per_step": (2 * 8 * N + 24) / args.steps,
           "what": "ads_set_state(host u, udot) + ads_step(K) + ads_energy + ads_get_state(host u, udot); "
                   "pinned host buffers; wall clock incl. copies", "energy": list(map(float, e))}

    line = {
        "metric": "Elasticity DOF-steps/sec (fp64)" if wl.elastic else METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "repeats": {"n": args.repeats, "ms": reps, "statistic": "median; each repeat restarts from the initial "
                    "state (set_state) and times exactly `steps` steps"},
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, workloads/)",
        "config": {"workload": f"{wl.name}: {wl.description}", "p": wl.p, "nel": list(wl.nel),
                   "n_dof": N, "tau": wl.tau, "parallelism": f"z-slabs x{world} (NCCL)" if world > 1 else "single",
                   "l2": "inputs larger than L2 (1.09 GB per field vs 126 MB L2); no flush"},
        "roofline": roofline, "kernels": kernels, "gpu_launches": int(launches),
        "clocks": clk.summary(), "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.cpu_full:
            val, dt, desc = oracle_sample(wl, wl.nel[0], 1)
        else:
            val, dt, desc = oracle_sample(wl, args.ref_nel, args.cpu_steps)
        line["cpu_baseline"] = {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
                                "seconds": dt, **host_info()}
    if rank == 0 and world == 1 and not args.no_configs:
        line["configs"] = config_table(ads, torch, hbm)
    if rank == 0:
        print(json.dumps(line), flush=True)
    s.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-nel", type=int, default=128, help="oracle sample grid (elements per direction)")
    ap.add_argument("--cpu-steps", type=int, default=40, help="oracle steps for the cpu_baseline sample")
    ap.add_argument("--cpu-full", action="store_true", help="time the oracle on one full-size step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config table (c1..c5)")
    ap.add_argument("--repeats", type=int, default=5, help="timed repeats of `steps` steps (median)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        ap.error("--warmup must be >= 3")
    rank, world, local = dist_init()
    if args.impl == "reference":
        rc = run_reference(args, rank, world)
    else:
        rc = run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
