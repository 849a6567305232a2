"""Multi-rank NCCL runs of the z-slab path (SURVEY.md §8 row e): one process per
GPU, ads_create_dist over a communicator of 2 (and 4) ranks, halos / SPIKE tips / all-to-all
pencils moved by ncclSend/ncclRecv, energies by ncclAllReduce.  Each rank compares its owned
planes with the single-GPU handle run on its own device, and bench.py's torchrun form prints
one JSON line.

These need one GPU per rank: they skip on a one-GPU box (this harness's gpurun and round-end
runs) and run wherever the node has >= 2 GPUs; the world-1 case runs the same worker on one
GPU.  The algorithm itself is covered on one GPU by the virtual-group tests
(tests/test_gpu_slabs.py), which run the same exchange schedule.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, nz, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1911_08158_b200 as ads
        import workloads
        wl = workloads.get("c4").scaled(16, 10)
        wl.nel = (21, 18, nz)
        u0 = oracle.project_separable(wl)
        ref = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc)
        ref.set_state(u0)
        ref.step(10)
        rs, re = ref.get_state(), ref.energy()
        out = {}
        for zsolve in (0, 1):
            uid = ads.broadcast_unique_id(rank)
            g = ads.Solver(wl.nel, wl.p, wl.tau, wl.bc, dist=(rank, world, uid))
            if zsolve:
                g.set_zsolve(1)
            zb, zc = g.z_begin, g.z_count
            g.set_state(np.ascontiguousarray(u0[zb:zb + zc]))
            g.step(10)
            errs = []
            for x, y in zip(g.get_state(), rs):
                y = y[zb:zb + zc]
                errs.append(float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)))
            out[zsolve] = {"extent": (zb, zc), "errs": errs, "energy": g.energy().tolist(), "ref_energy": re.tolist()}
            g.close()
        q.put((rank, out))
    except Exception as e:  # reported to the parent, which fails the test
        q.put((rank, {"error": repr(e)}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nz", [(1, 150), (2, 150), (4, 240)])  # world 1: the harness itself, on one GPU
def test_nccl_slabs_match_single_gpu(world, nz):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs (one per rank); this box has {_ngpus()}")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nz, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(world):
        assert "error" not in res[r], res[r]
    for zsolve in (0, 1):
        ext = sorted(res[r][zsolve]["extent"] for r in range(world))
        # the owned planes tile the global z extent nz + p exactly
        assert ext[0][0] == 0 and all(a[0] + a[1] == b[0] for a, b in zip(ext, ext[1:]))
        assert ext[-1][0] + ext[-1][1] == nz + 3
        for r in range(world):
            o = res[r][zsolve]
            # same bound as the virtual groups against the single-GPU path (tests/test_gpu_slabs.py)
            assert max(o["errs"]) < 1e-11, (zsolve, r, o["errs"])
            assert np.allclose(o["energy"], o["ref_energy"], rtol=1e-12), (zsolve, r)


def test_bench_torchrun_two_ranks():
    """The driver's N > 1 launch form: one JSON line from rank 0, whole-job value, n_gpus = 2."""
    if _ngpus() < 2:
        pytest.skip(f"needs 2 GPUs; this box has {_ngpus()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "4", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 4 and d["gpu_launches"] > 0
