"""Multi-process (world_size 2, gloo on CPU) checks of the host-side logic of the multi-GPU
path: slab plans agree and tile the grid, the NCCL unique id reaches every rank intact, and
bench.py's max-over-ranks timing reduction.  No GPU needed."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1911_08158_b200 as ads
        import bench
        out = {}
        # slab plan: every rank computes all extents; they agree and tile [0, nz + p)
        for nz, p in [(512, 3), (256, 2), (77, 1)]:
            mine = ads.slab_plan(nz, p, world, rank)
            t = torch.tensor(list(mine), dtype=torch.int64)
            allx = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allx, t)
            ext = [tuple(int(v) for v in x) for x in allx]
            out[(nz, p)] = ext
        uid = ads.broadcast_unique_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        out["uid_equal"] = all(i == ids[0] for i in ids) and len(uid) == 128 and any(uid)
        out["max"] = bench.max_over_ranks(float(rank + 1), world)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_dist_host_logic_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (nz, p), ext in ((k, v) for k, v in res[0].items() if isinstance(k, tuple)):
        assert ext == res[1][(nz, p)]
        assert ext[0][0] == 0 and ext[0][0] + ext[0][1] == ext[1][0] and ext[1][0] + ext[1][1] == nz + p
        assert abs(ext[0][1] - ext[1][1]) <= 1
    assert res[0]["uid_equal"] and res[1]["uid_equal"]
    assert res[0]["max"] == res[1]["max"] == float(world)
