"""RECORD OF A REVERTED EXPERIMENT (round 2): the chunk pipeline it drove (ADS_STEP_CHUNKS in abi.cu
enqueue_step: the operator kernel per z chunk on the handle's stream, each chunk's x/y sweeps on a
side stream, joined before the z sweep) measured slower at every chunk count
(profiles/r2_chunks_c4.log, r2_chunks_c3.log) and was removed.

Pipelined single-GPU step (abi.cu enqueue_step): ms/step of a config for several z-chunk counts
(ADS_STEP_CHUNKS, read at create), and the state after a few steps compared bitwise with the
unchunked step.  usage: python scripts/time_chunks.py cfg [chunks ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_08158_b200 as ads  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
counts = [int(v) for v in sys.argv[2:]] or [1, 2, 3, 4, 6, 8]
wl = workloads.get(cfg)
ref = None
for nch in counts:
    os.environ["ADS_STEP_CHUNKS"] = str(nch)
    s = ads.make_solver(wl)
    st = torch.cuda.Stream()
    s.set_stream(st)
    s.step(5)
    torch.cuda.synchronize()
    state = s.get_state()
    same = "" if ref is None else ("bitwise equal to chunks=%d" % counts[0] if all(
        np.array_equal(a, b) for a, b in zip(state, ref)) else "DIFFERS max %.3e" % max(
        float(np.abs(a - b).max()) for a, b in zip(state, ref)))
    if ref is None:
        ref = state
    K = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for rep in range(5):
        e0.record(st)
        s.step(K)
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1) / K)
    ms.sort()
    print(f"{cfg} chunks={nch}: median {ms[2]:.3f} ms/step (min {ms[0]:.3f}), "
          f"{wl.ndof / (ms[2] * 1e-3):.3e} DOF-steps/s {same}", flush=True)
    del s
    torch.cuda.empty_cache()
