"""Build libads_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libads_b200.so")
SOURCES = ["kernels.cu", "modal_tc.cu", "abi.cu", "host_setup.cpp"]
HEADERS = ["kernels.cuh", "host_setup.h", os.path.join("..", "..", "include", "ads.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr",
]


def _nvcc():
    for cand in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand == "nvcc" or os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, extra=(), out=None) -> str:
    """Compile the library; `out` (with `extra` nvcc flags) builds an experiment variant."""
    lib = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    objs = []
    nvcc = _nvcc()
    procs = []
    # objects of the product build are kept in build/ and reused while newer than their source and
    # every header (force rebuilds them all); experiment variants are compiled fresh and removed
    cache = os.path.join(HERE, "build")
    os.makedirs(cache, exist_ok=True)
    hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS if os.path.exists(os.path.join(CSRC, h)))
    for src in SOURCES:  # the translation units compile in parallel
        if out:
            obj = os.path.join(CSRC, src + "." + os.path.basename(out) + ".o")
        else:
            obj = os.path.join(cache, src + ".o")
            if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(
                    hdr_t, os.path.getmtime(os.path.join(CSRC, src))):
                objs.append(obj)
                continue
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for pr, cmd in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs, "-lcudart", "-lnccl"]
    subprocess.check_call(cmd)
    if out:
        for o in objs:
            os.remove(o)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else [])
    print(LIB)
