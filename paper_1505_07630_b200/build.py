"""In-tree build of libldu_b200.so (sm_100a) -- called by __graft_entry__.build() and the tests.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, linked against the NCCL that torch
ships (site-packages/nvidia/nccl, 2.28.x) with an rpath, so one NCCL is loaded per process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libldu_b200.so")
SRCS = [os.path.join(HERE, "csrc", f) for f in ("ldu_setup.cu", "ldu_solve.cu", "ldu_amg_setup.cu", "ldu_api.cu")]
DEPS = SRCS + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "ldu.h")]


def nccl_root() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        cand = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    raise RuntimeError("NCCL headers (nvidia/nccl wheel) not found")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile each translation unit in parallel (nvcc -c), then link the shared library."""
    if not force and not stale():
        return LIB
    nccl = nccl_root()
    common = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
              "-lineinfo", "-Xcompiler", "-fPIC", "--extended-lambda", "-Xptxas",
              "-v" if verbose else "-O3", "-I" + os.path.join(ROOT, "include"),
              "-I" + os.path.join(nccl, "include")]
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for src in SRCS:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append(subprocess.Popen(common + ["-c", src, "-o", obj]))
    codes = [p.wait() for p in procs]
    if any(codes):
        raise subprocess.CalledProcessError(max(codes), "nvcc -c")
    subprocess.check_call(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-o", LIB + ".tmp", *objs,
                           "-L" + os.path.join(nccl, "lib"), "-l:libnccl.so.2",
                           "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")])
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
