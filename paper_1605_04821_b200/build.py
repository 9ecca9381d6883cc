"""Build libhjb.so in-tree for sm_100a (nvcc, no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "hjb.cu")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("hjb.cu", "hjb_device.cuh", "hjb_kernels.cuh", "hjb_tma.cuh", "hjb_win.cuh", "hjb_search2.cuh", "hjb_galerkin.cuh", "hjb_agmg.cuh", "hjb_nested.cuh",
                                                    "hjb_comm.h")] + \
       [os.path.join(ROOT, "include", "hjb.h")]
LIB = os.path.join(HERE, "libhjb.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-lnccl",
              "-Xcompiler", "-fPIC", "-shared"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB, SRC]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
