"""Build libcm.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "cm_runtime.cu"),     # device runtime + kernels
       os.path.join(HERE, "csrc", "cm_persist.cc")]     # host-only persistence / serving
DEPS = SRC + [os.path.join(HERE, "csrc", "cm_kernels.cuh"), os.path.join(HERE, "csrc", "cm_segment.h"),
              os.path.join(ROOT, "include", "cm.h")]
OUT = os.path.join(HERE, "libcm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-fmad=false",                       # no FMA contraction anywhere (reading R4)
         "-Xcompiler", "-fPIC,-O2", "-shared", "-I" + os.path.join(ROOT, "include")]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT):
        t = os.path.getmtime(OUT)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return OUT
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, "-o", tmp, *SRC, "-lrt"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
