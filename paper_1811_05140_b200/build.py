"""Build the sm_100a library in-tree (it travels to the GPU box with gpurun).

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
-fmad=false: no FMA contraction anywhere, so device FP64 matches the
reference's FMA-free x86-64 build bit-for-bit.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libqcs_b200.so")
SOURCES = [os.path.join(HERE, "csrc", "qcs_engine.cu")]
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*"))) + [os.path.join(ROOT, "include", "qcs_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
         "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        extra = ["-DQCS_WATCHDOG"] if os.environ.get("QCS_WATCHDOG") else []
        cmd = [NVCC] + FLAGS + extra + ["-o", SO] + SOURCES
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
