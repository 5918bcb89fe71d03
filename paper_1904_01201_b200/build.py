"""Build the in-tree CUDA extension for sm_100a (``python -m paper_1904_01201_b200.build``)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "navsim_b200.cu")
OUT = os.path.join(HERE, "_lib", "libnavsim_b200.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in
        ("navsim_b200.cu", "kernels.cuh", "geom.cuh", "agent.cuh", "cast.cuh", "fill.cuh",
         "device.cuh", "exact_math.cuh", "nav.cuh",
         "codec.cuh", "nav_task_abi.inc", "codec_abi.inc")] + [
    os.path.join(HERE, "..", "include", "navsim_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",                 # exact FP64 path: no implicit contraction
    "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-o", tmp, SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
