"""Builds paper_2304_08232_b200/libslab_b200.so in-tree with nvcc for sm_100a.

The shared library is the whole product: hand-written CUDA kernels plus the C ABI declared in
include/slab_b200.h. It is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libslab_b200.so")
SOURCES = ["kernels.cu", "kernels_setup.cu", "containers.cu", "level.cu", "cg.cu", "dist.cu", "abi.cu"]
HEADERS = ["common.hpp", "kernels.cuh", "decomp.hpp", "dist.hpp", os.path.join("..", "..", "include", "slab_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-fmad=false",  # the reference is built without FMA contraction (proj/CMakeLists.txt:8-14)
    "-Xcompiler", "-fPIC,-O2,-Wall,-Wno-unused-function",
    "-shared", "-Xptxas=-v",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA extension cannot be built")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    built = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps += [os.path.normpath(os.path.join(CSRC, h)) for h in HEADERS]
    return any(os.path.getmtime(d) > built for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    sources = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", LIB, *sources, "-lcudart", "-ldl"]
    env = dict(os.environ)
    # /opt/gcc (the image's default CC) lacks some runtime pieces; nvcc works with the system g++
    if os.path.exists("/usr/bin/g++"):
        cmd[1:1] = ["-ccbin", "/usr/bin/g++"]
    proc = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if verbose or proc.returncode != 0:
        sys.stderr.write(proc.stdout)
        sys.stderr.write(proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError("nvcc failed building libslab_b200.so")
    log = os.path.join(HERE, "build_ptxas.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
