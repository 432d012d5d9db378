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
SOURCES = ["kernels.cu", "kernels_setup.cu", "packed.cu", "tile.cu", "plane.cu", "plane_spmv.cu", "sweep_cluster.cu", "coloring.cu", "containers.cu", "level.cu", "cg.cu", "dist.cu", "abi.cu"]
HEADERS = ["common.hpp", "kernels.cuh", "device_util.cuh", "packed_decode.cuh", "bulk_copy.cuh", "decomp.hpp", "dist.hpp", os.path.join("..", "..", "include", "slab_b200.h")]

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


STAMP = LIB + ".stamp"


def _source_digest() -> str:
    """sha256 over the sources, headers and flags the library is built from. The stamp next to the .so
    records it, so a copied tree (gpurun snapshot, fresh checkout + shipped .so) is recognised as up to
    date whatever the copy did to the file times."""
    import hashlib

    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.normpath(os.path.join(CSRC, x)) for x in HEADERS]
    for d in deps:
        if os.path.exists(d):
            h.update(d[len(HERE):].encode())
            with open(d, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    if os.path.exists(STAMP):
        with open(STAMP) as fh:
            return fh.read().strip() != _source_digest()
    built = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps += [os.path.normpath(os.path.join(CSRC, h)) for h in HEADERS]
    return any(os.path.getmtime(d) > built for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every translation unit to an object (in parallel, only the stale ones) and link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(HERE, "_build")
    os.makedirs(objdir, exist_ok=True)
    nvcc = [_nvcc()]
    # /opt/gcc (the image's default CC) lacks some runtime pieces; nvcc works with the system g++
    if os.path.exists("/usr/bin/g++"):
        nvcc += ["-ccbin", "/usr/bin/g++"]
    headers = [os.path.normpath(os.path.join(CSRC, h)) for h in HEADERS]
    newest_header = max(os.path.getmtime(h) for h in headers if os.path.exists(h))
    sources = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]

    def compile_one(name):
        src = os.path.join(CSRC, name)
        obj = os.path.join(objdir, name + ".o")
        log = os.path.join(objdir, name + ".log")
        stale = force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), newest_header)
        if not stale:
            return obj, 0, open(log).read() if os.path.exists(log) else ""
        cmd = [*nvcc, *[f for f in NVCC_FLAGS if f != "-shared"], "-c", "-o", obj, src]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        text = " ".join(cmd) + "\n" + proc.stdout + proc.stderr
        with open(log, "w") as fh:
            fh.write(text)
        return obj, proc.returncode, text

    with ThreadPoolExecutor(max_workers=min(8, len(sources))) as pool:
        results = list(pool.map(compile_one, sources))
    failed = [r for r in results if r[1] != 0]
    if verbose or failed:
        for _, _, text in (failed or results):
            sys.stderr.write(text)
    if failed:
        raise RuntimeError("nvcc failed building libslab_b200.so")
    link = [*nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *[r[0] for r in results],
            "-lcudart", "-ldl"]
    proc = subprocess.run(link, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed linking libslab_b200.so")
    with open(os.path.join(HERE, "build_ptxas.log"), "w") as fh:
        fh.write("\n".join(r[2] for r in results))
    with open(STAMP, "w") as fh:
        fh.write(_source_digest() + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
