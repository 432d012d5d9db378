"""The C++ facade (include/slab_b200.hpp) compiles against the C ABI on any box; on a GPU box the
facade program — the reference's own test shapes under `namespace slab = slab_b200` — must pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "facade_test.cpp")
EXE = os.path.join(ROOT, "tests", "cpp", "facade_test.bin")


def compile_facade(slab):
    libdir = os.path.dirname(slab.LIB_PATH)
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC, "-o", EXE,
           "-L", libdir, "-lslab_b200", f"-Wl,-rpath,{libdir}", "-L/usr/local/cuda/lib64", "-Wl,-rpath,/usr/local/cuda/lib64"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    assert proc.returncode == 0, proc.stderr[-3000:]
    assert "warning" not in proc.stderr, proc.stderr[-3000:]


def test_facade_compiles_and_links(slab):
    compile_facade(slab)
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_facade_program_passes_on_gpu(slab):
    compile_facade(slab)
    proc = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-2000:]
    assert "all checks passed" in proc.stdout
