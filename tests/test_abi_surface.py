"""CPU tests (no GPU): the C-ABI library builds for sm_100a, loads, and exports every symbol that
include/slab_b200.h declares; the Python mirror types all of them; and without a GPU the product
path fails loudly instead of falling back to anything.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "slab_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(slab_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_operator_surface():
    names = set(declared_functions())
    for required in ["slab_mxv", "slab_mxv_masked", "slab_dot", "slab_waxpby", "slab_set_all", "slab_rbgs_color_step",
                     "slab_rbgs_forward", "slab_rbgs_backward", "slab_rbgs_symmetric", "slab_restrict_vector",
                     "slab_refine_and_add", "slab_mg_vcycle", "slab_cg_solve", "slab_cg_solve_host",
                     "slab_residual_norm", "slab_hierarchy_create", "slab_level_create_csr", "slab_mat_create_csr",
                     "slab_mat_create_stencil27", "slab_mask_create", "slab_vec_upload", "slab_vec_download"]:
        assert required in names


def test_library_exports_every_declared_symbol(slab):
    lib = ctypes.CDLL(slab.LIB_PATH)
    missing = [name for name in declared_functions() if not hasattr(lib, name)]
    assert not missing, missing


def test_python_mirror_types_every_declared_symbol(slab):
    assert sorted(slab.SIGNATURES) == declared_functions()


def test_library_is_built_for_sm_100a_only(slab):
    out = subprocess.run(["cuobjdump", "--list-elf", slab.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump not available")
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_status_names_follow_the_reference_error_taxonomy(slab):
    lib = slab.load_library()
    assert lib.slab_abi_version() == 1
    assert lib.slab_status_name(1) == b"DimensionMismatch"   # error.hpp:30
    assert lib.slab_status_name(2) == b"InvalidArgument"     # error.hpp:35
    assert lib.slab_status_name(3) == b"SolverBreakdown"     # error.hpp:40


def test_no_cpu_fallback_without_a_gpu(slab):
    """On a box without a GPU creating a context must raise; on a GPU box it must succeed."""
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        slab.Context(0)
        return
    with pytest.raises(slab.CudaError) as info:
        slab.Context(0)
    assert "no CPU fallback" in str(info.value)


def test_product_never_imports_the_oracle():
    """oracle/ is test infrastructure: nothing under the package may reference it."""
    pkg = os.path.join(ROOT, "paper_2304_08232_b200")
    offenders = []
    for base, _dirs, files in os.walk(pkg):
        for name in files:
            if name.endswith((".py", ".cu", ".cuh", ".hpp", ".h")):
                text = open(os.path.join(base, name)).read()
                if re.search(r"import\s+oracle|from\s+oracle|slab_oracle|libslab_ref|oracle/|\bso_[a-z_]+\s*\(", text):
                    offenders.append(os.path.join(base, name))
    assert not offenders, offenders


def test_bench_counting_matches_survey_denominators():
    """per-iteration flops and fused-minimum bytes used by bench.py."""
    import bench

    assert bench.hpcg_flops_per_iteration((64, 64, 64)) == pytest.approx(94.78e6, rel=2e-4)
    assert bench.hpcg_flops_per_iteration((104, 104, 104)) == pytest.approx(412.1e6, rel=2e-4)
    assert bench.hpcg_flops_per_iteration((192, 192, 192)) == pytest.approx(2.618e9, rel=2e-4)
    assert bench.algorithmic_bytes_per_iteration((64, 64, 64)) == pytest.approx(0.5438e9, rel=2e-3)
    assert bench.algorithmic_bytes_per_iteration((104, 104, 104)) == pytest.approx(2.361e9, rel=2e-3)
    assert bench.algorithmic_bytes_per_iteration((192, 192, 192)) == pytest.approx(14.98e9, rel=2e-3)
    n, nnz = 256 ** 3, 766 ** 3
    assert 8 * bench.gs_step_bytes((256, 256, 256)) * 2 == 2 * (12 * nnz + 32 * n)  # 11.861 GB per symmetric sweep
    assert np.isclose(2 * (12 * nnz + 32 * n), 11.861e9, rtol=1e-3)
    assert bench.sweep_bytes_model((256, 256, 256)) == 2 * (12 * nnz + 32 * n)
    assert bench.spmv_bytes_model((256, 256, 256)) == 12 * nnz + 16 * n  # 5.662 GB
    # the matrix-free plane format: 52 B per row and symmetric sweep, 16 B per row and product
    assert bench.sweep_bytes_planes((192, 192, 192)) == 52 * 192 ** 3
    assert bench.spmv_bytes_planes((256, 256, 256)) == 16 * n
    assert bench.format_bytes_per_iteration((192, 192, 192)) < bench.algorithmic_bytes_per_iteration((192, 192, 192)) / 8


def test_reference_arm_prints_the_contract_line():
    """bench.py --impl reference (the CPU arm the driver runs beside ours) on the smallest workload: one JSON line with the
    contract's keys, `impl: reference`, zero copies, no kernel launches, and the same `config` object our arm prints."""
    import json
    import subprocess
    import sys

    import bench

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--workload", "hpcg16", "--steps", "2",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "vs_baseline",
                "dtype", "data", "config", "cpu_baseline", "e2e", "gpu_launches"):
        assert key in line, key
    assert line["impl"] == "reference" and line["metric"] == "hpcg_gflops" and line["unit"] == "GFLOP/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["vs_baseline"] is None and line["dtype"] == "f64" and line["gpu_launches"] == 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["config"] == bench.workload_config("hpcg16", bench.WORKLOADS["hpcg16"], 1)  # the same object as our arm's
    assert "note" not in line["config"]
