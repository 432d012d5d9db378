#!/usr/bin/env python
"""bench.py — HPCG-counted fp64 GFLOP/s of the MG-preconditioned CG solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

One "step" is one full cg_solve (4 MG levels, 1 pre/1 post coloured symmetric GS sweep, b = A*1,
x0 = 0, 50 fixed CG iterations) on synthetic HPCG input (HPCG's input *is* synthetic: the
27-point stencil). Default workload at N=1: the 192^3-per-GPU solve of BASELINE.json configs[4]
(the largest single-GPU configuration; configs[3] = 104^3 and configs[1] = 64^3 are reported
beside it under "other_workloads"). For N>1 the same local grid is weak-scaled over the process
grids 2x1x1 / 2x2x1 / 2x2x2 with NCCL halo exchange.

`value` times device-resident solves with CUDA events on the library's stream; `e2e` times the
host-buffer entry point slab_cg_solve_host (H2D of b and x0 from pinned memory, the solve, D2H of
x and the residual history) the same way. `--impl reference` times the reference's own CPU
implementation (oracle/_ref when built, else the oracle port) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CG_ITERS = 50
LEVELS = 4
WORKLOADS = {
    # name: local grid per GPU
    "hpcg192": (192, 192, 192),  # BASELINE.json configs[4]
    "hpcg104": (104, 104, 104),  # configs[3]
    "hpcg64": (64, 64, 64),      # configs[1]
    "hpcg16": (16, 16, 16),      # configs[0]
}
PROCESS_GRIDS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}


# ----------------------------------------------------------------------------- counting


def level_dims(dims, levels=LEVELS):
    out = [tuple(dims)]
    for _ in range(levels - 1):
        out.append(tuple(d // 2 for d in out[-1]))
    return out


def stencil_nnz(d):
    return (3 * d[0] - 2) * (3 * d[1] - 2) * (3 * d[2] - 2)


def color0_nnz(d):
    """stored nonzeros of the injected rows (parity class 0)."""
    def span_sum(n):
        return sum((1 if i > 0 else 0) + 1 + (1 if i + 1 < n else 0) for i in range(0, n, 2))
    return span_sum(d[0]) * span_sum(d[1]) * span_sum(d[2])


def hpcg_flops_per_iteration(dims, levels=LEVELS):
    """12 nnz0 + 12 n0 + 10 sum_mid nnz_l + 4 nnz_coarsest (the residual is counted
    as a full SpMV by HPCG convention although the kernel only computes the injected rows)."""
    ld = level_dims(dims, levels)
    n0 = ld[0][0] * ld[0][1] * ld[0][2]
    if levels == 1:
        return 2 * stencil_nnz(ld[0]) + 12 * n0 + 4 * stencil_nnz(ld[0])
    flops = 12 * stencil_nnz(ld[0]) + 12 * n0
    for d in ld[1:-1]:
        flops += 10 * stencil_nnz(d)
    flops += 4 * stencil_nnz(ld[-1])
    return flops


def algorithmic_bytes_per_iteration(dims, levels=LEVELS):
    """SURVEY.md §8(d) fused-minimum model: fp64 values + 32-bit columns (12 B/nnz), 8 B/element."""
    ld = level_dims(dims, levels)
    total = 0
    for k, d in enumerate(ld):
        n = d[0] * d[1] * d[2]
        nnz = stencil_nnz(d)
        sweep = 12 * nnz + 32 * n
        if k == len(ld) - 1 and levels > 1:
            total += 2 * sweep
            continue
        total += 4 * sweep
        if levels > 1:
            n_c = n // 8
            total += 12 * color0_nnz(d) + 8 * n + 16 * n_c  # fused residual + restriction
            total += 24 * n_c                                # prolongation + update
        if k == 0:
            total += 12 * nnz + 16 * n  # CG SpMV
            total += 40 * n             # 3 dots (16n, 16n, 8n)
            total += 72 * n             # 3 waxpby
    return total


def sweep_bytes_model(dims):
    """SURVEY.md §8(d) bytes of ONE symmetric sweep (16 colour steps): 2 (12 nnz + 32 n)."""
    n = dims[0] * dims[1] * dims[2]
    return 2 * (12 * stencil_nnz(dims) + 32 * n)


def spmv_bytes_model(dims):
    n = dims[0] * dims[1] * dims[2]
    return 12 * stencil_nnz(dims) + 16 * n


def gs_step_bytes(dims):
    """SURVEY model bytes of ONE colour-step launch on the finest level: (12 nnz + 32 n) / 8."""
    n = dims[0] * dims[1] * dims[2]
    return (12 * stencil_nnz(dims) + 32 * n) / 8.0


def gs_step_bytes_coded(dims, info):
    """bytes ONE colour-step launch has to move when the level is dictionary-coded (packed.cu; decomposed levels of the
    multi-GPU arm): per row of the colour 16 B code words x chunks + 4 B row index + r + z in + z out (8 B each), and
    the gathered vector once per sweep (n * 8 / 8 per step)."""
    n = dims[0] * dims[1] * dims[2]
    chunks = (info["width_class"] + 16) // 16
    return (n / 8.0) * (16 * chunks + 4 + 24) + n


def sweep_bytes_planes(dims):
    """bytes ONE symmetric sweep has to move in the matrix-free plane format (plane.cu, three launches): phase A
    reads z (8n) and r on the even planes (4n) and writes every plane (8n: the even ones updated, the odd ones
    copied along) = 20n; phases B and C each read z (8n) and r on their planes (4n) and write their planes (4n)
    = 16n. 52 bytes per row."""
    return 52 * dims[0] * dims[1] * dims[2]


def spmv_bytes_planes(dims):
    """plane_spmv.cu: x in, y out."""
    return 16 * dims[0] * dims[1] * dims[2]


def format_bytes_per_iteration(dims, levels=LEVELS):
    """compulsory bytes of one CG iteration (tree-dot mode) in the formats the kernels actually read:
    matrix-free plane sweeps (52 n per symmetric sweep; the first sweep of a V-cycle starts from a zero guess that is a
    flag, not a vector: 8 n less) and products (16 n), the fused transfers (16 n_c out, 8 n_c in), and on the finest
    level the p update 24 n and the fused x/r update + r'r 48 n; r'z rides on the last plane phases (nothing extra) from
    2^19 rows on, below that it is its own pass over r and z (16 n)."""
    ld = level_dims(dims, levels)
    total = 0
    for k, d in enumerate(ld):
        n = d[0] * d[1] * d[2]
        last = k == len(ld) - 1 and levels > 1
        total += (1 if last else 2) * sweep_bytes_planes(d) - 8 * n
        if not last and levels > 1:
            total += 24 * (n // 8)
        if k == 0:
            total += spmv_bytes_planes(d) + (24 + 48) * n + (0 if n >= (1 << 19) else 16 * n)
    return total


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def pump():
            for line in self.proc.stdout:
                self.samples.append(line.strip())

        self.thread = threading.Thread(target=pump, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.samples:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline / reference arm


def _oracle(kind_preference=("reference", "port")):
    from oracle.oracle import Oracle, available_kinds

    kinds = available_kinds()
    for k in kind_preference:
        if k in kinds:
            return Oracle(k)
    from oracle import oracle as omod

    omod.build(ref=False)
    return Oracle("port")


def cpu_solve_sample(o, dims, iters):
    """Times cg_solve on the host cores with `iters` of the 50 iterations (setup excluded, as the
    reference's own harness does: bench.hpp:170-172,190-192). Returns (seconds, hierarchy, b)."""
    h = o.build_hierarchy(*dims, LEVELS)
    b = o.level_mxv(h, np.ones(h.n))
    x0 = np.zeros(h.n)
    return h, b, x0


def cpu_sample_iterations(dims):
    n = dims[0] * dims[1] * dims[2]
    # ~0.11 us per row-iteration on 8 cores: keep a sample near 5-10 s
    per_iter = 1.1e-7 * n
    return int(max(1, min(CG_ITERS, round(6.0 / max(per_iter, 1e-9)))))


def run_cpu_baseline(dims):
    o = _oracle()
    iters = cpu_sample_iterations(dims)
    h, b, x0 = cpu_solve_sample(o, dims, iters)
    t0 = time.perf_counter()
    res = o.cg_solve(h, b, x0, max_iters=iters, fixed_iterations=iters)
    dt = time.perf_counter() - t0
    gflops = hpcg_flops_per_iteration(dims) * res.iterations / dt / 1e9
    return {
        "value": gflops, "unit": "GFLOP/s", "cores": o.threads, "kind": o.kind,
        "sample": f"{iters} of {CG_ITERS} CG iterations of the same {dims[0]}^3 4-level solve "
                  f"({dt:.2f} s; hierarchy generation excluded as in bench.hpp:170-172); ONE cold run, also the parity "
                  "check of the timed GPU solve — the number to quote is the --impl reference arm (mean of K steps after warm-up)",
    }, res


def run_reference_arm(args, dims):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    o = _oracle()
    iters = cpu_sample_iterations(dims)
    h, b, x0 = cpu_solve_sample(o, dims, iters)
    for _ in range(args.warmup):
        o.cg_solve(h, b, x0, max_iters=iters, fixed_iterations=iters)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.cg_solve(h, b, x0, max_iters=iters, fixed_iterations=iters)
    dt = time.perf_counter() - t0
    gflops = hpcg_flops_per_iteration(dims) * iters * args.steps / dt / 1e9
    sample = (f"each step = {iters} of {CG_ITERS} CG iterations of the {dims[0]}^3 4-level solve on the host cores "
              f"(setup excluded; a rate, so the bounded sample compares with the 50-iteration GPU step); single process "
              f"on the grid of rank 0's local size; mean of {args.steps} steps after {args.warmup} warm-ups: the CPU number to quote")
    line = {
        "impl": "reference", "metric": "hpcg_gflops", "value": gflops, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, dims, 1),
        "cpu_baseline": {"value": gflops, "unit": "GFLOP/s", "cores": o.threads, "kind": o.kind, "sample": sample},
        "e2e": {"value": gflops, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm


def workload_config(name, dims, n_gpus):
    grid = PROCESS_GRIDS.get(n_gpus, (n_gpus, 1, 1))
    cfg = {
        "workload": f"{name}: MG-preconditioned CG, local grid {dims[0]}x{dims[1]}x{dims[2]} per GPU, {LEVELS} MG levels, "
                    f"1 pre/1 post coloured SymGS, b=A*1, x0=0, {CG_ITERS} fixed iterations",
        "local_grid": list(dims), "process_grid": list(grid), "levels": LEVELS, "cg_iterations": CG_ITERS,
        "l2": "no flush: the vectors one iteration streams through (x, r, p, q, z, its out-of-place partner, b: "
              f"{7 * 8 * dims[0] * dims[1] * dims[2] / 1e6:.0f} MB on the finest level) exceed the 126 MB L2 at the headline "
              "size; smaller workloads are reported as they run, L2-resident",
    }
    return cfg


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def measured_traffic(key, dims):
    """dram bytes per launch (read + write, live caches) from the committed ncu capture, if any: profiles/traffic.json"""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    try:
        with open(path) as fh:
            data = json.load(fh)
        return data.get(key, {}).get("x".join(str(d) for d in dims))
    except (OSError, ValueError):
        return None


def time_solves(slab, ctx, h, b, x0, cfg, count, x):
    """CUDA events on the library's stream around `count` solves; cross-checked against the host
    clock (every solve ends with a stream synchronisation, so the two must agree)."""
    ctx.sync()
    t0 = time.perf_counter()
    ctx.timer_start()
    res = None
    inner = 0.0
    for _ in range(count):
        res = slab.cg_solve(h, b, x0, cfg, out=x)
        inner += res.solve_ms
    ms = ctx.timer_stop()
    wall = (time.perf_counter() - t0) * 1e3
    if count and not (inner <= ms * 1.001 + 0.05 and ms <= wall * 1.001 + 0.05):
        raise RuntimeError(f"inconsistent clocks: solves {inner:.3f} ms, events {ms:.3f} ms, host {wall:.3f} ms")
    return ms, res


def bench_one(slab, ctx, dims, steps, warmup, dot_mode):
    ctx.dot_mode = dot_mode
    h = ctx.build_hierarchy(dims, LEVELS)
    n = h.n()
    ones = ctx.DenseVector(n, 1.0)
    b = ctx.DenseVector(n)
    slab.mxv(b, h.A, ones)
    x0 = ctx.DenseVector(n, 0.0)
    cfg = slab.CGConfig(max_iters=CG_ITERS, fixed_iterations=CG_ITERS)
    x = ctx.DenseVector(n)
    time_solves(slab, ctx, h, b, x0, cfg, warmup, x)
    launches0 = slab.launch_count()
    ms, res = time_solves(slab, ctx, h, b, x0, cfg, steps, x)
    launches = slab.launch_count() - launches0
    flops = hpcg_flops_per_iteration(dims) * CG_ITERS * steps
    return {"h": h, "b": b, "x0": x0, "cfg": cfg, "ms": ms, "res": res, "launches": launches,
            "gflops": flops / (ms * 1e-3) / 1e9}


def microbench_256(slab, ctx, peak):
    """BASELINE.json configs[2]: (a) y = A x, x ~ U(-1,1) from Lcg64(0); (b) one coloured symmetric GS sweep on
    r = b - A x from z = 0 — on the 256^3 27-point matrix, checksums compared bit for bit with the reference's
    (tests/golden/micro_256.json, generated from the reference headers by tests/golden/make_golden.py)."""
    dims = (256, 256, 256)
    lvl = ctx.build_hierarchy(dims, 1)
    n = lvl.n()
    x, _ = ctx.random_vector(n, 0)
    y = ctx.DenseVector(n)
    ones = ctx.DenseVector(n, 1.0)
    b = ctx.DenseVector(n)
    slab.mxv(b, lvl.A, ones)
    slab.mxv(y, lvl.A, x)
    r = ctx.DenseVector(n)
    slab.waxpby(r, 1.0, b, -1.0, y)
    z = ctx.DenseVector(n, 0.0)
    slab.rbgs_symmetric(lvl, z, r)
    saved = ctx.dot_mode
    ctx.dot_mode = slab.DOT_EXACT  # the reference's reduction order: the checksums compare bit for bit
    try:
        sums = {"dot_yy": slab.dot(y, y), "dot_xy": slab.dot(x, y), "dot_zz_after_symmetric": slab.dot(z, z),
                "dot_rz_after_symmetric": slab.dot(r, z)}
    finally:
        ctx.dot_mode = saved
    out = {"workload": "micro256: SpMV and one coloured symmetric GS sweep on the 256^3 27-point matrix (n = 16.8 M)",
           "checksums": {k: float(v).hex() for k, v in sums.items()}}
    gpath = os.path.join(ROOT, "tests", "golden", "micro_256.json")
    if os.path.exists(gpath):
        with open(gpath) as fh:
            gold = json.load(fh)
        out["checksums_match_reference_bitwise"] = all(sums[k] == float.fromhex(gold[k + "_hex"]) for k in sums)
    reps = 20
    for _ in range(3):
        slab.mxv(y, lvl.A, x)
    ctx.timer_start()
    for _ in range(reps):
        slab.mxv(y, lvl.A, x)
    spmv_ms = ctx.timer_stop() / reps
    slab.set_all(z, 0.0)
    for _ in range(2):
        slab.rbgs_symmetric(lvl, z, r)
    launches0 = slab.launch_count()
    ctx.timer_start()
    for _ in range(reps):
        slab.rbgs_symmetric(lvl, z, r)
    gs_ms = ctx.timer_stop() / reps
    per_sweep = (slab.launch_count() - launches0) // reps
    info = lvl.format_info()
    planes = bool(info.get("plane_phases")) and per_sweep == 3
    spmv_planes = bool(lvl.A.format_info().get("plane_phases"))
    sp_fmt = spmv_bytes_planes(dims) if spmv_planes else spmv_bytes_model(dims)
    gs_fmt = sweep_bytes_planes(dims) if planes else sweep_bytes_model(dims)
    out["spmv"] = {"ms": spmv_ms, "format_bytes": sp_fmt, "format_gbs": sp_fmt / spmv_ms / 1e6,
                   "format_frac": sp_fmt / spmv_ms / 1e6 / peak, "model_frac": spmv_bytes_model(dims) / spmv_ms / 1e6 / peak,
                   "kernel": "k_spmv_planes (plane_spmv.cu)" if spmv_planes else "row kernels"}
    out["gs_symmetric_sweep"] = {"ms": gs_ms, "launches": per_sweep, "format_bytes": gs_fmt, "format_gbs": gs_fmt / gs_ms / 1e6,
                                 "format_frac": gs_fmt / gs_ms / 1e6 / peak,
                                 "model_frac": sweep_bytes_model(dims) / gs_ms / 1e6 / peak,
                                 "kernel": "k_gs_planes x3 (plane.cu)" if planes else "per-colour steps"}
    out["how"] = (f"CUDA events on the library stream, {reps} repetitions after warm-up, no L2 flush (a 256^3 vector is 134 MB, "
                  "larger than the 126 MB L2); format_* = 16 B (product) / 52 B (sweep) per row, model_* = SURVEY's 12 B/nnz")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="hpcg192", choices=sorted(WORKLOADS))
    ap.add_argument("--dot", default="tree", choices=["tree", "exact"],
                    help="reduction order of the three CG dots (exact = the reference's 4096-chunk order)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip other_workloads and the roofline micro-leg")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    dims = WORKLOADS[args.workload]

    if args.impl == "reference":
        return run_reference_arm(args, dims)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    # SLAB_BENCH_DISTRIBUTED=1 runs the multi-rank arm with a single rank (torchrun --nproc-per-node 1): the
    # rendezvous, the NCCL communicator and the library's exchange/allreduce calls on a 1x1x1 process grid
    if world > 1 or args.gpus > 1 or os.environ.get("SLAB_BENCH_DISTRIBUTED") == "1":
        from paper_2304_08232_b200 import distributed_bench

        return distributed_bench.main(args, dims)

    import torch  # device memory / pinned host buffers only

    import paper_2304_08232_b200 as slab

    ctx = slab.Context(0)
    dot_mode = slab.DOT_TREE if args.dot == "tree" else slab.DOT_EXACT
    sampler = ClockSampler(0)
    sampler.start()
    main_run = bench_one(slab, ctx, dims, args.steps, args.warmup, dot_mode)
    clocks = sampler.stop()
    h, b, cfg = main_run["h"], main_run["b"], main_run["cfg"]
    n = h.n()
    ms_per_step = main_run["ms"] / args.steps
    iter_bytes = algorithmic_bytes_per_iteration(dims)

    # ---- e2e: the host-buffer entry point, pinned host memory, copies inside the timed region
    hb = torch.empty(n, dtype=torch.float64).pin_memory()
    hx0 = torch.zeros(n, dtype=torch.float64).pin_memory()
    hx = torch.empty(n, dtype=torch.float64).pin_memory()
    hb.numpy()[:] = b.values()
    for _ in range(2):
        slab.cg_solve_host(h, hb.numpy(), hx0.numpy(), cfg, out=hx.numpy())
    ctx.timer_start()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        eres = slab.cg_solve_host(h, hb.numpy(), hx0.numpy(), cfg, out=hx.numpy())
    e2e_ms = ctx.timer_stop()
    e2e_wall_ms = (time.perf_counter() - t0) * 1e3
    e2e_ms = max(e2e_ms, e2e_wall_ms)  # the D2H tail is synchronous on the host: take the longer clock
    flops_step = hpcg_flops_per_iteration(dims) * CG_ITERS
    e2e = {"value": flops_step * args.steps / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
           "h2d_bytes_per_step": 2 * 8 * n, "d2h_bytes_per_step": 8 * n + 8 * (CG_ITERS + 1) + 16 + 16 * CG_ITERS,
           "ms_per_step": e2e_ms / args.steps,
           "final_residual": eres.residual_history[-1]}

    # ---- roofline of the dominant kernel: the plane phases of the finest-level smoother (three launches per
    #      symmetric sweep), timed alone with CUDA events on the launching stream
    peak, peak_src = peaks()
    roofline = None
    if not args.no_extras:
        z, _ = ctx.random_vector(n, 1)
        r, _ = ctx.random_vector(n, 2)  # b = A*1 is zero away from the boundary, and exact zeros take the division's slow path
        for _ in range(3):
            slab.rbgs_symmetric(h, z, r)
        reps = 20
        launches0 = slab.launch_count()
        ctx.timer_start()
        for _ in range(reps):
            slab.rbgs_symmetric(h, z, r)
        gs_ms = ctx.timer_stop()
        per_sweep = (slab.launch_count() - launches0) // reps
        info = h.format_info()
        planes = bool(info.get("plane_phases")) and per_sweep == 3
        per_launch_s = gs_ms * 1e-3 / (per_sweep * reps)
        fmt_bytes = (sweep_bytes_planes(dims) if planes else sweep_bytes_model(dims)) / per_sweep
        model_bytes = sweep_bytes_model(dims) / per_sweep
        achieved = fmt_bytes / per_launch_s / 1e9
        sweeps_per_iteration = 2  # finest level: one pre-, one post-smoothing sweep
        roofline = {
            "bound": "hbm",
            "kernel": ("k_gs_planes<kind,1,unit> (plane.cu: the finest level's symmetric sweep as three plane-phase launches; "
                       "smoother.hpp:60-113)") if planes else "per-colour steps (smoother.hpp:60-72)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": measured_traffic("gs_planes_launch", dims),
            "algorithmic_bytes_per_launch": fmt_bytes, "us_per_launch": per_launch_s * 1e6,
            "launches_per_step": per_sweep * sweeps_per_iteration * CG_ITERS,
            "share_of_step": per_sweep * sweeps_per_iteration * CG_ITERS * per_launch_s * 1e3 / ms_per_step,
            "peak_source": peak_src,
            "model_frac": model_bytes / per_launch_s / 1e9 / peak,
            "how": f"{per_sweep} launches of one symmetric sweep timed alone with CUDA events on the library stream, {reps} "
                   "repetitions after 3 warm-ups, averaged over the launches. achieved/frac count the bytes the matrix-free "
                   "plane format has to move (52 B per row and sweep: z in, r in, z out; DESIGN.md §4); model_frac keeps "
                   "SURVEY §8d's 12 B/nnz denominator (a format that streams the matrix), which this format beats by "
                   "construction. traffic = ncu dram read+write bytes per launch with live caches (--cache-control none, "
                   "profiles/r02_ncu_planes_192.txt). The launch is bound by the SM's shared-memory pipe, not by HBM",
        }

    flops_iter = hpcg_flops_per_iteration(dims)
    fmt_iter = format_bytes_per_iteration(dims)
    line = {
        "metric": "hpcg_gflops", "value": main_run["gflops"], "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, dims, 1),
        "dot_mode": args.dot,
        "final_residual": main_run["res"].residual_history[-1],
        "hbm": {
            "peak_gbs": peak,
            "format_bytes_per_iteration": fmt_iter,
            "format_gbs": fmt_iter * CG_ITERS / (ms_per_step * 1e-3) / 1e9,
            "format_frac": fmt_iter * CG_ITERS / (ms_per_step * 1e-3) / 1e9 / peak,
            "model_bytes_per_iteration": iter_bytes,
            "model_frac": iter_bytes * CG_ITERS / (ms_per_step * 1e-3) / 1e9 / peak,
            "what": "format_*: the bytes one iteration has to move in the formats the kernels read (matrix-free plane "
                    "sweeps and products, the zero initial guess of a V-cycle as a flag, r'z fused into the last plane "
                    "phases); model_*: SURVEY §8d's fused-minimum model with 12 B per stored nonzero, which "
                    "a matrix-free format exceeds by construction (kept for comparison with matrix-streaming codes)",
        },
        "clocks": clocks, "e2e": e2e, "gpu_launches": int(main_run["launches"]),
    }
    if roofline:
        line["roofline"] = roofline

    if not args.no_extras:
        # ---- the same solve in exact-dot mode (the reference's 4096-chunk order: histories bit-identical)
        other_mode = slab.DOT_EXACT if args.dot == "tree" else slab.DOT_TREE
        run = bench_one(slab, ctx, dims, 3, 3, other_mode)
        line["exact_dots" if args.dot == "tree" else "tree_dots"] = {
            "value": run["gflops"], "unit": "GFLOP/s", "ms_per_step": run["ms"] / 3,
            "final_residual": run["res"].residual_history[-1]}
        del run
        ctx.dot_mode = dot_mode

        # ---- the same solve read from the plain SELL-32 arrays (12 B per stored entry, the format SURVEY's byte
        #      model describes): what the matrix-free kernels buy, and the number to hold against the 12 B/nnz roofline
        plain_keys = {"packed": 0, "planes": 0, "spmv_planes": 0, "tile": 0}
        for key, value in plain_keys.items():
            slab.set_tuning(key, value)
        try:
            time_solves(slab, ctx, h, b, main_run["x0"], cfg, 2, ctx.DenseVector(n))
            plain_ms, _ = time_solves(slab, ctx, h, b, main_run["x0"], cfg, 3, ctx.DenseVector(n))
        finally:
            for key in plain_keys:
                slab.set_tuning(key, 1)
        plain_per = plain_ms / 3
        line["plain_sell_format"] = {"value": flops_step / (plain_per * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": plain_per,
                                     "model_frac": iter_bytes * CG_ITERS / (plain_per * 1e-3) / 1e9 / peak}
        others = []
        for name in ("hpcg104", "hpcg64", "hpcg16"):
            if name == args.workload:
                continue
            d = WORKLOADS[name]
            run = bench_one(slab, ctx, d, max(args.steps, 5), 3, dot_mode)
            per = run["ms"] / max(args.steps, 5)
            others.append({"workload": name, "value": run["gflops"], "unit": "GFLOP/s", "ms_per_step": per,
                           "format_frac": format_bytes_per_iteration(d) * CG_ITERS / (per * 1e-3) / 1e9 / peak,
                           "model_frac": algorithmic_bytes_per_iteration(d) * CG_ITERS / (per * 1e-3) / 1e9 / peak})
            del run
        line["other_workloads"] = others
        # the 192^3 hierarchy is not needed any more: make room for the 256^3 matrices
        del z, r
        main_run_res = main_run["res"]
        main_run.clear()
        main_run["res"] = main_run_res
        del h, b
        line["microbench_256"] = microbench_256(slab, ctx, peak)

    if not args.no_cpu_baseline:
        cpu, cres = run_cpu_baseline(dims)
        line["cpu_baseline"] = cpu
        k = cres.iterations
        got = np.array(main_run["res"].residual_history[: k + 1])
        want = np.array(cres.residual_history)
        line["parity_max_rel_diff_vs_cpu_sample"] = float(np.max(np.abs(got - want) / want))
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
