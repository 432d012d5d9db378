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


def gs_step_bytes(dims):
    """algorithmic bytes of ONE colour-step launch on the finest level: (12 nnz + 32 n) / 8."""
    n = dims[0] * dims[1] * dims[2]
    return (12 * stencil_nnz(dims) + 32 * n) / 8.0


def gs_step_bytes_coded(dims, info):
    """bytes ONE colour-step launch has to move when the level is dictionary-coded (packed.cu): per row of the
    colour 16 B code words x chunks + 4 B row index + r + z in + z out (8 B each), and the gathered vector once
    per sweep (n * 8 / 8 per step) — the SURVEY model with the 12 B/nnz matrix term replaced by the codes."""
    n = dims[0] * dims[1] * dims[2]
    chunks = (info["width_class"] + 16) // 16
    return (n / 8.0) * (16 * chunks + 4 + 24) + n


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
                  f"({dt:.2f} s; hierarchy generation excluded as in bench.hpp:170-172)",
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
              f"(setup excluded)")
    line = {
        "impl": "reference", "metric": "hpcg_gflops", "value": gflops, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, dims, 1, note="CPU reference arm, single process on the global grid of rank 0's local size"),
        "cpu_baseline": {"value": gflops, "unit": "GFLOP/s", "cores": o.threads, "kind": o.kind, "sample": sample},
        "e2e": {"value": gflops, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm


def workload_config(name, dims, n_gpus, note=None):
    grid = PROCESS_GRIDS.get(n_gpus, (n_gpus, 1, 1))
    cfg = {
        "workload": f"{name}: MG-preconditioned CG, local grid {dims[0]}x{dims[1]}x{dims[2]} per GPU, {LEVELS} MG levels, "
                    f"1 pre/1 post coloured SymGS, b=A*1, x0=0, {CG_ITERS} fixed iterations",
        "local_grid": list(dims), "process_grid": list(grid), "levels": LEVELS, "cg_iterations": CG_ITERS,
        "l2": "per-iteration working set (matrix twice + vectors) far exceeds the 126 MB L2; no flush needed",
    }
    if note:
        cfg["note"] = note
    return cfg


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def measured_traffic(dims):
    """dram bytes per colour-step launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    try:
        with open(path) as fh:
            data = json.load(fh)
        return data.get("gs_color_step", {}).get("x".join(str(d) for d in dims))
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

    # ---- roofline of the dominant kernel: the finest-level colour step, timed alone with CUDA
    #      events on the launching stream (16 launches per symmetric sweep)
    peak, peak_src = peaks()
    roofline = None
    if not args.no_extras:
        z = ctx.DenseVector(n, 0.0)
        r = main_run["b"]
        for _ in range(3):
            slab.rbgs_symmetric(h, z, r)
        reps = 10
        ctx.timer_start()
        for _ in range(reps):
            slab.rbgs_symmetric(h, z, r)
        gs_ms = ctx.timer_stop()
        per_launch_s = gs_ms * 1e-3 / (16 * reps)
        achieved = gs_step_bytes(dims) / per_launch_s / 1e9
        info = h.format_info()
        coded = bool(info["packed"]) and n // 8 >= 65536
        kernel = ("k_gs_color_packed_multi<27,2,2,32>" if n // 8 >= 300000 else "k_gs_color_packed<27,2,2,32>") if coded \
            else "k_gs_color_batched<9,5>"
        roofline = {"bound": "hbm", "kernel": kernel + " (finest-level colour step, smoother.hpp:60-72)",
                    "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": measured_traffic(dims), "algorithmic_bytes_per_launch": gs_step_bytes(dims),
                    "us_per_launch": per_launch_s * 1e6, "launches_per_step": 32 * CG_ITERS,
                    "share_of_step": 32 * CG_ITERS * per_launch_s * 1e3 / ms_per_step, "peak_source": peak_src,
                    "how": "16 launches of one symmetric sweep timed alone with CUDA events on the library stream, "
                           "10 repetitions after 3 warm-ups; traffic = dram bytes per launch from profiles/r01_ncu_gs_packed_192.txt "
                           "(cold cache: the gathered vector comes from DRAM there, from L2 in the live run)"}
        if coded:
            fb = gs_step_bytes_coded(dims, info)
            roofline["format"] = {
                "matrix": "dictionary-coded SELL-32 (packed.cu): 1 B per stored entry instead of the 12 B the SURVEY "
                          "model counts, decoded exactly; frac > 1 means the launch beats the HBM time of the 12 B/nnz model",
                "width_class": info["width_class"], "dict_size": info["dict_size"], "escaped_rows": info["escaped_rows"],
                "bytes_per_launch": fb, "achieved": fb / per_launch_s / 1e9, "frac": fb / per_launch_s / 1e9 / peak,
                "bound_now": "L1/L2 gather path and instruction issue (profiles/r01_ncu_gs_packed_192.txt), not HBM"}

    line = {
        "metric": "hpcg_gflops", "value": main_run["gflops"], "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload, dims, 1),
        "dot_mode": args.dot,
        "final_residual": main_run["res"].residual_history[-1],
        "hbm_gbs_algorithmic": iter_bytes * CG_ITERS / (ms_per_step * 1e-3) / 1e9,
        "hbm_frac_of_measured_peak": iter_bytes * CG_ITERS / (ms_per_step * 1e-3) / 1e9 / peak,
        "clocks": clocks, "e2e": e2e, "gpu_launches": int(main_run["launches"]),
    }
    if roofline:
        line["roofline"] = roofline

    if not args.no_extras:
        # the same solve from the plain SELL-32 arrays (12 B per stored entry, the format SURVEY's byte model
        # describes): what the dictionary-coded copy buys, and the number to hold against the 12 B/nnz roofline
        slab.set_tuning("packed", 0)
        try:
            time_solves(slab, ctx, h, b, main_run["x0"], cfg, 2, ctx.DenseVector(n))
            plain_ms, _ = time_solves(slab, ctx, h, b, main_run["x0"], cfg, 3, ctx.DenseVector(n))
        finally:
            slab.set_tuning("packed", 1)
        plain_per = plain_ms / 3
        line["plain_sell_format"] = {"value": flops_step / (plain_per * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": plain_per,
                                     "hbm_frac_of_measured_peak": iter_bytes * CG_ITERS / (plain_per * 1e-3) / 1e9 / peak}
        others = []
        for name in ("hpcg104", "hpcg64"):
            if name == args.workload:
                continue
            d = WORKLOADS[name]
            run = bench_one(slab, ctx, d, max(args.steps, 5), 3, dot_mode)
            ib = algorithmic_bytes_per_iteration(d)
            per = run["ms"] / max(args.steps, 5)
            others.append({"workload": name, "value": run["gflops"], "unit": "GFLOP/s", "ms_per_step": per,
                           "hbm_frac_of_measured_peak": ib * CG_ITERS / (per * 1e-3) / 1e9 / peak})
        line["other_workloads"] = others

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
