"""bench.py's N>1 arm: one process per GPU (torchrun), weak scaling of the MG-preconditioned CG solve.

The local grid per GPU is fixed (BASELINE.json configs[3]/[4]); the global grid is local x process
grid (2x1x1, 2x2x1, 2x2x2). torch.distributed (NCCL backend) is the plumbing: rendezvous, the
broadcast of the NCCL unique id, barriers and the max-over-ranks of the device time. The data path —
halo exchange per colour step / SpMV and the allreduce of the three dots — is the library's own
NCCL send/recv/allreduce on its stream, captured in the iteration graph.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np


def _flops_per_iteration(slab, h) -> int:
    """HPCG-counted flops of one iteration for THIS rank's rows (summed over ranks later)."""
    levels = []
    lvl = h
    while lvl is not None:
        levels.append((lvl.n(), lvl.A.nnz()))
        lvl = lvl.coarser
    n0, nnz0 = levels[0]
    if len(levels) == 1:
        return 6 * nnz0 + 12 * n0
    flops = 12 * nnz0 + 12 * n0
    for _n, nnz in levels[1:-1]:
        flops += 10 * nnz
    flops += 4 * levels[-1][1]
    return flops


def main(args, dims) -> int:
    import torch
    import torch.distributed as dist

    import bench
    import paper_2304_08232_b200 as slab

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} must be launched with {args.gpus} ranks (torchrun), got {world}")
    if args.gpus not in bench.PROCESS_GRIDS:
        raise SystemExit(f"no process grid defined for {args.gpus} GPUs (supported: {sorted(bench.PROCESS_GRIDS)})")
    grid = bench.PROCESS_GRIDS[args.gpus]
    torch.cuda.set_device(local_rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    ctx = slab.Context(local_rank)
    ctx.set_process_grid(grid, rank)
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.tensor(list(slab.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    ctx.init_nccl(bytes(uid.cpu().tolist()))
    ctx.dot_mode = slab.DOT_TREE if args.dot == "tree" else slab.DOT_EXACT

    h = ctx.build_hierarchy(dims, bench.LEVELS)
    n = h.n()
    ones = ctx.DenseVector(n, 1.0)
    b = ctx.DenseVector(n)
    slab.mxv(b, h.A, ones)
    x0 = ctx.DenseVector(n, 0.0)
    x = ctx.DenseVector(n)
    cfg = slab.CGConfig(max_iters=bench.CG_ITERS, fixed_iterations=bench.CG_ITERS)

    def timed(count):
        dist.barrier()
        torch.cuda.synchronize()
        ctx.sync()
        ctx.timer_start()
        res = None
        for _ in range(count):
            res = slab.cg_solve(h, b, x0, cfg, out=x)
        ms = ctx.timer_stop()
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item(), res

    sampler = bench.ClockSampler(local_rank)
    timed(max(args.warmup, 3))
    sampler.start()
    launches0 = slab.launch_count()
    ms, res = timed(args.steps)
    launches = slab.launch_count() - launches0
    clocks = sampler.stop()

    flops = torch.tensor([float(_flops_per_iteration(slab, h))], dtype=torch.float64, device="cuda")
    dist.all_reduce(flops)
    total_flops_iter = flops.item()
    value = total_flops_iter * bench.CG_ITERS * args.steps / (ms * 1e-3) / 1e9

    # e2e: the host-buffer entry point on every rank (its own slice of b / x), pinned memory
    hb = torch.empty(n, dtype=torch.float64).pin_memory()
    hx0 = torch.zeros(n, dtype=torch.float64).pin_memory()
    hx = torch.empty(n, dtype=torch.float64).pin_memory()
    hb.numpy()[:] = b.values()
    slab.cg_solve_host(h, hb.numpy(), hx0.numpy(), cfg, out=hx.numpy())
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        slab.cg_solve_host(h, hb.numpy(), hx0.numpy(), cfg, out=hx.numpy())
    e2e_local = (time.perf_counter() - t0) * 1e3
    t = torch.tensor([e2e_local], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = t.item()

    peak, peak_src = bench.peaks()
    z = ctx.DenseVector(n, 0.0)
    for _ in range(3):
        slab.rbgs_symmetric(h, z, b)
    reps = 10
    launches0 = slab.launch_count()
    ctx.timer_start()
    for _ in range(reps):
        slab.rbgs_symmetric(h, z, b)
    gs_ms = ctx.timer_stop()
    per_sweep = max(1, (slab.launch_count() - launches0) // reps)
    per_sweep_s = gs_ms * 1e-3 / reps
    info = ctx.dist_info()
    finfo = h.format_info()

    if rank == 0:
        iter_bytes = bench.algorithmic_bytes_per_iteration(dims) * world
        ms_per_step = ms / args.steps
        # one symmetric sweep = 16 colour steps; on a decomposed level they read the dictionary-coded copy (rows that
        # look across a cut: the plain arrays), each step followed or overlapped by its halo exchange
        coded = bool(finfo["packed"])
        fmt_sweep = 16 * bench.gs_step_bytes_coded(dims, finfo) if coded else bench.sweep_bytes_model(dims)
        if per_sweep == 3 and finfo.get("plane_phases"):
            fmt_sweep = bench.sweep_bytes_planes(dims)  # 1x1x1 process grid: the single-process plane phases
        gdims = tuple(d * g for d, g in zip(dims, grid))
        parity = None
        gpath = os.path.join(bench.ROOT, "tests", "golden", "history_%dx%dx%d.json" % gdims)
        if gdims[0] == gdims[1] == gdims[2] and not os.path.exists(gpath):
            gpath = os.path.join(bench.ROOT, "tests", "golden", "history_%d.json" % gdims[0])
        if os.path.exists(gpath):
            with open(gpath) as fh:
                gold = json.load(fh)
            want = np.array([float.fromhex(v) for v in gold["residual_history_hex"]])
            got = np.array(res.residual_history)
            if want.shape == got.shape:
                parity = float(np.max(np.abs(got - want) / want))
        line = {
            "metric": "hpcg_gflops", "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench.workload_config(args.workload, dims, world),
            "dot_mode": args.dot, "final_residual": res.residual_history[-1],
            "hbm": {"peak_gbs": peak, "model_bytes_per_iteration": iter_bytes,
                    "model_frac": iter_bytes * bench.CG_ITERS / (ms_per_step * 1e-3) / 1e9 / (peak * world),
                    "what": "SURVEY §8d's fused-minimum model (12 B per stored nonzero) over all ranks, against N x the measured peak"},
            "clocks": clocks,
            "e2e": {"value": total_flops_iter * bench.CG_ITERS * args.steps / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": 2 * 8 * n * world,
                    "d2h_bytes_per_step": (8 * n + 8 * (bench.CG_ITERS + 1) + 16 + 16 * bench.CG_ITERS) * world,
                    "ms_per_step": e2e_ms / args.steps},
            "gpu_launches": int(launches),
            "halo_exchanges_per_rank": info["exchanges"],
            "roofline": {"bound": "hbm",
                         "kernel": ("k_gs_color_packed* (coded copy)" if coded else "k_gs_color_batched")
                         + " — one symmetric sweep of rank 0's finest level (16 colour steps), halo exchanges included",
                         "format": finfo,
                         "achieved": fmt_sweep / per_sweep_s / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": fmt_sweep / per_sweep_s / 1e9 / peak,
                         "model_frac": bench.sweep_bytes_model(dims) / per_sweep_s / 1e9 / peak,
                         "algorithmic_bytes_per_launch": fmt_sweep / per_sweep, "us_per_launch": per_sweep_s / per_sweep * 1e6,
                         "launches_per_sweep": per_sweep, "traffic": None, "peak_source": peak_src,
                         "how": "frac counts the bytes of the format the launches read (coded rows + vectors); model_frac "
                                "keeps SURVEY's 12 B/nnz; no ncu capture exists for a multi-rank run (traffic null)"},
            "parity_max_rel_diff": parity,
            "parity_against": os.path.relpath(gpath, bench.ROOT) if parity is not None else None,
            "cpu_baseline": {"value": None, "unit": "GFLOP/s", "cores": None, "kind": "reference",
                             "sample": "timed at N=1 only (bench contract): see the N=1 line or --impl reference"},
            "nccl_debug": os.environ.get("NCCL_DEBUG"),
        }
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()
    return 0
