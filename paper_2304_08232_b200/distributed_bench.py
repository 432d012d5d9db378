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
    ctx.timer_start()
    for _ in range(reps):
        slab.rbgs_symmetric(h, z, b)
    gs_ms = ctx.timer_stop()
    per_launch_s = gs_ms * 1e-3 / (16 * reps)
    info = ctx.dist_info()

    if rank == 0:
        iter_bytes = bench.algorithmic_bytes_per_iteration(dims) * world
        line = {
            "metric": "hpcg_gflops", "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench.workload_config(args.workload, dims, world),
            "dot_mode": args.dot, "final_residual": res.residual_history[-1],
            "hbm_gbs_algorithmic": iter_bytes * bench.CG_ITERS / (ms / args.steps * 1e-3) / 1e9,
            "clocks": clocks,
            "e2e": {"value": total_flops_iter * bench.CG_ITERS * args.steps / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": 2 * 8 * n * world,
                    "d2h_bytes_per_step": (8 * n + 8 * (bench.CG_ITERS + 1) + 16 + 16 * bench.CG_ITERS) * world,
                    "ms_per_step": e2e_ms / args.steps},
            "gpu_launches": int(launches),
            "halo_exchanges_per_rank": info["exchanges"],
            "roofline": {"bound": "hbm",
                         "kernel": ("k_gs_color_packed* (coded copy)" if h.format_info()["packed"] else "k_gs_color_batched")
                         + " — finest-level colour step of rank 0, including its halo exchange",
                         "format": h.format_info(),
                         "achieved": bench.gs_step_bytes(dims) / per_launch_s / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": bench.gs_step_bytes(dims) / per_launch_s / 1e9 / peak, "traffic": bench.measured_traffic(dims),
                         "peak_source": peak_src},
        }
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()
    return 0
