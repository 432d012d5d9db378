#!/usr/bin/env python
"""The target of an ncu capture: warms up, then runs the chosen operation inside a cudaProfilerStart/Stop range.

    ncu --profile-from-start off --set full --clock-control none --import-source on -o out \
        python tools/ncu_target.py --dims 192 --what sweep [--levels 1] [--sets planes=1,plane_ty=8]

what: sweep (one rbgs_symmetric of the finest level), spmv (one mxv), vcycle (one mg_vcycle),
iteration (--count CG iterations of a solve: eager launches, graphs off, so that every kernel is its own ncu row).
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_08232_b200 as slab  # noqa: E402
from paper_2304_08232_b200 import _capi  # noqa: E402


def cudart():
    for name in ("libcudart.so", "libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    raise RuntimeError("libcudart not found")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs="+", default=[192])
    ap.add_argument("--levels", type=int, default=1)
    ap.add_argument("--what", default="sweep", choices=["sweep", "spmv", "vcycle", "iteration"])
    ap.add_argument("--count", type=int, default=1)
    ap.add_argument("--dot", default="tree", choices=["tree", "exact"])
    ap.add_argument("--sets", default="")
    args = ap.parse_args()
    dims = tuple(args.dims * 3) if len(args.dims) == 1 else tuple(args.dims)
    for pair in filter(None, args.sets.split(",")):
        key, value = pair.split("=")
        _capi.set_tuning(key, int(value))
    rt = cudart()
    ctx = slab.Context(0)
    ctx.set_graphs(False)
    ctx.dot_mode = slab.DOT_TREE if args.dot == "tree" else slab.DOT_EXACT
    h = ctx.build_hierarchy(dims, args.levels)
    n = h.n()
    ones = ctx.DenseVector(n, 1.0)
    b = ctx.DenseVector(n)
    slab.mxv(b, h.A, ones)
    x, _ = ctx.random_vector(n, 0)
    y = ctx.DenseVector(n)
    z, _ = ctx.random_vector(n, 1)
    rr, _ = ctx.random_vector(n, 2)  # b = A*1 is zero away from the boundary: exact zeros take the division's slow path

    def op():
        if args.what == "sweep":
            slab.rbgs_symmetric(h, z, rr)
        elif args.what == "spmv":
            slab.mxv(y, h.A, x)
        elif args.what == "vcycle":
            slab.mg_vcycle(h, z, rr)
        else:
            k = args.count
            slab.cg_solve(h, b, ctx.DenseVector(n, 0.0), slab.CGConfig(max_iters=k, fixed_iterations=k), out=y)

    for _ in range(3):
        op()
    ctx.sync()
    rt.cudaProfilerStart()
    op()
    ctx.sync()
    rt.cudaProfilerStop()
    print("ok", args.what, dims, "launches so far:", slab.launch_count())


if __name__ == "__main__":
    main()
