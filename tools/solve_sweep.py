#!/usr/bin/env python
"""Whole-solve timing under different tuning sets (run on the GPU box):

    python tools/solve_sweep.py --dims 192 104 64 --sets packed=0 packed=1 packed=1,packed_batch=2

Each set is a comma-separated list of slab_set_tuning key=value pairs applied on top of the defaults
(every key named by any set is reset to its default before each set). Reports ms per 50-iteration
solve (CUDA events inside cg_solve, best and median of --reps) and the final residual, which must not
depend on the set.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_08232_b200 as slab  # noqa: E402
from paper_2304_08232_b200 import _capi  # noqa: E402

DEFAULTS = {"packed": 1, "packed_block": 256, "packed_batch": 2, "packed_min_rows": 65536, "packed_rows": 2, "packed_rows_spmv": 3, "packed_multi_min_rows": 300000, "cluster_rows": 384,
            "stream_rows": 200000, "stream_variant": 2, "pdl": 1, "planes": 1, "plane_ty": 0, "plane_cz": 0, "plane_ns": 0, "plane_rows": 0,
            "plane_min_rows": 0, "plane_warp_sync": 1, "plane_pad_lines": 1, "fuse_rz": 1, "side_rr": 1, "lazy_x": 1, "iter_batch": 50, "inline_record": 1, "lazy_x_blocks": 1, "lazy_x_prio": 1, "spmv_planes": 1, "spmv_plane_ty": 0, "spmv_plane_cz": 0, "spmv_plane_ns": 0, "tile": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs="*", default=[192, 104, 64])
    ap.add_argument("--sets", nargs="*", default=["packed=0", "packed=1"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--levels", type=int, default=4)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    ctx = slab.Context(0)
    ctx.dot_mode = slab.DOT_TREE
    out = []
    for d in args.dims:
        dims = (d, d, d)
        h = ctx.build_hierarchy(dims, args.levels)
        n = h.n()
        ones = ctx.DenseVector(n, 1.0)
        b = ctx.DenseVector(n)
        slab.mxv(b, h.A, ones)
        x0 = ctx.DenseVector(n, 0.0)
        x = ctx.DenseVector(n)
        cfg = slab.CGConfig(max_iters=50, fixed_iterations=50)
        for s in args.sets:
            pairs = dict(p.split("=") for p in s.split(","))
            for key in DEFAULTS:
                _capi.set_tuning(key, DEFAULTS[key])
            for key, value in pairs.items():
                _capi.set_tuning(key, int(value))
            for _ in range(2):
                slab.cg_solve(h, b, x0, cfg, out=x)
            times = []
            for _ in range(args.reps):
                res = slab.cg_solve(h, b, x0, cfg, out=x)
                times.append(res.solve_ms)
            rec = {"dims": d, "set": s, "ms_best": min(times), "ms_median": statistics.median(times),
                   "final_residual": res.residual_history[-1]}
            out.append(rec)
            print(json.dumps(rec), flush=True)
        del h, b, x0, x, ones
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
