#!/usr/bin/env python
"""Repeats the fixed-iteration solve and checks that every repetition returns the bits of the first one (history and
solution) — a race between the main stream and the helper streams (lazy x update, side-stream r'r) would show up as
run-to-run differences.

    python tools/soak_determinism.py --dims 104 --reps 300
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_08232_b200 as slab  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs="*", default=[104, 192])
    ap.add_argument("--reps", type=int, default=100)
    args = ap.parse_args()
    ctx = slab.Context(0)
    bad = 0
    for d in args.dims:
        h = ctx.build_hierarchy((d, d, d), 4)
        n = h.n()
        b = ctx.DenseVector(n)
        slab.mxv(b, h.A, ctx.DenseVector(n, 1.0))
        x0, _ = ctx.random_vector(n, 3)
        x = ctx.DenseVector(n)
        cfg = slab.CGConfig(max_iters=50, fixed_iterations=50)
        for mode, name in ((slab.DOT_TREE, "tree"), (slab.DOT_EXACT, "exact")):
            ctx.dot_mode = mode
            first = None
            for rep in range(args.reps):
                res = slab.cg_solve(h, b, x0, cfg, out=x)
                got = (list(res.residual_history), x.values().view(np.uint64).copy())
                if first is None:
                    first = got
                elif got[0] != first[0] or not np.array_equal(got[1], first[1]):
                    bad += 1
                    print(f"{d}^3 {name}: repetition {rep} differs from the first", flush=True)
            print(f"{d}^3 {name}: {args.reps} repetitions, final residual {first[0][-1]!r}", flush=True)
    print("differences:", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
