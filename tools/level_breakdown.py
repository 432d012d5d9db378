#!/usr/bin/env python
"""Per-level time shares of a solve from the LevelStats timers (run on the GPU box):

    python tools/level_breakdown.py --dims 192 [--runs 3]

Uses the benchmark harness with the timers on (launch by launch, CUDA events around the reference's
sections), so the absolute solve time is a little above the graph-replayed one that bench.py reports.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_08232_b200 as slab  # noqa: E402
from paper_2304_08232_b200 import harness  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, default=192)
    ap.add_argument("--runs", type=int, default=3)
    args = ap.parse_args()
    ctx = slab.Context(0)
    ctx.dot_mode = slab.DOT_TREE
    cfg = harness.BenchConfig(dims=(args.dims,) * 3, levels=4, runs=args.runs, fixed_iterations=50, max_iters=50,
                              skip_symmetry=True)
    rep = harness.run_benchmark(ctx, cfg, profile_levels=True)
    run = rep.runs[-1]
    print(json.dumps({"solve_ms": run.solve_seconds * 1e3,
                      "levels": [{"level": l.level, "n": l.n, "smoother_ms": l.smoother_seconds * 1e3,
                                  "transfer_ms": l.transfer_seconds * 1e3, "mg_ms": l.mg_seconds * 1e3} for l in run.levels]}))
    fast = harness.run_benchmark(ctx, cfg, profile_levels=False)
    print(json.dumps({"graph_replayed_solve_ms": fast.runs[-1].solve_seconds * 1e3}))


if __name__ == "__main__":
    main()
