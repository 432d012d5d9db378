"""Probe: one symmetric sweep of a small one-level grid as 15 per-colour launches (cluster_rows=0) against the
one-launch cluster sweep (sweep_cluster.cu), inside a CUDA graph with programmatic launches. Microseconds per sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab  # noqa: E402
from paper_2304_08232_b200 import _capi  # noqa: E402

ctx = slab.Context(0)
for d in (8, 12, 13, 16, 24, 26, 32):
    lvl = ctx.build_hierarchy((d, d, d), 1)
    n = lvl.n()
    r, _ = ctx.random_vector(n, 1)
    row = {"dims": d, "rows_per_step": n // 8}
    for rows in (0, 4096):
        _capi.set_tuning("cluster_rows", rows)
        z = ctx.DenseVector(n, 0.0)  # new vector => new graph capture with the current knobs
        for _ in range(3):
            slab.mg_vcycle(lvl, z, r)
        ctx.timer_start()
        for _ in range(200):
            slab.mg_vcycle(lvl, z, r)
        row["cluster" if rows else "per_colour"] = round(ctx.timer_stop() / 200 * 1e3, 2)
    _capi.set_tuning("cluster_rows", 4096)
    print(row)
