"""Probe: time per colour-step launch of a one-level V-cycle (one symmetric sweep: 15 launches with the
turnaround), eager launches vs one CUDA graph, with and without programmatic dependent launch."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
from paper_2304_08232_b200 import _capi
ctx = slab.Context(0)
for dims in [(96,)*3, (48,)*3, (24,)*3, (52,)*3, (26,)*3, (13,)*3, (104,)*3]:
    lvl = ctx.build_hierarchy(dims, 1)
    n = lvl.n()
    r, _ = ctx.random_vector(n, 1)
    row = {"dims": dims[0], "rows_per_step": n // 8}
    for graphs in (0, 1):
        ctx.set_graphs(bool(graphs))
        for pdl in (1, 0):
            _capi.set_tuning("pdl", pdl)
            z2 = ctx.DenseVector(n, 0.0)   # new vector => new graph capture with the current knobs
            for _ in range(3): slab.mg_vcycle(lvl, z2, r)
            ctx.timer_start()
            for _ in range(50): slab.mg_vcycle(lvl, z2, r)
            row[("graph" if graphs else "eager") + ("+pdl" if pdl else "")] = round(ctx.timer_stop() / 50 / 15 * 1e3, 2)
    _capi.set_tuning("pdl", 1)
    ctx.set_graphs(True)
    print(row)
