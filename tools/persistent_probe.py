"""Probe: where does a phase of the persistent V-cycle kernel spend its time? (timing only)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
from paper_2304_08232_b200 import _capi
ctx = slab.Context(0)
for dims, levels in [((16,)*3, 4), ((32,)*3, 4), ((64,)*3, 4), ((52,)*3, 3)]:
    h = ctx.build_hierarchy(dims, levels)
    n = h.n()
    r, _ = ctx.random_vector(n, 1)
    phases = sum((2 if k + 1 < levels else 1) * 16 for k in range(levels))
    row = {"dims": dims[0], "phases": phases}
    for name, (rows, dbg) in {"launches": (0, 0), "persistent": (1 << 40, 0), "barriers_only": (1 << 40, 1), "work_only": (1 << 40, 2)}.items():
        _capi.set_tuning("persist_rows", rows); _capi.set_tuning("persist_debug", dbg)
        z = ctx.DenseVector(n, 0.0)
        for _ in range(3): slab.mg_vcycle(h, z, r)
        ctx.timer_start()
        for _ in range(20): slab.mg_vcycle(h, z, r)
        row[name + "_us_per_phase"] = round(ctx.timer_stop() / 20 / phases * 1e3, 2)
    print(row)
