"""Probe: per-colour-step time of small levels, eager launches vs one CUDA graph per V-cycle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
from paper_2304_08232_b200 import _capi
ctx = slab.Context(0)
for dims in [(96,)*3, (48,)*3, (24,)*3, (52,)*3, (26,)*3, (13,)*3, (104,)*3]:
    lvl = ctx.build_hierarchy(dims, 1)
    n = lvl.n()
    r, _ = ctx.random_vector(n, 1)
    z = ctx.DenseVector(n, 0.0)
    row = {"dims": dims[0]}
    for graphs in (0, 1):
        ctx.set_graphs(bool(graphs))
        for name, (sr, pdl) in {"preload+pdl": (1<<40, 1), "preload": (1<<40, 0), "stream+pdl": (0, 1), "stream": (0, 0)}.items():
            _capi.set_tuning("stream_rows", sr); _capi.set_tuning("pdl", pdl)
            z2 = ctx.DenseVector(n, 0.0)   # new vector => new graph capture with the current knobs
            for _ in range(3): slab.mg_vcycle(lvl, z2, r)
            ctx.timer_start()
            for _ in range(20): slab.mg_vcycle(lvl, z2, r)
            row[("graph:" if graphs else "eager:") + name] = round(ctx.timer_stop() / 20 / 16 * 1e3, 2)
    print(row)
