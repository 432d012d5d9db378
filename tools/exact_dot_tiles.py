"""Probe: the exact dot under tile sizes and chunks per block (tuning keys dot_tile, dot_cpb); device time per dot
from a burst of dots into a scratch slot (no read-back inside the timed region)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
from paper_2304_08232_b200 import _capi
ctx = slab.Context(0)
ctx.dot_mode = slab.DOT_EXACT
for n in (4096, 4096 * 148, 192 ** 3):
    x, _ = ctx.random_vector(n, 1); y, _ = ctx.random_vector(n, 2)
    ref = slab.dot(x, y)
    for tile in (0, 64, 128, 256, 512, 1024):
        for cpb in (0,) if n != 192 ** 3 else (0, 6, 24):
            _capi.set_tuning("dot_tile", tile); _capi.set_tuning("dot_cpb", cpb)
            assert slab.dot(x, y) == ref
            for _ in range(3): slab.dot(x, y)
            ctx.timer_start()
            for _ in range(20): slab.dot(x, y)
            print({"n": n, "tile": tile, "cpb": cpb, "us": round(ctx.timer_stop() / 20 * 1e3, 1)})
_capi.set_tuning("dot_tile", 0); _capi.set_tuning("dot_cpb", 0)
