import sys, os, json
sys.path.insert(0, '/root/repo')
import paper_2304_08232_b200 as slab
from paper_2304_08232_b200 import _capi
ctx = slab.Context(0)
import ctypes
for dims in [(192,)*3, (256,)*3, (104,)*3]:
    lvl = ctx.build_hierarchy(dims, 1)
    n = lvl.n(); nnz = lvl.A.nnz()
    r, _ = ctx.random_vector(n, 1)
    z = ctx.DenseVector(n, 0.0)
    for win in (0, 1, 0, 1):
        _capi.set_tuning("l2_window", win)
        for _ in range(3): slab.rbgs_symmetric(lvl, z, r)
        ctx.timer_start()
        for _ in range(10): slab.rbgs_symmetric(lvl, z, r)
        ms = ctx.timer_stop() / 10
        print(dims[0], "l2_window", win, "gs_sym_ms %.4f" % ms, "frac %.3f" % (2 * (12 * nnz + 32 * n) / ms / 1e6 / 6551))
