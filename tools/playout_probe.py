"""Timing experiment: symmetric GS sweep with colour-major vectors vs the natural layout."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
lib = slab.load_library()
lib.slab_debug_playout_sweep.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
ctx = slab.Context(0)
for dims in [(104,)*3, (192,)*3, (256,)*3]:
    lvl = ctx.build_hierarchy(dims, 1)
    n, nnz = lvl.n(), lvl.A.nnz()
    r, _ = ctx.random_vector(n, 1)
    z, _ = ctx.random_vector(n, 2)
    ms, diff = C.c_double(), C.c_double()
    rc = lib.slab_debug_playout_sweep(lvl._h, z._h, r._h, 10, C.byref(ms), C.byref(diff))
    assert rc == 0, lib.slab_last_error()
    for _ in range(3): slab.rbgs_symmetric(lvl, z, r)
    ctx.timer_start()
    for _ in range(10): slab.rbgs_symmetric(lvl, z, r)
    nat = ctx.timer_stop() / 10
    b = 2 * (12 * nnz + 32 * n)
    print(dims[0], "colour-major vectors: %.4f ms (frac %.3f)  natural: %.4f ms (frac %.3f)  max|diff| %g" % (ms.value, b / ms.value / 1e6 / 6551, nat, b / nat / 1e6 / 6551, diff.value))
