import sys, os, ctypes as C
sys.path.insert(0, '/root/repo')
import paper_2304_08232_b200 as slab
from paper_2304_08232_b200 import _capi
lib = slab.load_library()
lib.slab_debug_read_barrier_words.argtypes = [C.c_void_p, C.POINTER(C.c_longlong * 6)]
ctx = slab.Context(0)
for dims, levels in [((16,)*3, 4), ((64,)*3, 4), ((52,)*3, 3)]:
    h = ctx.build_hierarchy(dims, levels)
    r, _ = ctx.random_vector(h.n(), 1)
    _capi.set_tuning("persist_rows", 1 << 40); _capi.set_tuning("persist_debug", 3)
    z = ctx.DenseVector(h.n(), 0.0)
    for _ in range(3): slab.mg_vcycle(h, z, r)
    out = (C.c_longlong * 6)()
    lib.slab_debug_read_barrier_words(ctx._h, C.byref(out))
    n = out[5]
    print(dims[0], "cycles per phase (block 0 thread 0): work %.0f rest %.0f arrive %.0f prefetch-issue %.0f wait %.0f" % tuple(out[i] / n for i in range(5)))
