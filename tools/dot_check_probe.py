import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2304_08232_b200 as slab
from oracle.oracle import Oracle
o = Oracle("port"); ctx = slab.Context(0); ctx.dot_mode = slab.DOT_EXACT
for n in (1, 33, 513, 4096, 4097, 100000):
    buf, _ = o.random_vector(2 * n, 3); x, y = buf[:n], buf[n:]
    g = slab.dot(ctx.DenseVector(x), ctx.DenseVector(y)); w = o.dot(x, y)
    print(n, g == w)
dims = (16, 16, 16)
h = ctx.build_hierarchy(dims, 2)
b = ctx.DenseVector(h.n()); slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))
oh = o.build_hierarchy(*dims, 2); ob = o.level_mxv(oh, np.ones(oh.n))
for graphs in (True, False):
    ctx.set_graphs(graphs)
    try:
        res = slab.cg_solve(h, b, ctx.DenseVector(h.n(), 0.0), slab.CGConfig(max_iters=4, fixed_iterations=4))
        print("graphs", graphs, res.residual_history)
    except Exception as e:
        print("graphs", graphs, "error", e)
print("oracle", o.cg_solve(oh, ob, np.zeros(oh.n), max_iters=4, fixed_iterations=4).residual_history)
