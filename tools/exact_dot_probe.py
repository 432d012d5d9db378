"""Probe: cost of the exact (4096-chunk ordered) dot against the tree dot at the 192^3 vector length, and the
whole solve in both modes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
ctx = slab.Context(0)
n = 192 ** 3
x, _ = ctx.random_vector(n, 1); y, _ = ctx.random_vector(n, 2)
for mode, name in ((slab.DOT_EXACT, "exact"), (slab.DOT_TREE, "tree")):
    ctx.dot_mode = mode
    for _ in range(3): slab.dot(x, y)
    ctx.timer_start()
    for _ in range(20): v = slab.dot(x, y)
    print(name, "dot incl. scalar read-back: %.1f us" % (ctx.timer_stop() / 20 * 1e3), v.hex())
h = ctx.build_hierarchy((192,) * 3, 4)
b = ctx.DenseVector(n); slab.mxv(b, h.A, ctx.DenseVector(n, 1.0)); x0 = ctx.DenseVector(n, 0.0); out = ctx.DenseVector(n)
cfg = slab.CGConfig(max_iters=50, fixed_iterations=50)
for mode, name in ((slab.DOT_EXACT, "exact"), (slab.DOT_TREE, "tree")):
    ctx.dot_mode = mode
    for _ in range(2): slab.cg_solve(h, b, x0, cfg, out=out)
    print(name, "solve: %.2f ms" % min(slab.cg_solve(h, b, x0, cfg, out=out).solve_ms for _ in range(3)))
