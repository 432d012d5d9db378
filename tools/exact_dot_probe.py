"""Probe: cost of the exact (4096-chunk ordered) dot against the tree dot for growing vectors (1 chunk, one chunk
per SM, the 192^3 vector), and the whole 192^3 solve in both modes. Times include the scalar read-back (~22 us)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
ctx = slab.Context(0)
for n in (4096, 4096 * 148, 4096 * 148 * 4, 192 ** 3):
    x, _ = ctx.random_vector(n, 1); y, _ = ctx.random_vector(n, 2)
    row = {"n": n, "chunks": (n + 4095) // 4096}
    for mode, name in ((slab.DOT_EXACT, "exact_us"), (slab.DOT_TREE, "tree_us")):
        ctx.dot_mode = mode
        for _ in range(3): slab.dot(x, y)
        ctx.timer_start()
        for _ in range(20): slab.dot(x, y)
        row[name] = round(ctx.timer_stop() / 20 * 1e3, 1)
    print(row)
if "--solve" in sys.argv:
    n = 192 ** 3
    h = ctx.build_hierarchy((192,) * 3, 4)
    b = ctx.DenseVector(n); slab.mxv(b, h.A, ctx.DenseVector(n, 1.0)); x0 = ctx.DenseVector(n, 0.0); out = ctx.DenseVector(n)
    cfg = slab.CGConfig(max_iters=50, fixed_iterations=50)
    for mode, name in ((slab.DOT_EXACT, "exact"), (slab.DOT_TREE, "tree")):
        ctx.dot_mode = mode
        for _ in range(2): slab.cg_solve(h, b, x0, cfg, out=out)
        print(name, "solve: %.2f ms" % min(slab.cg_solve(h, b, x0, cfg, out=out).solve_ms for _ in range(3)))
