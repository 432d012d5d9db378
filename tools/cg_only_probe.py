import sys, os
sys.path.insert(0, '/root/repo')
import paper_2304_08232_b200 as slab
ctx = slab.Context(0); ctx.dot_mode = slab.DOT_TREE
for d in (192, 104):
    h = ctx.build_hierarchy((d,)*3, 4)
    n = h.n(); b = ctx.DenseVector(n); slab.mxv(b, h.A, ctx.DenseVector(n, 1.0)); x0 = ctx.DenseVector(n, 0.0); x = ctx.DenseVector(n)
    for pre in (True, False):
        cfg = slab.CGConfig(max_iters=50, fixed_iterations=50, use_preconditioner=pre)
        for _ in range(2): slab.cg_solve(h, b, x0, cfg, out=x)
        t = min(slab.cg_solve(h, b, x0, cfg, out=x).solve_ms for _ in range(5))
        print(d, "preconditioned" if pre else "cg only", round(t, 3), "ms ->", round(t / 50 * 1e3, 1), "us/iter")
