"""Probe: achieved HBM bandwidth of the vector kernels at the fine-level size of the 192^3 solve."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
ctx = slab.Context(0); ctx.dot_mode = slab.DOT_TREE
for d in (192, 256):
    n = d ** 3
    x, _ = ctx.random_vector(n, 1); y, _ = ctx.random_vector(n, 2); w = ctx.DenseVector(n, 0.0)
    def timed(f, reps=50):
        for _ in range(5): f()
        ctx.timer_start()
        for _ in range(reps): f()
        return ctx.timer_stop() / reps * 1e3  # us
    t_fill = timed(lambda: slab.set_all(w, 0.0))
    t_wax = timed(lambda: slab.waxpby(w, 1.0, x, 0.5, y))
    t_wax_alias = timed(lambda: slab.waxpby(w, 1.0, x, 0.5, w))
    t_dot = timed(lambda: slab.dot(x, y))   # includes the scalar read-back (a stream sync)
    mb = n * 8 / 1e6
    print(d, {"fill_us": round(t_fill, 1), "fill_GBs": round(mb / t_fill * 1e3), "waxpby_us": round(t_wax, 1),
              "waxpby_GBs": round(3 * mb / t_wax * 1e3), "waxpby_alias_GBs": round(3 * mb / t_wax_alias * 1e3),
              "dot_us": round(t_dot, 1), "dot_GBs": round(2 * mb / t_dot * 1e3)})
