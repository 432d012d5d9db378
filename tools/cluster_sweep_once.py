"""One-level 16^3 (or argv[1]) symmetric sweep through the cluster kernel, a few times, eager: the target of an ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ctx = slab.Context(0)
ctx.set_graphs(False)
lvl = ctx.build_hierarchy((d, d, d), 1)
r, _ = ctx.random_vector(lvl.n(), 1)
z = ctx.DenseVector(lvl.n(), 0.0)
for _ in range(6):
    slab.mg_vcycle(lvl, z, r)
print("ok", float(z.values()[0]))
