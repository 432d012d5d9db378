"""Probe: time to build a 4-level hierarchy on the device, with and without the dictionary-coded copies."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08232_b200 as slab
ctx = slab.Context(0)
def build(d):
    ctx.sync(); t0 = time.perf_counter(); h = ctx.build_hierarchy((d,) * 3, 4); ctx.sync()
    return (time.perf_counter() - t0) * 1e3
for d in (104, 192, 256):
    build(d)  # warm-up (module load, allocator)
    coded = min(build(d) for _ in range(3))
    slab.set_tuning("pack_build", 0)
    plain = min(build(d) for _ in range(3))
    slab.set_tuning("pack_build", 1)
    print(d, "hierarchy build: %.1f ms with the coded copies, %.1f ms without" % (coded, plain))
