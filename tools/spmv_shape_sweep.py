#!/usr/bin/env python
"""Times the slab-staged product (plane_spmv.cu) over tile shapes: python tools/spmv_shape_sweep.py [--dims 192]"""
import argparse
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_08232_b200 as slab  # noqa: E402
from paper_2304_08232_b200 import _capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs="+", default=[192])
    ap.add_argument("--ty", type=int, nargs="+", default=[0, 4, 6, 8, 12, 16])
    ap.add_argument("--cz", type=int, nargs="+", default=[0, 8, 12, 16, 24, 32, 48, 64])
    ap.add_argument("--ns", type=int, nargs="+", default=[0, 3, 6])
    args = ap.parse_args()
    dims = tuple(args.dims * 3) if len(args.dims) == 1 else tuple(args.dims)
    ctx = slab.Context(0)
    lvl = ctx.build_hierarchy(dims, 1)
    n = lvl.n()
    x, _ = ctx.random_vector(n, 0)
    y = ctx.DenseVector(n)
    rows = []
    for ty, cz, ns in itertools.product(args.ty, args.cz, args.ns):
        if (ty == 0) != (cz == 0):
            continue
        _capi.set_tuning("spmv_plane_ty", ty)
        _capi.set_tuning("spmv_plane_cz", cz)
        _capi.set_tuning("spmv_plane_ns", ns)
        try:
            for _ in range(3):
                slab.mxv(y, lvl.A, x)
            ctx.timer_start()
            for _ in range(20):
                slab.mxv(y, lvl.A, x)
            us = ctx.timer_stop() / 20 * 1e3
        except Exception as exc:  # a shape that does not fit
            print(ty, cz, ns, "failed:", str(exc)[:80])
            continue
        rows.append((us, ty, cz, ns))
        print(f"ty {ty:2d} cz {cz:3d} ns {ns}: {us:7.2f} us  {16 * n / us / 1e3:7.0f} GB/s")
    rows.sort()
    print("best:", rows[:5])


if __name__ == "__main__":
    main()
