#!/usr/bin/env python
"""Kernel microbench (BASELINE.json configs[2] and tuning sweeps), run on the GPU box:

    python tools/kernel_microbench.py [--dims 256 256 256] [--variants 0 1 2 ...] [--check]

(a) SpMV y = A*x with x ~ U(-1,1) from Lcg64(0); (b) one coloured symmetric GS sweep on
r = b - A*x from z = 0 (b = A*1). Reports device time (CUDA events on the library's stream, L2
not flushed: the matrix alone is far larger than L2) and achieved algorithmic GB/s against the
measured HBM peak. With --check at 256^3 the dot-product checksums are compared with the
reference values recorded in tests/golden/micro_256.json.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_08232_b200 as slab  # noqa: E402
from paper_2304_08232_b200 import _capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, default=[256, 256, 256])
    ap.add_argument("--variants", type=int, nargs="*", default=[0])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--json", default=None)
    ap.add_argument("--sets", nargs="*", default=None,
                    help="tuning sets to time, each 'key=value,key=value' (slab_set_tuning keys), e.g. packed=0 packed=1,packed_block=512")
    args = ap.parse_args()
    dims = tuple(args.dims)
    peak = 6551.0
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peak = float(json.load(open(pk))["hbm_gbs"])

    ctx = slab.Context(0)
    lvl = ctx.build_hierarchy(dims, 1)
    n = lvl.n()
    nnz = lvl.A.nnz()
    x, _ = ctx.random_vector(n, 0)
    y = ctx.DenseVector(n)
    ones = ctx.DenseVector(n, 1.0)
    b = ctx.DenseVector(n)
    slab.mxv(b, lvl.A, ones)
    slab.mxv(y, lvl.A, x)
    r = ctx.DenseVector(n)
    slab.waxpby(r, 1.0, b, -1.0, y)
    z = ctx.DenseVector(n, 0.0)
    spmv_bytes = 12 * nnz + 16 * n
    gs_bytes = 2 * (12 * nnz + 32 * n)
    out = {"dims": dims, "n": n, "nnz": nnz, "peak_gbs": peak, "results": []}

    if args.check:
        slab.rbgs_symmetric(lvl, z, r)
        sums = {"dot_yy": slab.dot(y, y), "dot_xy": slab.dot(x, y), "dot_zz_after_symmetric": slab.dot(z, z),
                "dot_rz_after_symmetric": slab.dot(r, z)}
        out["checksums"] = sums
        gpath = os.path.join(ROOT, "tests", "golden", "micro_256.json")
        if dims == (256, 256, 256) and os.path.exists(gpath):
            gold = json.load(open(gpath))
            ok = all(sums[k] == float.fromhex(gold[k + "_hex"]) for k in sums)
            out["checksums_match_reference_bitwise"] = ok
            print("checksums match the reference bitwise:", ok, sums)

    runs = [("stream_variant=%d" % v) for v in args.variants] if args.sets is None else args.sets
    defaults = {"packed": 1, "packed_block": 256, "packed_batch": 2, "packed_min_rows": 65536, "packed_rows": 2,
                "packed_rows_spmv": 3, "packed_multi_min_rows": 300000, "stream_rows": 200000, "stream_variant": 2}
    for variant in runs:
        for key, value in defaults.items():  # every set starts from the defaults
            _capi.set_tuning(key, value)
        for pair in variant.split(","):
            key, value = pair.split("=")
            _capi.set_tuning(key, int(value))
        for _ in range(3):
            slab.mxv(y, lvl.A, x)
        ctx.timer_start()
        for _ in range(args.reps):
            slab.mxv(y, lvl.A, x)
        spmv_ms = ctx.timer_stop() / args.reps
        slab.set_all(z, 0.0)
        for _ in range(2):
            slab.rbgs_symmetric(lvl, z, r)
        ctx.timer_start()
        for _ in range(args.reps):
            slab.rbgs_symmetric(lvl, z, r)
        gs_ms = ctx.timer_stop() / args.reps
        res = {"variant": variant, "spmv_ms": spmv_ms, "spmv_gbs": spmv_bytes / spmv_ms / 1e6,
               "spmv_frac": spmv_bytes / spmv_ms / 1e6 / peak, "gs_sym_ms": gs_ms, "gs_gbs": gs_bytes / gs_ms / 1e6,
               "gs_frac": gs_bytes / gs_ms / 1e6 / peak}
        out["results"].append(res)
        print(json.dumps(res))
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
