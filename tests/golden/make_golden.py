"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference headers.

Run in the build container (where /root/reference exists):  python tests/golden/make_golden.py [--big] [--scale]
It loads oracle/_ref/libslab_ref.so (oracle/ref_shim.cpp compiled against
/root/reference/proj/include by oracle/Makefile) and records

  history_<n>.json     residual histories of BASELINE.json configs[0..1] (16^3, 64^3; 4 levels,
                       50 fixed iterations, b = A*1, x0 = 0) and, with --big, 104^3
  small_cases.json     seeded small-case vectors: SpMV, masked/transposed mxv, dot, waxpby,
                       forward/backward/symmetric smoothing, a 2-level V-cycle, LCG outputs
  micro_256.json       (--big) the 256^3 microbench checksums of BASELINE.md §4
  history_208x104x104.json, history_208x208x104.json, history_208x208x208.json
                       (--scale) histories on the global grids of the 2-, 4- and 8-rank 104^3-per-GPU runs

Nothing on the GPU box reads /root/reference: the tests read these JSON files only.
Doubles are stored as hex strings (float.hex) so that the fixtures are bit-exact.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def hexlist(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(obj, fh, indent=0, separators=(",", ":"))
        fh.write("\n")
    print("wrote", name)


def history(ref, n, levels=4, iters=50):
    dims = (n, n, n) if isinstance(n, int) else tuple(n)
    h = ref.build_hierarchy(*dims, levels)
    b = ref.level_mxv(h, np.ones(h.n))
    res = ref.cg_solve(h, b, np.zeros(h.n), max_iters=iters, fixed_iterations=iters)
    stats = []
    lvl = h
    while lvl is not None:
        stats.append({"n": lvl.n, "nnz": lvl.nnz, "nnz_visited": lvl.nnz_visited})
        lvl = lvl.coarser
    return {
        "source": "reference headers via oracle/_ref (cg.hpp:77-142)",
        "dims": list(dims), "levels": levels, "rhs": "A*ones", "x0": "zeros",
        "iterations": res.iterations,
        "residual_history": res.residual_history,
        "residual_history_hex": hexlist(res.residual_history),
        "solution_checksum_dot_xx_hex": float(ref.dot(res.solution, res.solution)).hex(),
        "levels_stats": stats,
    }


def small_cases(ref):
    out = {"source": "reference headers via oracle/_ref"}
    # rng.hpp first outputs (test_algebra.cpp:382-388)
    out["lcg_first_seed0"] = ref.lcg_next(0)
    out["lcg_first_seed1"] = ref.lcg_next(1)
    v, state = ref.random_vector(8, 42)
    out["random_vector_seed42_n8_hex"] = hexlist(v)
    out["random_vector_seed42_state"] = state

    # 6x4x8 stencil: SpMV, masked mxv, transpose, dot, waxpby
    dims = (6, 4, 8)
    n = dims[0] * dims[1] * dims[2]
    csr = ref.build_matrix(*dims)
    x, st = ref.random_vector(n, 7)
    y = ref.mxv(csr, x)
    out["spmv_6x4x8"] = {"dims": dims, "x_seed": 7, "y_hex": hexlist(y), "nnz": int(csr[0][-1])}
    members = np.arange(1, n, 3, dtype=np.uint64)
    y0, _ = ref.random_vector(n, 9)
    ym = ref.mxv(csr, x, mask=members, y=y0)
    out["masked_mxv_6x4x8"] = {"members_start": 1, "members_step": 3, "y0_seed": 9, "y_hex": hexlist(ym)}
    xx, _ = ref.random_vector(20000, 3)
    yy, _ = ref.random_vector(20000, 4)
    out["dot_n20000"] = {"x_seed": 3, "y_seed": 4, "dot_hex": float(ref.dot(xx, yy)).hex(),
                         "dot_xx_hex": float(ref.dot(xx, xx)).hex()}
    out["dot_n4096"] = {"dot_hex": float(ref.dot(xx[:4096], yy[:4096])).hex()}
    out["dot_n4097"] = {"dot_hex": float(ref.dot(xx[:4097], yy[:4097])).hex()}
    out["dot_n100"] = {"dot_hex": float(ref.dot(xx[:100], yy[:100])).hex()}
    out["waxpby_n1000"] = {"alpha": 0.3, "beta": -1.7, "w_hex": hexlist(ref.waxpby(0.3, xx[:1000], -1.7, yy[:1000]))}

    # restriction transpose (refinement) on 4x4x4
    rc = ref.build_restriction_cols(4, 4, 4)
    out["restriction_cols_4x4x4"] = [int(c) for c in rc]

    # smoother on 4x4x4 with seed 42 (test_smoother.cpp:70-84) and on 5x7x9 (odd dims)
    for dims, seed in (((4, 4, 4), 42), ((5, 7, 9), 43)):
        lvl = ref.level_from_csr(*ref.build_matrix(*dims))
        nn = lvl.n
        buf, _ = ref.random_vector(2 * nn, seed)
        r, z = buf[:nn], buf[nn:]
        key = "smoother_%dx%dx%d" % dims
        out[key] = {
            "seed": seed, "num_colors": lvl.num_colors,
            "color_sizes": [len(lvl.color_members(k)) for k in range(lvl.num_colors)],
            "color_nnz": [lvl.color_nnz(k) for k in range(lvl.num_colors)],
            "forward_hex": hexlist(ref.rbgs_forward(lvl, z, r)),
            "backward_hex": hexlist(ref.rbgs_backward(lvl, z, r)),
            "symmetric2_hex": hexlist(ref.rbgs_symmetric(lvl, z, r, 2)),
        }

    # two-level V-cycle on 8^3 from zero (test_multigrid.cpp:49-71) and 3-level with odd coarsest
    for dims, levels, seed in (((8, 8, 8), 2, 7), ((12, 12, 12), 3, 8)):
        h = ref.build_hierarchy(*dims, levels)
        r, _ = ref.random_vector(h.n, seed)
        z = ref.mg_vcycle(h, np.zeros(h.n), r)
        stats = []
        lvl = h
        while lvl is not None:
            stats.append(lvl.nnz_visited)
            lvl = lvl.coarser
        out["vcycle_%dx%dx%d_L%d" % (*dims, levels)] = {"seed": seed, "z_hex": hexlist(z), "nnz_visited": stats}

    # 13^3 colour sizes
    lvl = ref.level_from_csr(*ref.build_matrix(13, 13, 13))
    out["color_sizes_13"] = [len(lvl.color_members(k)) for k in range(lvl.num_colors)]
    return out


def micro_256(ref):
    n = 256
    csr = ref.build_matrix(n, n, n)
    N = n ** 3
    x, _ = ref.random_vector(N, 0)
    y = ref.mxv(csr, x)
    out = {"source": "reference headers via oracle/_ref", "dims": [n, n, n], "x_seed": 0,
           "dot_yy_hex": float(ref.dot(y, y)).hex(), "dot_xy_hex": float(ref.dot(x, y)).hex()}
    b = ref.mxv(csr, np.ones(N))
    r = ref.waxpby(1.0, b, -1.0, y)
    lvl = ref.level_from_csr(*csr)
    del csr
    z = ref.rbgs_symmetric(lvl, np.zeros(N), r, 1)
    out["dot_zz_after_symmetric_hex"] = float(ref.dot(z, z)).hex()
    out["dot_rz_after_symmetric_hex"] = float(ref.dot(r, z)).hex()
    return out


if __name__ == "__main__":
    ref = Oracle("reference")
    assert ref.kind == "reference"
    dump("small_cases.json", small_cases(ref))
    for n in (16, 64):
        dump(f"history_{n}.json", history(ref, n))
    if "--big" in sys.argv:
        dump("history_104.json", history(ref, 104))
        dump("micro_256.json", micro_256(ref))
    if "--scale" in sys.argv:
        # the GLOBAL grids of the weak-scaled 104^3-per-GPU runs (BASELINE.json configs[3]: process grids 2x1x1, 2x2x1,
        # 2x2x2): the oracle of an N-rank solve is the single-process solve on the global grid
        for dims in ((208, 104, 104), (208, 208, 104), (208, 208, 208)):
            dump("history_%dx%dx%d.json" % dims, history(ref, dims))
