"""GPU tests of the dictionary-coded matrix copy (packed.cu): whatever the format, whatever the kernel
shape, products and colour steps must return the same bits as the plain SELL kernels and as the CPU
oracle (operations.hpp:116-125 row sums in ascending column order, smoother.hpp:60-72 updates).

The packed kernels normally serve only launches of 65536 rows and more; the tests lower the thresholds
so that small matrices run through them, and restore the defaults afterwards.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEFAULTS = {"packed": 1, "packed_min_rows": 65536, "packed_multi_min_rows": 300000, "packed_rows": 2,
            "packed_rows_spmv": 3, "packed_batch": 2, "packed_block": 256}


@pytest.fixture()
def tune(slab):
    from paper_2304_08232_b200 import _capi

    def apply(**kw):
        for key, value in {**DEFAULTS, **kw}.items():
            _capi.set_tuning(key, value)

    # these tests are about the per-colour kernels: keep small levels off the one-launch sweep (sweep_cluster.cu)
    _capi.set_tuning("cluster_rows", 0)
    yield apply
    apply()
    _capi.set_tuning("cluster_rows", 384)


# kernel shapes: (rows per thread of colour steps, of products, words per batch, block)
SHAPES = [dict(packed_rows=1, packed_rows_spmv=1, packed_batch=1), dict(packed_rows=1, packed_rows_spmv=1, packed_batch=2),
          dict(packed_rows=2, packed_rows_spmv=2), dict(packed_rows=3, packed_rows_spmv=3, packed_block=128),
          dict(packed_rows=4, packed_rows_spmv=4)]


def csr_from_rows(rows, n):
    ro = np.zeros(n + 1, dtype=np.uint64)
    co, va = [], []
    for i, entries in enumerate(rows):
        for c in sorted(entries):
            co.append(c)
            va.append(entries[c])
        ro[i + 1] = len(co)
    return ro, np.array(co, dtype=np.uint64), np.array(va, dtype=np.float64)


def banded(n, offsets, values, diag):
    """every row i has diag at i and values[k] at i + offsets[k] when inside [0, n)"""
    rows = []
    for i in range(n):
        entries = {i: diag}
        for off, v in zip(offsets, values):
            if 0 <= i + off < n:
                entries[i + off] = v
        rows.append(entries)
    return rows


def run_level_ops(slab, ctx, lvl, x, r, z0):
    """product, masked product, one symmetric sweep: everything the packed kernels implement"""
    n = lvl.n()
    out = {}
    y = ctx.DenseVector(n, 0.0)
    slab.mxv(y, lvl.A, ctx.DenseVector(x))
    out["mxv"] = y.values()
    members = lvl.color_members(lvl.num_colors - 1)
    mask = slab.IndexMask(ctx, n, members)
    ym = ctx.DenseVector(np.full(n, 7.25))
    slab.mxv(ym, mask, lvl.A, ctx.DenseVector(x))
    out["masked"] = ym.values()
    z = ctx.DenseVector(z0)
    slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r))
    out["symmetric"] = z.values()
    return out


def test_stencil_level_formats(slab, ctx):
    """the 27-point operator has 27 (offset, value) pairs: width class 27, 28 dictionary entries, no escapes;
    rows one x-line apart repeat their codes (64 rows per line and colour... 32 here: one slice)"""
    h = ctx.build_hierarchy((64, 64, 64), 3)
    for info in (h.A.format_info(), h.format_info()):
        assert info["packed"] == 1 and info["width_class"] == 27 and info["dict_size"] == 28
        assert info["escaped_rows"] == 0 and info["stride"] >= 1
        assert info["packed_bytes"] * 8 < info["plain_bytes"]  # 32 B per row against 324 B
    coarse = h.coarser.coarser  # 16^3: x-lines of 8 rows per colour, codes repeat every slice as well
    assert coarse.format_info()["packed"] == 1


@pytest.mark.parametrize("dims", [(16, 16, 16), (10, 6, 14), (5, 7, 9), (32, 8, 4)])
def test_packed_stencil_kernels_bitwise(slab, ctx, oracle, tune, dims):
    """plain vs packed (every kernel shape) vs oracle on even, odd and skewed grids"""
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(3 * n, 5)
    x, r, z0 = buf[:n], buf[n:2 * n], buf[2 * n:]
    olvl = oracle.build_hierarchy(*dims, 1)
    want = {"mxv": oracle.level_mxv(olvl, x), "symmetric": oracle.rbgs_symmetric(olvl, z0, r)}
    levels = [ctx.build_hierarchy(dims, 1), slab.ProblemLevel(ctx, oracle.build_matrix(*dims))]
    for lvl in levels:
        assert lvl.format_info()["packed"] == 1
        tune(packed=0)
        plain = run_level_ops(slab, ctx, lvl, x, r, z0)
        assert np.array_equal(plain["mxv"], want["mxv"]) and np.array_equal(plain["symmetric"], want["symmetric"])
        for shape in SHAPES:
            tune(packed=1, packed_min_rows=0, packed_multi_min_rows=0, **shape)
            got = run_level_ops(slab, ctx, lvl, x, r, z0)
            for key in plain:
                assert np.array_equal(got[key], plain[key]), (key, shape)


def test_packed_solve_history_bitwise(slab, ctx, tune):
    """a whole 4-level solve (fused transfers included) from the packed copies equals the plain one, in
    exact-dot mode bit for bit and with the reference's golden history"""
    import json
    import os

    ctx.dot_mode = slab.DOT_EXACT
    dims = (16, 16, 16)
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "history_16.json")))
    want = gold["residual_history"]
    h = ctx.build_hierarchy(dims, 4)
    b = ctx.DenseVector(h.n())
    slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))  # b = A*1
    x0 = ctx.DenseVector(h.n(), 0.0)
    cfg = slab.CGConfig(max_iters=50, fixed_iterations=50)
    tune(packed=0)
    plain = slab.cg_solve(h, b, x0, cfg)
    assert plain.residual_history == want
    for shape in SHAPES:
        tune(packed=1, packed_min_rows=0, packed_multi_min_rows=0, **shape)
        got = slab.cg_solve(h, b, x0, cfg)
        assert got.residual_history == want, shape
        assert np.array_equal(got.solution.values(), plain.solution.values())


def test_general_matrices_pack_when_they_repeat_and_stay_exact(slab, ctx, oracle, tune):
    """banded matrices with a handful of distinct pairs pack; a few irregular rows become escapes that
    are read from the plain arrays; results equal the oracle bitwise either way"""
    n = 700
    rng = np.random.default_rng(3)
    rows = banded(n, [-17, -3, -1, 1, 3, 17], [-1.0, -0.5, -2.0, -2.0, -0.5, -1.0], 9.0)
    irregular = sorted(rng.choice(n, size=60, replace=False))
    for i in irregular:  # five entries each that no other row has: more new pairs than the dictionary holds
        for c in rng.choice(n, size=5, replace=False):
            rows[i][int(c)] = float(rng.random()) - 0.5
        rows[i][i] = 9.0
    csr = csr_from_rows(rows, n)
    lvl = slab.ProblemLevel(ctx, csr)
    info = lvl.A.format_info()
    assert info["packed"] == 1 and info["width_class"] == 16 and info["dict_size"] == 255
    assert 0 < info["escaped_rows"] <= len(irregular)
    cinfo = lvl.format_info()
    assert cinfo["packed"] == 1 and 0 < cinfo["escaped_rows"] <= len(irregular)
    olvl = oracle.level_from_csr(*csr)
    buf, _ = oracle.random_vector(3 * n, 9)
    x, r, z0 = buf[:n], buf[n:2 * n], buf[2 * n:]
    for shape in SHAPES:
        tune(packed=1, packed_min_rows=0, packed_multi_min_rows=0, **shape)
        got = run_level_ops(slab, ctx, lvl, x, r, z0)
        assert np.array_equal(got["mxv"], oracle.level_mxv(olvl, x)), shape
        assert np.array_equal(got["symmetric"], oracle.rbgs_symmetric(olvl, z0, r)), shape


def test_matrices_that_do_not_repeat_keep_the_plain_format(slab, ctx, oracle, tune):
    """random values: every entry is its own pair, the dictionary overflows, the matrix stays plain;
    rows wider than 64 entries are not coded at all"""
    n = 300
    rng = np.random.default_rng(5)
    rows = [{i: 10.0 + float(rng.random())} for i in range(n)]
    for i in range(n):
        for c in rng.choice(n, size=6, replace=False):
            rows[i][int(c)] = float(rng.random()) - 0.5
        rows[i][i] = 10.0 + float(rng.random())
    A = slab.SparseMatrix.from_csr(ctx, n, n, *csr_from_rows(rows, n))
    assert A.format_info()["packed"] == 0 and A.format_info()["packed_bytes"] == 0
    wide = banded(200, list(range(1, 71)), [-0.01] * 70, 4.0)
    W = slab.SparseMatrix.from_csr(ctx, 200, 200, *csr_from_rows(wide, 200))
    assert W.format_info()["packed"] == 0
    tune(packed=1, packed_min_rows=0, packed_multi_min_rows=0)
    x, _ = oracle.random_vector(200, 1)
    y = ctx.DenseVector(200, 0.0)
    slab.mxv(y, W, ctx.DenseVector(x))
    assert np.array_equal(y.values(), oracle.mxv(csr_from_rows(wide, 200), x))


@pytest.mark.parametrize("width,cls", [(12, 16), (30, 32), (40, 64)])
def test_width_classes(slab, ctx, oracle, tune, width, cls):
    """rows of 12 / 30 / 40 entries land in the 16 / 32 / 64 classes; shorter rows at the ends are ragged"""
    n = 500
    offsets = [k for k in range(-(width // 2), width - width // 2) if k != 0]
    values = [-1.0 / (1 + abs(k)) for k in offsets]
    csr = csr_from_rows(banded(n, offsets, values, 50.0), n)
    lvl = slab.ProblemLevel(ctx, csr)
    assert lvl.A.format_info()["width_class"] == cls and lvl.A.format_info()["escaped_rows"] == 0
    olvl = oracle.level_from_csr(*csr)
    buf, _ = oracle.random_vector(3 * n, 21)
    x, r, z0 = buf[:n], buf[n:2 * n], buf[2 * n:]
    for shape in SHAPES[1:4]:
        tune(packed=1, packed_min_rows=0, packed_multi_min_rows=0, **shape)
        got = run_level_ops(slab, ctx, lvl, x, r, z0)
        assert np.array_equal(got["mxv"], oracle.level_mxv(olvl, x)), shape
        assert np.array_equal(got["symmetric"], oracle.rbgs_symmetric(olvl, z0, r)), shape


def test_pack_build_can_be_switched_off(slab, ctx, tune):
    from paper_2304_08232_b200 import _capi

    _capi.set_tuning("pack_build", 0)
    try:
        h = ctx.build_hierarchy((8, 8, 8), 1)
        assert h.format_info()["packed"] == 0 and h.A.format_info()["packed"] == 0
    finally:
        _capi.set_tuning("pack_build", 1)


def test_plain_arrays_can_be_dropped(slab, ctx, tune):
    """keep_plain = 0: matrices created afterwards keep only their coded copy (no escaped rows here), always
    run the coded kernels — thresholds or not — and still reproduce the reference history bit for bit"""
    import json
    import os
    from paper_2304_08232_b200 import _capi

    ctx.dot_mode = slab.DOT_EXACT
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "history_16.json")))
    _capi.set_tuning("keep_plain", 0)
    try:
        h = ctx.build_hierarchy((16, 16, 16), 4)
    finally:
        _capi.set_tuning("keep_plain", 1)
    for info in (h.A.format_info(), h.format_info(), h.coarser.format_info()):
        assert info["packed"] == 1 and info["plain_bytes"] < info["packed_bytes"]  # only the slice table is left
    b = ctx.DenseVector(h.n())
    slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))
    res = slab.cg_solve(h, b, ctx.DenseVector(h.n(), 0.0), slab.CGConfig(max_iters=50, fixed_iterations=50))
    assert res.residual_history == gold["residual_history"]
    with pytest.raises(slab.InvalidArgument):
        h.A.csr()
    kept = ctx.build_hierarchy((16, 16, 16), 1)  # created after the knob went back: plain arrays present
    assert kept.A.format_info()["plain_bytes"] > kept.A.format_info()["packed_bytes"]
    kept.A.csr()


def test_microbench_256_checksums_with_both_kernel_families(slab, ctx, tune):
    """BASELINE.json configs[2] at its real size (256^3, one level): y = A*x for x ~ U(-1,1) from seed 0, then one
    coloured symmetric sweep on r = b - A*x from z = 0 (b = A*1). The four checksums (the reference's 4096-chunk
    ordered dot) equal the reference's doubles with the coded kernels (products with 3 rows per thread, colour
    steps with 2, the sweep turnaround) and with the plain SELL kernels."""
    import json
    import os

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "micro_256.json")))
    ctx.dot_mode = slab.DOT_EXACT
    lvl = ctx.build_hierarchy((256, 256, 256), 1)
    n = lvl.n()
    x, _ = ctx.random_vector(n, 0)
    b = ctx.DenseVector(n)
    slab.mxv(b, lvl.A, ctx.DenseVector(n, 1.0))
    for packed in (1, 0):
        tune(packed=packed)
        y = ctx.DenseVector(n)
        slab.mxv(y, lvl.A, x)
        r = ctx.DenseVector(n)
        slab.waxpby(r, 1.0, b, -1.0, y)
        z = ctx.DenseVector(n, 0.0)
        slab.rbgs_symmetric(lvl, z, r)
        got = {"dot_yy": slab.dot(y, y), "dot_xy": slab.dot(x, y), "dot_zz_after_symmetric": slab.dot(z, z),
               "dot_rz_after_symmetric": slab.dot(r, z)}
        for key, value in got.items():
            assert value == float.fromhex(gold[key + "_hex"]), (key, packed)


@pytest.mark.parametrize("seed", range(12))
def test_random_banded_matrices_coded_equals_plain(slab, ctx, tune, seed):
    """randomised shapes: row counts that are no multiple of 32, 2 to 60 bands at random offsets with random
    values (so the width class, the dictionary size, the stride vote and the ragged ends all vary), a few rows
    with private entries (escapes); every coded kernel shape must equal the plain kernels bit for bit"""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(40, 1500))
    nbands = int(rng.integers(2, 61))
    offsets = sorted(set(int(o) for o in rng.integers(-min(n - 1, 400), min(n - 1, 400) + 1, size=nbands) if o != 0))
    values = [float(rng.integers(-8, 9)) / 4.0 or -0.25 for _ in offsets]
    rows = banded(n, offsets, values, float(len(offsets)) * 3.0 + 1.0)
    for i in rng.choice(n, size=int(rng.integers(0, max(1, n // 40))), replace=False):
        rows[int(i)][int(rng.integers(0, n))] = float(rng.random()) + 0.125
        rows[int(i)][int(i)] = float(len(offsets)) * 3.0 + 1.0
    csr = csr_from_rows(rows, n)
    lvl = slab.ProblemLevel(ctx, csr)
    x, _ = ctx.random_vector(n, 5 + seed)
    r, _ = ctx.random_vector(n, 6 + seed)
    z0, _ = ctx.random_vector(n, 7 + seed)
    tune(packed=0)
    plain = run_level_ops(slab, ctx, lvl, x.values(), r.values(), z0.values())
    for shape in SHAPES:
        tune(packed=1, packed_min_rows=0, packed_multi_min_rows=0, **shape)
        got = run_level_ops(slab, ctx, lvl, x.values(), r.values(), z0.values())
        for key in plain:
            assert np.array_equal(got[key], plain[key]), (key, shape, lvl.A.format_info(), lvl.format_info())
