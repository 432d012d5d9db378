"""The slab-staged product of csrc/plane_spmv.cu (y = A x of a regular box matrix: no matrix stream, the vector staged
through shared memory by bulk-async copies, three rows per column in flight so that a staged value is read once) must
give the bits of the row-by-row kernels and of the oracle: operations.hpp:116-125, :164-167; cg.hpp:122-123."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEFAULTS = {"spmv_planes": 1, "spmv_plane_min_rows": 4096, "spmv_plane_ty": 0, "spmv_plane_cz": 0, "spmv_plane_ns": 0}


@pytest.fixture()
def tuning():
    from paper_2304_08232_b200 import _capi

    def apply(**kw):
        for key, value in kw.items():
            _capi.set_tuning(key, value)

    yield apply
    apply(**DEFAULTS)


SHAPES = [(4, 4, 4), (8, 8, 8), (16, 12, 10), (6, 10, 14), (8, 5, 7), (12, 7, 9), (32, 8, 20), (64, 6, 6), (40, 24, 16),
          (10, 33, 5), (96, 20, 6), (14, 4, 37), (104, 9, 11)]


@pytest.mark.parametrize("dims", SHAPES)
def test_product_bitwise(slab, ctx, oracle, tuning, dims):
    """line lengths that are and are not multiples of the six columns a thread owns, boxes thinner than a tile,
    odd y/z extents (a last tile and a last chunk that are cut short)"""
    tuning(spmv_plane_min_rows=0)
    n = dims[0] * dims[1] * dims[2]
    x, _ = oracle.random_vector(n, 41)
    olvl = oracle.build_hierarchy(*dims, 1)
    lvl = ctx.build_hierarchy(dims, 1)
    assert lvl.A.format_info()["plane_phases"] == 1
    want = oracle.level_mxv(olvl, x)
    y = ctx.DenseVector(n, 7.0)
    slab.mxv(y, lvl.A, ctx.DenseVector(x))
    assert np.array_equal(y.values(), want), dims
    # the standalone stencil matrix takes the same path
    A = ctx.build_matrix(dims)
    y2 = ctx.DenseVector(n, -3.0)
    slab.mxv(y2, A, ctx.DenseVector(x))
    assert np.array_equal(y2.values(), want), dims


@pytest.mark.parametrize("shape", [dict(spmv_plane_ty=1, spmv_plane_cz=2, spmv_plane_ns=2), dict(spmv_plane_ty=2, spmv_plane_cz=3, spmv_plane_ns=3),
                                   dict(spmv_plane_ty=4, spmv_plane_cz=2, spmv_plane_ns=4), dict(spmv_plane_ty=8, spmv_plane_cz=16, spmv_plane_ns=6),
                                   dict(spmv_plane_ty=16, spmv_plane_cz=4, spmv_plane_ns=3), dict(spmv_plane_ty=32, spmv_plane_cz=6, spmv_plane_ns=8),
                                   dict(spmv_plane_ty=3, spmv_plane_cz=12, spmv_plane_ns=5), dict(spmv_plane_ty=6, spmv_plane_cz=64, spmv_plane_ns=2),
                                   dict(spmv_plane_ty=12, spmv_plane_cz=8, spmv_plane_ns=8), dict(spmv_plane_ty=24, spmv_plane_cz=24)])
def test_product_shapes_bitwise(slab, ctx, oracle, tuning, shape):
    """every ring depth / tile height / march length gives the same bits (slot reuse, planes outside the box entering
    a re-used slot, partial tiles and chunks)"""
    tuning(spmv_plane_min_rows=0)
    for dims in ((24, 22, 26), (12, 21, 13)):
        n = dims[0] * dims[1] * dims[2]
        x, _ = oracle.random_vector(n, 9)
        want = oracle.level_mxv(oracle.build_hierarchy(*dims, 1), x)
        tuning(**shape)
        lvl = ctx.build_hierarchy(dims, 1)
        y = ctx.DenseVector(n, 1.0)
        slab.mxv(y, lvl.A, ctx.DenseVector(x))
        assert np.array_equal(y.values(), want), (shape, dims)


def test_signed_zeros_and_non_finite_inputs_match_row_kernels(slab, ctx, tuning):
    """the zero padding stands in for absent neighbours: whatever the vector holds, the bits are those of the
    row-by-row kernels (which never touch an absent neighbour)"""
    tuning(spmv_plane_min_rows=0)
    dims = (8, 6, 10)
    n = dims[0] * dims[1] * dims[2]
    rng = np.random.default_rng(3)
    x = rng.standard_normal(n)
    x[rng.integers(0, n, 60)] = -0.0
    x[rng.integers(0, n, 60)] = 0.0
    x[rng.integers(0, n, 6)] = 1e300
    x[7] = np.inf
    x[n - 3] = np.nan
    x[n // 2: n // 2 + 40] = -0.0  # a whole neighbourhood of negative zeros: the sum must stay +0
    lvl = ctx.build_hierarchy(dims, 1)
    got = {}
    for on in (1, 0):
        tuning(spmv_planes=on)
        y = ctx.DenseVector(n, 5.0)
        slab.mxv(y, lvl.A, ctx.DenseVector(x))
        got[on] = y.values()
    assert np.array_equal(got[0].view(np.uint64), got[1].view(np.uint64))


def test_general_values_take_the_multiplying_kernel(slab, ctx, oracle, tuning):
    """a box matrix whose off-diagonal values are not all -1.0 (built from CSR, so nothing is known about its origin)
    stays with the row kernels; the stencil with its -1.0 entries takes the add-only variant. Both agree with the
    oracle's product of the same CSR."""
    tuning(spmv_plane_min_rows=0)
    dims = (12, 8, 6)
    ro, co, va = oracle.build_matrix(*dims)
    n = len(ro) - 1
    x, _ = oracle.random_vector(n, 77)
    want = oracle.mxv((ro, co, va), x)
    A = ctx.build_matrix(dims)
    y = ctx.DenseVector(n)
    slab.mxv(y, A, ctx.DenseVector(x))
    assert np.array_equal(y.values(), want)
    B = slab.SparseMatrix.from_csr(ctx, n, n, ro, co, va * 1.5)
    want_b = oracle.mxv((ro, co, va * 1.5), x)
    yb = ctx.DenseVector(n)
    slab.mxv(yb, B, ctx.DenseVector(x))
    assert np.array_equal(yb.values(), want_b)


def test_tree_mode_solve_uses_the_fused_dot_and_stays_within_tolerance(slab, ctx, tuning):
    """cg.hpp:122-123 on the product's epilogue: 64^3 history against the reference's golden, 1e-10 (tree dots differ
    from the reference's chunked order by rounding only); the same solve with the row kernels gives the same
    p'Ap up to the shape of the reduction tree"""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "history_64.json")))
    want = np.array([float.fromhex(v) for v in gold["residual_history_hex"]]) if "residual_history_hex" in gold \
        else np.array(gold["residual_history"])
    ctx.dot_mode = slab.DOT_TREE
    try:
        h = ctx.build_hierarchy((64, 64, 64), 4)
        b = ctx.DenseVector(h.n())
        slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))
        res = slab.cg_solve(h, b, ctx.DenseVector(h.n(), 0.0), slab.CGConfig(max_iters=50, fixed_iterations=50))
    finally:
        ctx.dot_mode = slab.DOT_EXACT
    got = np.array(res.residual_history)
    assert got.shape == want.shape
    assert np.max(np.abs(got - want) / want) <= 1e-10


def test_exact_mode_solve_bitwise(slab, ctx, tuning):
    """exact dots: the product alone changes kernels, the history must keep the reference's bits (16^3 golden)"""
    tuning(spmv_plane_min_rows=0)
    ctx.dot_mode = slab.DOT_EXACT
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "history_16.json")))
    h = ctx.build_hierarchy((16, 16, 16), 4)
    b = ctx.DenseVector(h.n())
    slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))
    res = slab.cg_solve(h, b, ctx.DenseVector(h.n(), 0.0), slab.CGConfig(max_iters=50, fixed_iterations=50))
    assert res.residual_history == gold["residual_history"]
