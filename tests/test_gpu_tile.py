"""The shared-memory-staged kernels of csrc/tile.cu (bulk-async copies of plane slabs into a ring, one launch per
pair of colours that differ in the parity of x, rows as 32-bit masks over the 27 offsets) must give the bits of the
colour-by-colour steps and of the oracle: smoother.hpp:60-113, multigrid.hpp:87-116, operations.hpp:116-125."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEFAULTS = {"planes": 1, "tile": 1, "tile_min_rows": 200000, "tile_ty": 0, "tile_cz": 0, "tile_ns": 0}


@pytest.fixture()
def tuning():
    from paper_2304_08232_b200 import _capi

    def apply(**kw):
        for key, value in kw.items():
            _capi.set_tuning(key, value)

    yield apply
    apply(**DEFAULTS)


SHAPES = [(4, 4, 4), (8, 8, 8), (16, 12, 10), (6, 10, 14), (8, 5, 7), (12, 7, 9), (32, 8, 20), (64, 6, 6), (40, 24, 16)]


@pytest.mark.parametrize("dims", SHAPES)
def test_sweeps_bitwise(slab, ctx, oracle, tuning, dims):
    """forward, backward and symmetric sweeps through the pair launches: even and odd y/z extents (unequal colour
    sizes), boxes thinner than a tile, x-lines shorter and longer than a warp of pairs"""
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(2 * n, 17)
    r, z0 = buf[:n], buf[n:]
    olvl = oracle.build_hierarchy(*dims, 1)
    tuning(planes=0, tile_min_rows=0)
    lvl = ctx.build_hierarchy(dims, 1)
    assert lvl.format_info()["mask_bytes"] > 0
    for name in ("rbgs_forward", "rbgs_backward", "rbgs_symmetric"):
        want = getattr(oracle, name)(olvl, z0, r)
        z = ctx.DenseVector(z0)
        getattr(slab, name)(lvl, z, ctx.DenseVector(r))
        assert np.array_equal(z.values(), want), (name, dims)


@pytest.mark.parametrize("shape", [dict(tile_ty=1, tile_cz=1, tile_ns=4), dict(tile_ty=2, tile_cz=3, tile_ns=5),
                                   dict(tile_ty=4, tile_cz=2, tile_ns=7), dict(tile_ty=8, tile_cz=16, tile_ns=6),
                                   dict(tile_ty=2, tile_cz=5, tile_ns=16)])
def test_tile_shapes_bitwise(slab, ctx, oracle, tuning, shape):
    """every ring depth / tile height / march length gives the same bits (slot reuse, partial tiles and chunks)"""
    dims = (24, 22, 26)
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(2 * n, 5)
    r, z0 = buf[:n], buf[n:]
    want = oracle.rbgs_symmetric(oracle.build_hierarchy(*dims, 1), z0, r)
    tuning(planes=0, tile_min_rows=0, **shape)
    lvl = ctx.build_hierarchy(dims, 1)
    z = ctx.DenseVector(z0)
    slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r))
    assert np.array_equal(z.values(), want), shape


def test_tile_equals_per_colour_launches_two_sweeps(slab, ctx, oracle, tuning):
    dims = (48, 20, 12)
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(2 * n, 23)
    r, z0 = buf[:n], buf[n:]
    lvl = ctx.build_hierarchy(dims, 1)
    got = {}
    for rows in (0, 1 << 40):
        tuning(planes=0, tile_min_rows=rows)
        z = ctx.DenseVector(z0)
        slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r), slab.SmootherConfig(sweeps=2))
        got[rows] = z.values()
    assert np.array_equal(got[0], got[1 << 40])
    want = oracle.rbgs_symmetric(oracle.build_hierarchy(*dims, 1), z0, r, sweeps=2)
    assert np.array_equal(got[0], want)


def test_vcycle_with_fused_transfers_bitwise(slab, ctx, oracle, tuning):
    """prolongation on the first forward pair, residual + restriction on the last backward pair (multigrid.hpp:87-116)"""
    dims = (32, 16, 24)
    tuning(planes=0, tile_min_rows=0)
    h = ctx.build_hierarchy(dims, 3)
    oh = oracle.build_hierarchy(*dims, 3)
    r, _ = oracle.random_vector(h.n(), 29)
    want = oracle.mg_vcycle(oh, np.zeros(h.n()), r)
    z = ctx.DenseVector(h.n(), 0.0)
    slab.mg_vcycle(h, z, ctx.DenseVector(r))
    assert np.array_equal(z.values(), want)


def test_solve_history_bitwise_through_tiles(slab, ctx, tuning):
    """16^3, 4 levels, exact dots: the 16^3 and 8^3 levels run the pair launches; golden history of the reference"""
    ctx.dot_mode = slab.DOT_EXACT
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "history_16.json")))
    tuning(planes=0, tile_min_rows=0)
    slab.set_tuning("cluster_rows", 0)
    try:
        h = ctx.build_hierarchy((16, 16, 16), 4)
        b = ctx.DenseVector(h.n())
        slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))
        res = slab.cg_solve(h, b, ctx.DenseVector(h.n(), 0.0), slab.CGConfig(max_iters=50, fixed_iterations=50))
    finally:
        slab.set_tuning("cluster_rows", 384)
    assert res.residual_history == gold["residual_history"]
