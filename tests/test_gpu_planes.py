"""The plane phases of csrc/plane.cu (a symmetric sweep as three out-of-place launches: even planes colours 0-3, odd
planes colours 4-7 and 7-4, even planes colours 3-0; zero-padded slabs staged through shared memory by bulk-async
copies, no matrix stream) must give the bits of the colour-by-colour steps and of the oracle:
smoother.hpp:60-113, multigrid.hpp:87-116, operations.hpp:116-125."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DEFAULTS = {"planes": 1, "plane_min_rows": 0, "plane_ty": 0, "plane_cz": 0, "plane_ns": 0, "plane_rows": 0}


@pytest.fixture()
def tuning():
    from paper_2304_08232_b200 import _capi

    def apply(**kw):
        for key, value in kw.items():
            _capi.set_tuning(key, value)

    yield apply
    apply(**DEFAULTS)


SHAPES = [(4, 4, 4), (8, 8, 8), (16, 12, 10), (6, 10, 14), (8, 5, 7), (12, 7, 9), (32, 8, 20), (64, 6, 6), (40, 24, 16),
          (10, 33, 5), (96, 20, 6)]


@pytest.mark.parametrize("dims", SHAPES)
def test_sweeps_bitwise(slab, ctx, oracle, tuning, dims):
    """forward, backward and symmetric sweeps through the plane phases: even and odd y/z extents (a last plane
    without a partner, a last tile that is cut short), boxes thinner than a tile, short and long x-lines"""
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(2 * n, 17)
    r, z0 = buf[:n], buf[n:]
    olvl = oracle.build_hierarchy(*dims, 1)
    lvl = ctx.build_hierarchy(dims, 1)
    assert lvl.format_info()["plane_phases"] == 1
    for name in ("rbgs_forward", "rbgs_backward", "rbgs_symmetric"):
        want = getattr(oracle, name)(olvl, z0, r)
        z = ctx.DenseVector(z0)
        getattr(slab, name)(lvl, z, ctx.DenseVector(r))
        assert np.array_equal(z.values(), want), (name, dims)


@pytest.mark.parametrize("shape", [dict(plane_ty=2, plane_cz=1, plane_ns=3), dict(plane_ty=2, plane_cz=3, plane_ns=5),
                                   dict(plane_ty=4, plane_cz=2, plane_ns=4), dict(plane_ty=8, plane_cz=16, plane_ns=6),
                                   dict(plane_ty=16, plane_cz=4, plane_ns=3), dict(plane_ty=32, plane_cz=6, plane_ns=8),
                                   dict(plane_ty=4, plane_cz=12, plane_ns=7), dict(plane_rows=1), dict(plane_rows=2),
                                   dict(plane_ty=8, plane_cz=2, plane_rows=2), dict(plane_ty=2, plane_cz=5, plane_rows=2),
                                   dict(plane_ty=16, plane_cz=3, plane_ns=4, plane_rows=2), dict(plane_ty=32, plane_cz=1, plane_rows=1)])
def test_plane_shapes_bitwise(slab, ctx, oracle, tuning, shape):
    """every ring depth / tile height / march length gives the same bits (slot reuse, recomputed edge lines, partial
    tiles and chunks, planes outside the box entering a re-used slot)"""
    for dims in ((24, 22, 26), (12, 21, 13)):
        n = dims[0] * dims[1] * dims[2]
        buf, _ = oracle.random_vector(2 * n, 5)
        r, z0 = buf[:n], buf[n:]
        olvl = oracle.build_hierarchy(*dims, 1)
        tuning(**shape)
        lvl = ctx.build_hierarchy(dims, 1)
        for name in ("rbgs_forward", "rbgs_backward", "rbgs_symmetric"):
            want = getattr(oracle, name)(olvl, z0, r)
            z = ctx.DenseVector(z0)
            getattr(slab, name)(lvl, z, ctx.DenseVector(r))
            assert np.array_equal(z.values(), want), (shape, dims, name)


def test_planes_equal_per_colour_launches_two_sweeps(slab, ctx, oracle, tuning):
    dims = (48, 20, 12)
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(2 * n, 23)
    r, z0 = buf[:n], buf[n:]
    lvl = ctx.build_hierarchy(dims, 1)
    got = {}
    for on in (1, 0):
        tuning(planes=on)
        z = ctx.DenseVector(z0)
        slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r), slab.SmootherConfig(sweeps=2))
        got[on] = z.values()
    assert np.array_equal(got[0], got[1])
    want = oracle.rbgs_symmetric(oracle.build_hierarchy(*dims, 1), z0, r, sweeps=2)
    assert np.array_equal(got[1], want)


def test_signed_zeros_and_non_finite_inputs_match_per_colour_launches(slab, ctx, tuning):
    """the zero padding stands in for absent neighbours: +-0 products must not change any bit, whatever the vector
    holds (negative zeros, huge values, infinities and NaNs inside the box behave as in the row-by-row kernels)"""
    dims = (8, 6, 10)
    n = dims[0] * dims[1] * dims[2]
    rng = np.random.default_rng(3)
    z0 = rng.standard_normal(n)
    z0[rng.integers(0, n, 40)] = -0.0
    z0[rng.integers(0, n, 40)] = 0.0
    z0[rng.integers(0, n, 6)] = 1e300
    z0[7] = np.inf
    z0[n - 3] = np.nan
    r = rng.standard_normal(n)
    r[rng.integers(0, n, 30)] = -0.0
    lvl = ctx.build_hierarchy(dims, 1)
    got = {}
    for on in (1, 0):
        tuning(planes=on)
        z = ctx.DenseVector(z0)
        slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r))
        got[on] = z.values()
    assert np.array_equal(got[0].view(np.uint64), got[1].view(np.uint64))


@pytest.mark.parametrize("dims,levels", [((32, 16, 24), 3), ((16, 16, 16), 2), ((48, 40, 24), 3)])
def test_vcycle_with_fused_transfers_bitwise(slab, ctx, oracle, tuning, dims, levels):
    """prolongation on the first sub-phase of phase A, residual + restriction on the last sub-phase of phase C
    (multigrid.hpp:87-116)"""
    h = ctx.build_hierarchy(dims, levels)
    oh = oracle.build_hierarchy(*dims, levels)
    r, _ = oracle.random_vector(h.n(), 29)
    want = oracle.mg_vcycle(oh, np.zeros(h.n()), r)
    z = ctx.DenseVector(h.n(), 0.0)
    slab.mg_vcycle(h, z, ctx.DenseVector(r))
    assert np.array_equal(z.values(), want)
    ctx.fused_transfers = 0
    try:
        z2 = ctx.DenseVector(h.n(), 0.0)
        slab.mg_vcycle(h, z2, ctx.DenseVector(r))
    finally:
        ctx.fused_transfers = 1
    assert np.array_equal(z2.values(), want)


def test_solve_history_bitwise_through_planes(slab, ctx, tuning):
    """16^3, 4 levels, exact dots: every level but the 2^3 one runs the plane phases; golden history of the reference"""
    ctx.dot_mode = slab.DOT_EXACT
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "history_16.json")))
    h = ctx.build_hierarchy((16, 16, 16), 4)
    b = ctx.DenseVector(h.n())
    slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))
    res = slab.cg_solve(h, b, ctx.DenseVector(h.n(), 0.0), slab.CGConfig(max_iters=50, fixed_iterations=50))
    assert res.residual_history == gold["residual_history"]


def test_fused_rz_dot_and_zero_guess_keep_the_history(slab, ctx, tuning):
    """tree-dot mode: r'z on the last two plane phases of the V-cycle (cg.hpp:116 fused; another tree shape, so 1e-12
    against the separate dot), and the V-cycle's zero initial guess taken as a flag of the first phase (bit-identical:
    exact-dot mode reproduces the reference's golden history through it)"""
    from paper_2304_08232_b200 import _capi

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "history_64.json")))
    want = np.array(gold["residual_history"])
    h = ctx.build_hierarchy((64, 64, 64), 4)
    b = ctx.DenseVector(h.n())
    slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))
    cfg = slab.CGConfig(max_iters=50, fixed_iterations=50)
    ctx.dot_mode = slab.DOT_EXACT
    res = slab.cg_solve(h, b, ctx.DenseVector(h.n(), 0.0), cfg)
    assert res.residual_history == gold["residual_history"]
    got = {}
    try:
        ctx.dot_mode = slab.DOT_TREE
        for mode in (2, 0):
            _capi.set_tuning("fuse_rz", mode)
            got[mode] = np.array(slab.cg_solve(h, b, ctx.DenseVector(h.n(), 0.0), cfg).residual_history)
    finally:
        _capi.set_tuning("fuse_rz", 1)
        ctx.dot_mode = slab.DOT_EXACT
    assert np.max(np.abs(got[2] - got[0]) / got[0]) <= 1e-12
    assert np.max(np.abs(got[2] - want) / want) <= 1e-10


def test_zero_numerators_take_the_fast_path_with_the_right_sign(slab, ctx, oracle, tuning):
    """(+-0) / d without the division's slow path (plane.cu, divide): right-hand sides and guesses that are zero or
    negative zero over most of the box — the benchmark's b = A 1 is zero away from the faces — give the bits of the
    per-colour kernels and of the oracle, signs of the zeros included"""
    dims = (12, 10, 8)
    n = dims[0] * dims[1] * dims[2]
    rng = np.random.default_rng(11)
    lvl = ctx.build_hierarchy(dims, 1)
    olvl = oracle.build_hierarchy(*dims, 1)
    cases = []
    for zfill, rfill in ((0.0, 0.0), (-0.0, -0.0), (0.0, -0.0), (-0.0, 0.0)):
        z0 = np.full(n, zfill)
        r = np.full(n, rfill)
        cases.append((z0.copy(), r.copy()))
        hot = rng.integers(0, n, 5)
        z0[hot] = rng.standard_normal(5)
        r[rng.integers(0, n, 5)] = rng.standard_normal(5)
        cases.append((z0, r))
    for z0, r in cases:
        got = {}
        for on in (1, 0):
            tuning(planes=on)
            z = ctx.DenseVector(z0)
            slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r))
            got[on] = z.values()
        want = oracle.rbgs_symmetric(olvl, z0, r)
        assert np.array_equal(got[1].view(np.uint64), got[0].view(np.uint64))
        assert np.array_equal(got[1].view(np.uint64), np.asarray(want).view(np.uint64))


def test_tile_shape_cache_file_round_trip(slab, ctx, oracle, tuning, tmp_path, monkeypatch):
    """SLAB_PLANE_TUNE_CACHE: the shapes a level measured are appended to the file and re-used by the next level of the
    same box (a profiler's run then executes the measured shapes); results do not depend on it"""
    path = tmp_path / "shapes.txt"
    monkeypatch.setenv("SLAB_PLANE_TUNE_CACHE", str(path))
    dims = (32, 24, 16)
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(2 * n, 5)
    r, z0 = buf[:n], buf[n:]
    want = oracle.rbgs_symmetric(oracle.build_hierarchy(*dims, 1), z0, r)
    lines = None
    for _ in range(2):
        lvl = ctx.build_hierarchy(dims, 1)
        z = ctx.DenseVector(z0)
        slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r))
        assert np.array_equal(z.values(), want)
        text = path.read_text().splitlines() if path.exists() else []
        if lines is None:
            lines = text
            assert 1 <= len(lines) <= 3 and all(len(l.split()) == 7 and l.startswith("32 24 16 ") for l in lines)
        else:
            assert text == lines  # the second build read its shapes, measured nothing, wrote nothing
