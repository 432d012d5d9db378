"""GPU parity of the primitive layer (operations.hpp) and the smoother / grid transfers against the
golden fixtures generated from the reference headers and against the CPU oracle. The cases
restate the reference's own tests (proj/tests/test_algebra.cpp, test_smoother.cpp,
test_multigrid.cpp, test_problem.cpp, test_coloring.cpp); all comparisons are bitwise.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def small():
    with open(os.path.join(GOLDEN, "small_cases.json")) as fh:
        return json.load(fh)


def unhex(values):
    return np.array([float.fromhex(v) for v in values], dtype=np.float64)


def tridiag(n, diag=2.0, off=-1.0):
    """oracles.hpp:233-245"""
    ro, co, va = [0], [], []
    for i in range(n):
        if i > 0:
            co.append(i - 1)
            va.append(off)
        co.append(i)
        va.append(diag)
        if i + 1 < n:
            co.append(i + 1)
            va.append(off)
        ro.append(len(co))
    return np.array(ro, dtype=np.uint64), np.array(co, dtype=np.uint64), np.array(va)


# ------------------------------------------------------------------ rng / containers


def test_lcg_known_answers(slab, ctx, small):
    """test_algebra.cpp:382-388 — first raw outputs, and random_vector front to back."""
    assert small["lcg_first_seed0"] == 1442695040888963407
    assert small["lcg_first_seed1"] == 7806831264735756412
    v, state = ctx.random_vector(8, 42)
    assert np.array_equal(v.values(), unhex(small["random_vector_seed42_n8_hex"]))
    assert state == small["random_vector_seed42_state"]


def test_stencil_generated_on_device_equals_reference_csr(slab, ctx, oracle):
    """problem.hpp:90-131: structure, values and column order, even and odd dimensions."""
    for dims in [(2, 2, 2), (4, 4, 4), (6, 4, 8), (5, 7, 9), (13, 13, 13), (33, 2, 3)]:
        A = ctx.build_matrix(dims)
        ro, co, va = A.csr()
        oro, oco, ova = oracle.build_matrix(*dims)
        assert A.nnz() == oracle.stencil_nnz(*dims) == (3 * dims[0] - 2) * (3 * dims[1] - 2) * (3 * dims[2] - 2)
        assert np.array_equal(ro, oro) and np.array_equal(co, oco) and np.array_equal(va, ova), dims


def test_csr_round_trip_and_validation(slab, ctx):
    ro, co, va = tridiag(70)
    A = slab.SparseMatrix.from_csr(ctx, 70, 70, ro, co, va)
    r2, c2, v2 = A.csr()
    assert np.array_equal(ro, r2) and np.array_equal(co, c2) and np.array_equal(va, v2)
    with pytest.raises(slab.InvalidArgument):  # columns must be strictly increasing
        slab.SparseMatrix.from_csr(ctx, 2, 2, [0, 2, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(slab.InvalidArgument):  # column out of range
        slab.SparseMatrix.from_csr(ctx, 2, 2, [0, 1, 1], [2], [1.0])
    with pytest.raises(slab.InvalidArgument):  # offsets not monotone
        slab.SparseMatrix.from_csr(ctx, 2, 2, [0, 1, 0], [0], [1.0])
    with pytest.raises(slab.InvalidArgument):  # duplicate coordinate
        slab.SparseMatrix.from_triplets(ctx, 2, 2, [(0, 0, 1.0), (0, 0, 2.0)])
    with pytest.raises(slab.InvalidArgument):
        slab.IndexMask(ctx, 4, [0, 2, 2])
    with pytest.raises(slab.InvalidArgument):
        slab.IndexMask(ctx, 4, [0, 4])


def test_restriction_structure(slab, ctx, small):
    """test_problem.cpp:143-173 — one 1.0 per row at (2cx,2cy,2cz); odd dims rejected."""
    R = ctx.build_restriction((4, 4, 4))
    ro, co, va = R.csr()
    assert R.nrows() == 8 and R.ncols() == 64 and R.nnz() == 8
    assert list(co) == small["restriction_cols_4x4x4"]
    assert np.array_equal(ro, np.arange(9, dtype=np.uint64)) and np.all(va == 1.0)
    with pytest.raises(slab.InvalidArgument):
        ctx.build_restriction((4, 5, 4))


# ------------------------------------------------------------------ operations.hpp


def test_spmv_matches_golden(slab, ctx, small):
    g = small["spmv_6x4x8"]
    A = ctx.build_matrix(g["dims"])
    x, _ = ctx.random_vector(A.ncols(), g["x_seed"])
    y = ctx.DenseVector(A.nrows())
    slab.mxv(y, A, x)
    assert A.nnz() == g["nnz"]
    assert np.array_equal(y.values(), unhex(g["y_hex"]))


def test_masked_mxv_leaves_unmasked_untouched(slab, ctx, small):
    """test_algebra.cpp:153-177"""
    g = small["masked_mxv_6x4x8"]
    dims = small["spmv_6x4x8"]["dims"]
    n = dims[0] * dims[1] * dims[2]
    A = ctx.build_matrix(dims)
    x, _ = ctx.random_vector(n, small["spmv_6x4x8"]["x_seed"])
    y, _ = ctx.random_vector(n, g["y0_seed"])
    before = y.values()
    members = np.arange(g["members_start"], n, g["members_step"], dtype=np.uint64)
    mask = slab.IndexMask(ctx, n, members)
    slab.mxv(y, mask, A, x, slab.descriptors.structural)
    got = y.values()
    assert np.array_equal(got, unhex(g["y_hex"]))
    untouched = np.setdiff1d(np.arange(n), members)
    assert np.array_equal(got[untouched], before[untouched])
    full = ctx.DenseVector(n)
    slab.mxv(full, A, x)
    assert np.array_equal(got[members.astype(np.int64)], full.values()[members.astype(np.int64)])


def test_transpose_descriptor_matches_oracle_scatter(slab, ctx, oracle):
    """test_algebra.cpp:179-214 — the reference scatters serially in row order; the device gathers
    over the explicit transpose in the same accumulation order, so results are bitwise equal."""
    rng = np.random.default_rng(5)
    nrows, ncols = 37, 53
    dense = (rng.random((nrows, ncols)) < 0.15) * rng.standard_normal((nrows, ncols))
    ro = np.zeros(nrows + 1, dtype=np.uint64)
    co, va = [], []
    for i in range(nrows):
        nz = np.nonzero(dense[i])[0]
        co.extend(nz)
        va.extend(dense[i, nz])
        ro[i + 1] = len(co)
    co, va = np.array(co, dtype=np.uint64), np.array(va)
    A = slab.SparseMatrix.from_csr(ctx, nrows, ncols, ro, co, va)
    xh = rng.standard_normal(nrows)
    x = ctx.DenseVector(xh)
    y = ctx.DenseVector(ncols, 7.0)
    slab.mxv(y, A, x, slab.descriptors.transpose_matrix)
    want = oracle.mxv((ro, co, va), xh, transpose=True, ncols=ncols)
    assert np.array_equal(y.values(), want)
    members = np.arange(0, ncols, 4, dtype=np.uint64)
    y2 = ctx.DenseVector(ncols, 7.0)
    slab.mxv(y2, slab.IndexMask(ctx, ncols, members), A, x, slab.descriptors.structural_transpose)
    want2 = oracle.mxv((ro, co, va), xh, transpose=True, ncols=ncols, mask=members, y=np.full(ncols, 7.0))
    assert np.array_equal(y2.values(), want2)


def test_mxv_rejects_shape_mismatch_and_aliasing(slab, ctx):
    """test_algebra.cpp:216-224"""
    A = ctx.build_matrix((2, 2, 2))
    x = ctx.DenseVector(8, 1.0)
    with pytest.raises(slab.DimensionMismatch):
        slab.mxv(ctx.DenseVector(7), A, x)
    with pytest.raises(slab.DimensionMismatch):
        slab.mxv(ctx.DenseVector(8), A, ctx.DenseVector(9))
    with pytest.raises(slab.DimensionMismatch):
        slab.mxv(ctx.DenseVector(8), slab.IndexMask(ctx, 7, [0]), A, x)
    with pytest.raises(slab.InvalidArgument):
        slab.mxv(x, A, x)


def test_dot_matches_golden_in_exact_mode(slab, ctx, small):
    """test_algebra.cpp:226-262 — chunked, order-fixed reduction: n below, at and above one chunk."""
    ctx.dot_mode = slab.DOT_EXACT
    x, _ = ctx.random_vector(20000, small["dot_n20000"]["x_seed"])
    y, _ = ctx.random_vector(20000, small["dot_n20000"]["y_seed"])
    assert slab.dot(x, y) == float.fromhex(small["dot_n20000"]["dot_hex"])
    assert slab.dot(y, x) == float.fromhex(small["dot_n20000"]["dot_hex"])
    assert slab.dot(x, x) == float.fromhex(small["dot_n20000"]["dot_xx_hex"])
    xh, yh = x.values(), y.values()
    for n in (4096, 4097, 100):
        assert slab.dot(ctx.DenseVector(xh[:n]), ctx.DenseVector(yh[:n])) == float.fromhex(small[f"dot_n{n}"]["dot_hex"])
    assert slab.dot(ctx.DenseVector(0), ctx.DenseVector(0)) == 0.0
    with pytest.raises(slab.DimensionMismatch):
        slab.dot(ctx.DenseVector(3), ctx.DenseVector(4))


def test_tree_dot_is_deterministic_and_close(slab, ctx, small):
    x, _ = ctx.random_vector(200000, 3)
    y, _ = ctx.random_vector(200000, 4)
    exact = slab.dot(x, y)
    ctx.dot_mode = slab.DOT_TREE
    try:
        first = slab.dot(x, y)
        assert all(slab.dot(x, y) == first for _ in range(5))
    finally:
        ctx.dot_mode = slab.DOT_EXACT
    assert abs(first - exact) <= 1e-12 * np.sqrt(slab.dot(x, x) * slab.dot(y, y))


def test_waxpby_matches_golden_and_aliases(slab, ctx, small):
    """test_algebra.cpp:264-294"""
    g = small["waxpby_n1000"]
    x, _ = ctx.random_vector(20000, 3)
    y, _ = ctx.random_vector(20000, 4)
    xs, ys = ctx.DenseVector(x.values()[:1000]), ctx.DenseVector(y.values()[:1000])
    w = ctx.DenseVector(1000)
    slab.waxpby(w, g["alpha"], xs, g["beta"], ys)
    want = unhex(g["w_hex"])
    assert np.array_equal(w.values(), want)
    xa = xs.copy()
    slab.waxpby(xa, g["alpha"], xa, g["beta"], ys)  # w aliases x
    assert np.array_equal(xa.values(), want)
    ya = ys.copy()
    slab.waxpby(ya, g["alpha"], xs, g["beta"], ya)  # w aliases y
    assert np.array_equal(ya.values(), want)
    with pytest.raises(slab.DimensionMismatch):
        slab.waxpby(w, 1.0, xs, 1.0, ctx.DenseVector(999))


def test_set_all(slab, ctx):
    v = ctx.DenseVector(1000, 3.0)
    assert np.all(v.values() == 3.0)
    slab.set_all(v, -0.5)
    assert np.all(v.values() == -0.5)
    assert slab.set_all(ctx.DenseVector(0), 1.0).size() == 0


# ------------------------------------------------------------------ coloring / levels


def test_hierarchy_shape_and_colors(slab, ctx, small):
    """test_problem.cpp:187-245, test_coloring.cpp:47-68"""
    h = ctx.build_hierarchy((16, 16, 16), 4)
    assert h.depth() == 4
    lvl, n = h, 16
    while lvl is not None:
        assert lvl.dims == (n, n, n) and lvl.n() == n ** 3 and lvl.num_colors == 8
        assert sum(lvl.color_nnz) == lvl.A.nnz() == (3 * n - 2) ** 3
        assert np.all(lvl.a_diag.values() == 26.0)
        if lvl.coarser is not None:
            assert lvl.restriction.nrows() == (n // 2) ** 3
        else:
            assert lvl.restriction is None
        lvl, n = lvl.coarser, n // 2
    lvl = ctx.build_hierarchy((4, 4, 4), 1)
    for k in range(8):  # colour == parity class, members ascending
        want = [ix + 4 * (iy + 4 * iz) for iz in range(4) for iy in range(4) for ix in range(4)
                if (ix % 2) + 2 * (iy % 2) + 4 * (iz % 2) == k]
        assert list(lvl.color_members(k)) == want
    odd = ctx.build_hierarchy((13, 13, 13), 1)
    assert [odd.color_info(k)[0] for k in range(8)] == small["color_sizes_13"] == [343, 294, 294, 252, 294, 252, 252, 216]


def test_hierarchy_rejection_rules(slab, ctx):
    """test_problem.cpp:223-236; and dimensions whose product wraps around 2^64 must not slip under the size limit"""
    for dims, levels in [((1, 4, 4), 1), ((4, 4, 4), 0), ((6, 4, 4), 3), ((4, 4, 4), 3), ((12, 12, 10), 3),
                         ((1 << 22, 1 << 22, 1 << 22), 1), ((1 << 32, 1 << 32, 2), 1), ((1 << 31, 2, 2), 1)]:
        with pytest.raises(slab.InvalidArgument):
            ctx.build_hierarchy(dims, levels)
    for dims in [(1 << 22, 1 << 22, 1 << 22), (1 << 40, 1 << 24, 4)]:
        with pytest.raises(slab.InvalidArgument):
            ctx.build_matrix(dims)


def test_general_level_coloring_matches_oracle_greedy(slab, ctx, oracle):
    """ProblemLevel(matrix) on non-stencil inputs: greedy colours, members and colour nnz must equal
    the oracle's (coloring.hpp:114-158), including a non-symmetric pattern."""
    rng = np.random.default_rng(11)
    n = 90
    dense = (rng.random((n, n)) < 0.06).astype(float) * -1.0
    np.fill_diagonal(dense, 8.0)
    ro = np.zeros(n + 1, dtype=np.uint64)
    co, va = [], []
    for i in range(n):
        nz = np.nonzero(dense[i])[0]
        co.extend(nz)
        va.extend(dense[i, nz])
        ro[i + 1] = len(co)
    co, va = np.array(co, dtype=np.uint64), np.array(va)
    lvl = slab.ProblemLevel(ctx, (ro, co, va))
    olvl = oracle.level_from_csr(ro, co, va)
    assert lvl.num_colors == olvl.num_colors
    for k in range(lvl.num_colors):
        assert np.array_equal(lvl.color_members(k), olvl.color_members(k))
        assert lvl.color_info(k)[1] == olvl.color_nnz(k)
    assert np.array_equal(lvl.a_diag.values(), olvl.diag())
    with pytest.raises(slab.InvalidArgument):  # missing diagonal
        slab.ProblemLevel(ctx, ([0, 1, 2], [1, 0], [1.0, 1.0]))


def _csr_of(dense):
    n = dense.shape[0]
    ro = np.zeros(n + 1, dtype=np.uint64)
    co, va = [], []
    for i in range(n):
        nz = np.nonzero(dense[i])[0]
        co.extend(nz)
        va.extend(dense[i, nz])
        ro[i + 1] = len(co)
    return ro, np.array(co, dtype=np.uint64), np.array(va, dtype=np.float64)


def _same_coloring(lvl, olvl):
    assert lvl.num_colors == olvl.num_colors
    for k in range(lvl.num_colors):
        assert np.array_equal(lvl.color_members(k), olvl.color_members(k))
        assert lvl.color_info(k)[1] == olvl.color_nnz(k)


def test_device_greedy_coloring_is_the_sequential_greedy(slab, ctx, oracle):
    """greedy_color as a device wavefront (coloring.cu) against the oracle's sequential loop (coloring.hpp:114-158):
    a tridiagonal chain (every row waits for the one before: as many rounds as rows, several ticketed blocks), the
    random symmetric matrices of tests/oracles.hpp:233-272, a strictly lower-triangular pattern (the neighbours come
    from A^T only), the 5x7x9 stencil handed in as a general matrix (eight parity classes), and a dense block whose
    rows need more than 256 colours (the search beyond the bit mask)."""
    n = 1500
    tri = np.zeros((n, n))
    idx = np.arange(n)
    tri[idx, idx] = 2.0
    tri[idx[1:], idx[:-1]] = -1.0
    tri[idx[:-1], idx[1:]] = -1.0
    ro, co, va = _csr_of(tri)
    lvl = slab.ProblemLevel(ctx, (ro, co, va))
    _same_coloring(lvl, oracle.level_from_csr(ro, co, va))
    assert lvl.num_colors == 2
    rng = np.random.default_rng(5)
    for n, density in ((40, 0.2), (300, 0.03), (700, 0.01)):
        m = (rng.random((n, n)) < density).astype(float)
        m = -(m + m.T > 0).astype(float)
        np.fill_diagonal(m, n)
        ro, co, va = _csr_of(m)
        _same_coloring(slab.ProblemLevel(ctx, (ro, co, va)), oracle.level_from_csr(ro, co, va))
    low = np.tril((rng.random((200, 200)) < 0.05).astype(float) * -1.0, -1)
    np.fill_diagonal(low, 4.0)
    ro, co, va = _csr_of(low)
    _same_coloring(slab.ProblemLevel(ctx, (ro, co, va)), oracle.level_from_csr(ro, co, va))
    ro, co, va = oracle.build_matrix(5, 7, 9)
    lvl = slab.ProblemLevel(ctx, (ro, co, va))
    olvl = oracle.level_from_csr(ro, co, va)
    _same_coloring(lvl, olvl)
    assert lvl.num_colors == 8
    for k in range(8):
        want = [ix + 5 * (iy + 7 * iz) for iz in range(9) for iy in range(7) for ix in range(5)
                if (ix % 2) + 2 * (iy % 2) + 4 * (iz % 2) == k]
        assert list(lvl.color_members(k)) == want
    n = 300
    full = -np.ones((n, n))
    np.fill_diagonal(full, float(n))
    ro, co, va = _csr_of(full)
    lvl = slab.ProblemLevel(ctx, (ro, co, va))
    _same_coloring(lvl, oracle.level_from_csr(ro, co, va))
    assert lvl.num_colors == n


# ------------------------------------------------------------------ smoother.hpp


def test_identity_solves_exactly(slab, ctx):
    """test_smoother.cpp:40-52"""
    ro = np.arange(6, dtype=np.uint64)
    lvl = slab.ProblemLevel(ctx, (ro, np.arange(5, dtype=np.uint64), np.ones(5)))
    assert lvl.num_colors == 1
    r, _ = ctx.random_vector(5, 1)
    z = ctx.DenseVector(5, 0.0)
    slab.rbgs_forward(lvl, z, r)
    assert z == r
    slab.set_all(z, 0.0)
    slab.rbgs_backward(lvl, z, r)
    assert z == r


def test_sweeps_match_oracle_on_tridiagonal(slab, ctx, oracle):
    """test_smoother.cpp:54-68, :86-98"""
    for n in (4, 9, 16):
        csr = tridiag(n)
        lvl = slab.ProblemLevel(ctx, csr)
        olvl = oracle.level_from_csr(*csr)
        buf, _ = oracle.random_vector(2 * n, 7 + n)
        r, z0 = buf[:n], buf[n:]
        z = ctx.DenseVector(z0)
        slab.rbgs_forward(lvl, z, ctx.DenseVector(r))
        assert np.array_equal(z.values(), oracle.rbgs_forward(olvl, z0, r))
        z = ctx.DenseVector(z0)
        slab.rbgs_backward(lvl, z, ctx.DenseVector(r))
        assert np.array_equal(z.values(), oracle.rbgs_backward(olvl, z0, r))


@pytest.mark.parametrize("dims", [(4, 4, 4), (5, 7, 9)])
def test_sweeps_match_reference_golden(slab, ctx, oracle, small, dims):
    """test_smoother.cpp:70-84 (4^3, seed 42) plus an odd grid; general-level path AND the
    device-generated stencil level must both reproduce the reference bitwise."""
    g = small["smoother_%dx%dx%d" % dims]
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(2 * n, g["seed"])
    r, z0 = buf[:n], buf[n:]
    general = slab.ProblemLevel(ctx, oracle.build_matrix(*dims))
    levels = [general]
    if all(d % 1 == 0 for d in dims):
        levels.append(ctx.build_hierarchy(dims, 1))
    for lvl in levels:
        assert lvl.num_colors == g["num_colors"] == 8
        assert [lvl.color_info(k)[0] for k in range(8)] == g["color_sizes"]
        assert lvl.color_nnz == g["color_nnz"]
        rv = ctx.DenseVector(r)
        z = ctx.DenseVector(z0)
        slab.rbgs_forward(lvl, z, rv)
        assert np.array_equal(z.values(), unhex(g["forward_hex"]))
        z = ctx.DenseVector(z0)
        slab.rbgs_backward(lvl, z, rv)
        assert np.array_equal(z.values(), unhex(g["backward_hex"]))
        z = ctx.DenseVector(z0)
        slab.rbgs_symmetric(lvl, z, rv, slab.SmootherConfig(2))
        assert np.array_equal(z.values(), unhex(g["symmetric2_hex"]))


def test_symmetric_is_forward_then_backward(slab, ctx):
    """test_smoother.cpp:134-155 incl. sweeps validation and the visit counter (:234-249)."""
    lvl = ctx.build_hierarchy((2, 2, 4), 1)
    r, _ = ctx.random_vector(lvl.n(), 17)
    composed = ctx.DenseVector(lvl.n(), 0.0)
    lvl.reset_stats()
    slab.rbgs_forward(lvl, composed, r)
    assert lvl.stats.nnz_visited == lvl.A.nnz()
    slab.rbgs_backward(lvl, composed, r)
    assert lvl.stats.nnz_visited == 2 * lvl.A.nnz()
    direct = ctx.DenseVector(lvl.n(), 0.0)
    slab.rbgs_symmetric(lvl, direct, r)
    assert direct == composed
    stepwise = ctx.DenseVector(lvl.n(), 0.0)
    for k in list(range(8)) + list(range(7, -1, -1)):
        slab.rbgs_color_step(lvl, k, stepwise, r)
    assert stepwise == composed
    with pytest.raises(slab.InvalidArgument):
        slab.rbgs_symmetric(lvl, direct, r, slab.SmootherConfig(0))
    with pytest.raises(slab.DimensionMismatch):
        slab.rbgs_forward(lvl, ctx.DenseVector(3), r)


# ------------------------------------------------------------------ multigrid.hpp


@pytest.mark.parametrize("key,dims,levels", [("vcycle_8x8x8_L2", (8, 8, 8), 2), ("vcycle_12x12x12_L3", (12, 12, 12), 3)])
def test_vcycle_matches_reference_golden(slab, ctx, small, key, dims, levels):
    """test_multigrid.cpp:49-71 — the cycle from zero against the reference's result, and the
    per-level visit counters."""
    g = small[key]
    h = ctx.build_hierarchy(dims, levels)
    r, _ = ctx.random_vector(h.n(), g["seed"])
    z = ctx.DenseVector(h.n(), 0.0)
    h.reset_stats()
    slab.mg_vcycle(h, z, r)
    assert np.array_equal(z.values(), unhex(g["z_hex"]))
    visited, lvl = [], h
    while lvl is not None:
        visited.append(lvl.stats.nnz_visited)
        lvl = lvl.coarser
    assert visited == g["nnz_visited"]


def test_vcycle_equals_scripted_composition(slab, ctx):
    """test_multigrid.cpp:49-71 scripted on the device primitives themselves."""
    direct = ctx.build_hierarchy((8, 8, 8), 2)
    scripted = ctx.build_hierarchy((8, 8, 8), 2)
    r, _ = ctx.random_vector(direct.n(), 7)
    z = ctx.DenseVector(direct.n(), 0.0)
    slab.mg_vcycle(direct, z, r)
    w = ctx.DenseVector(scripted.n(), 0.0)
    slab.rbgs_symmetric(scripted, w, r)
    f = ctx.DenseVector(scripted.n())
    slab.mxv(f, scripted.A, w)
    slab.waxpby(f, 1.0, r, -1.0, f)
    r_c = slab.restrict_vector(scripted, f)
    z_c = ctx.DenseVector(scripted.coarser.n(), 0.0)
    slab.rbgs_symmetric(scripted.coarser, z_c, r_c)
    slab.refine_and_add(scripted, w, z_c)
    slab.rbgs_symmetric(scripted, w, r)
    assert z == w


def test_transfer_operators(slab, ctx):
    """test_multigrid.cpp:73-143"""
    level = ctx.build_hierarchy((4, 4, 4), 2)
    assert slab.restrict_vector(level, ctx.DenseVector(64, 1.0)) == np.ones(8)
    z, _ = ctx.random_vector(64, 13)
    before = z.values()
    slab.refine_and_add(level, z, ctx.DenseVector(8, 0.0))
    assert z == before
    zeros = ctx.DenseVector(64, 0.0)
    slab.refine_and_add(level, zeros, ctx.DenseVector(8, 1.0))
    got = zeros.values().reshape(4, 4, 4)  # [iz, iy, ix]
    for iz in range(4):
        for iy in range(4):
            for ix in range(4):
                assert got[iz, iy, ix] == (1.0 if ix % 2 == 0 and iy % 2 == 0 and iz % 2 == 0 else 0.0)
    big = ctx.build_hierarchy((8, 8, 8), 2)
    z_c, _ = ctx.random_vector(64, 17)
    fine = ctx.DenseVector(512, 0.0)
    slab.refine_and_add(big, fine, z_c)
    assert slab.restrict_vector(big, fine) == z_c  # R R^T = I
    single = ctx.build_hierarchy((4, 4, 4), 1)
    with pytest.raises(slab.InvalidArgument):
        slab.restrict_vector(single, ctx.DenseVector(64), ctx.DenseVector(8))
    with pytest.raises(slab.InvalidArgument):
        slab.refine_and_add(single, ctx.DenseVector(64), ctx.DenseVector(8))
    with pytest.raises(slab.DimensionMismatch):
        slab.mg_vcycle(single, ctx.DenseVector(3), ctx.DenseVector(64))


def test_single_level_cycle_is_one_symmetric_smooth_and_zero_is_fixed(slab, ctx):
    """test_multigrid.cpp:28-47"""
    a = ctx.build_hierarchy((4, 4, 4), 1)
    r, _ = ctx.random_vector(64, 3)
    z1, z2 = ctx.DenseVector(64, 0.0), ctx.DenseVector(64, 0.0)
    slab.mg_vcycle(a, z1, r)
    slab.rbgs_symmetric(a, z2, r)
    assert z1 == z2
    h = ctx.build_hierarchy((4, 4, 4), 2)
    z = ctx.DenseVector(64, 0.0)
    slab.mg_vcycle(h, z, ctx.DenseVector(64, 0.0))
    assert z == np.zeros(64)


# ------------------------------------------------------------------ cg.hpp


def test_cg_small_cases(slab, ctx):
    """test_cg.cpp:40-52, :167-195 — identity in one iteration, breakdown, config validation."""
    ro = np.arange(7, dtype=np.uint64)
    ident = slab.ProblemLevel(ctx, (ro, np.arange(6, dtype=np.uint64), np.ones(6)))
    b, _ = ctx.random_vector(6, 1)
    res = slab.cg_solve(ident, b, ctx.DenseVector(6, 0.0), slab.CGConfig(use_preconditioner=False, rtol=1e-12))
    assert res.iterations == 1 and res.converged and res.solution == b and len(res.residual_history) == 2
    neg = slab.ProblemLevel(ctx, (ro, np.arange(6, dtype=np.uint64), -np.ones(6)))
    with pytest.raises(slab.SolverBreakdown):
        slab.cg_solve(neg, b, ctx.DenseVector(6, 0.0), slab.CGConfig(use_preconditioner=False))
    with pytest.raises(slab.SolverBreakdown):
        slab.cg_solve(neg, b, ctx.DenseVector(6, 0.0), slab.CGConfig(use_preconditioner=False, fixed_iterations=3))
    with pytest.raises(slab.InvalidArgument):
        slab.cg_solve(ident, b, ctx.DenseVector(6, 0.0), slab.CGConfig(rtol=0.0))
    with pytest.raises(slab.InvalidArgument):
        slab.cg_solve(ident, b, ctx.DenseVector(6, 0.0), slab.CGConfig(max_iters=0))
    with pytest.raises(slab.DimensionMismatch):
        slab.cg_solve(ident, ctx.DenseVector(5), ctx.DenseVector(6, 0.0))
    zero_rhs = slab.cg_solve(ident, ctx.DenseVector(6, 0.0), ctx.DenseVector(6, 0.0))
    assert zero_rhs.iterations == 0 and zero_rhs.residual_history == [0.0]


def test_residual_norm_and_recurrence_drift(slab, ctx):
    """test_cg.cpp:93-127 — ||b - A x|| through the primitives; recurrence vs recomputed residual."""
    h = ctx.build_hierarchy((8, 8, 8), 3)
    b = ctx.build_rhs((8, 8, 8))
    assert slab.residual_norm(h.A, ctx.DenseVector(512, 0.0), b) == pytest.approx(np.sqrt(512.0), rel=1e-15)
    res = slab.cg_solve(h, b, ctx.DenseVector(512, 0.0), slab.CGConfig(rtol=1e-10))
    assert res.converged
    true_res = slab.residual_norm(h.A, res.solution, b)
    assert abs(true_res - res.residual_history[-1]) <= 1e-10 * np.sqrt(512.0)
    again = slab.cg_solve(h, b, ctx.DenseVector(512, 0.0), slab.CGConfig(max_iters=10, fixed_iterations=10))
    again2 = slab.cg_solve(h, b, ctx.DenseVector(512, 0.0), slab.CGConfig(max_iters=10, fixed_iterations=10))
    assert again.residual_history == again2.residual_history and again.solution == again2.solution  # :155-165
