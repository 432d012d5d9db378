"""The one-launch sweep (csrc/sweep_cluster.cu, tuning key cluster_rows: one CTA, up to 512 rows per colour; levels
with larger colours keep their other kernels whatever the key says) must give the bits of the per-colour launches
and of the oracle: smoother.hpp:103-113, multigrid.hpp:87-116. The plane phases are switched off here so that the
even boxes reach this kernel too."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture()
def cluster_rows():
    from paper_2304_08232_b200 import _capi

    def apply(rows):
        _capi.set_tuning("cluster_rows", rows)

    _capi.set_tuning("planes", 0)
    yield apply
    apply(384)  # the library default
    _capi.set_tuning("planes", 1)


@pytest.mark.parametrize("dims", [(8, 8, 8), (16, 16, 16), (5, 7, 9), (26, 26, 26), (32, 32, 32), (3, 3, 3)])
def test_symmetric_sweep_bitwise(slab, ctx, oracle, cluster_rows, dims):
    """even, odd (unequal colour sizes), the largest eligible grid (16^3: 512 rows per colour) and two that are too large"""
    n = dims[0] * dims[1] * dims[2]
    buf, _ = oracle.random_vector(2 * n, 11)
    r, z0 = buf[:n], buf[n:]
    want = oracle.rbgs_symmetric(oracle.build_hierarchy(*dims, 1), z0, r)
    lvl = ctx.build_hierarchy(dims, 1)
    got = {}
    for rows in (0, 4096):
        cluster_rows(rows)
        z = ctx.DenseVector(z0)
        slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r))
        got[rows] = z.values()
    assert np.array_equal(got[0], want)
    assert np.array_equal(got[4096], want)


def test_solve_history_bitwise_with_cluster_sweeps(slab, ctx, cluster_rows):
    """16^3, 4 levels, exact dots: every level runs the cluster sweep (fused transfers on the first and last
    step included) and the history is the reference's golden one"""
    ctx.dot_mode = slab.DOT_EXACT
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "history_16.json")))
    h = ctx.build_hierarchy((16, 16, 16), 4)
    b = ctx.DenseVector(h.n())
    slab.mxv(b, h.A, ctx.DenseVector(h.n(), 1.0))
    x0 = ctx.DenseVector(h.n(), 0.0)
    cfg = slab.CGConfig(max_iters=50, fixed_iterations=50)
    cluster_rows(0)
    plain = slab.cg_solve(h, b, x0, cfg)
    cluster_rows(4096)
    got = slab.cg_solve(h, b, x0, cfg)
    assert plain.residual_history == gold["residual_history"]
    assert got.residual_history == gold["residual_history"]
    assert np.array_equal(got.solution.values(), plain.solution.values())


def test_general_matrix_level_with_cluster_sweep(slab, ctx, oracle, cluster_rows):
    """a non-stencil system (greedy colours from the matrix, coloring.hpp:114-158): tridiagonal, 2 colours"""
    n = 300
    ro = np.zeros(n + 1, dtype=np.uint64)
    co, va = [], []
    for i in range(n):
        for c, v in ((i - 1, -1.0), (i, 4.0 + 0.01 * (i % 7)), (i + 1, -1.5)):
            if 0 <= c < n:
                co.append(c)
                va.append(v)
        ro[i + 1] = len(co)
    csr = (ro, np.array(co, dtype=np.uint64), np.array(va, dtype=np.float64))
    lvl = slab.ProblemLevel(ctx, csr)
    assert lvl.format_info()["packed"] == 1
    buf, _ = oracle.random_vector(2 * n, 3)
    r, z0 = buf[:n], buf[n:]
    want = oracle.rbgs_symmetric(oracle.level_from_csr(*csr), z0, r)
    got = {}
    for rows in (0, 4096):
        cluster_rows(rows)
        z = ctx.DenseVector(z0)
        slab.rbgs_symmetric(lvl, z, ctx.DenseVector(r))
        got[rows] = z.values()
    assert np.array_equal(got[0], want)
    assert np.array_equal(got[4096], want)
