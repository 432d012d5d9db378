"""GPU tests of the 3D domain decomposition on ONE device: every rank of a process grid lives in this
process as its own context in manual-exchange mode (no communicator), and the test moves the halo
messages between the ranks itself, in lockstep — exactly the messages the NCCL path would send.
(The profiling guide forbids standing in for several GPUs with kernels that wait on one another;
lockstep emulation has no such waits.)

Oracle for every distributed result: the single-process run on the GLOBAL grid.
SpMV, the colour steps, the grid transfers and therefore the whole V-cycle must agree bitwise;
only the CG dots are combined across ranks and agree to rounding.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["default-kernels", "packed-kernels"])
def kernel_family(request, slab):
    """Every case runs twice: with the default launch-size thresholds (these small boxes then use the plain
    SELL kernels) and with the thresholds at zero, so that the dictionary-coded kernels run — ghost
    columns, escaped rows, boundary position lists and skip flags included."""
    packed = request.param == "packed-kernels"
    slab.set_tuning("packed_min_rows", 0 if packed else 65536)
    slab.set_tuning("packed_multi_min_rows", 0 if packed else 300000)
    yield request.param
    slab.set_tuning("packed_min_rows", 65536)
    slab.set_tuning("packed_multi_min_rows", 300000)


class World:
    def __init__(self, slab, grid, local_dims, levels):
        self.slab = slab
        self.grid = grid
        self.local = local_dims
        self.nranks = grid[0] * grid[1] * grid[2]
        self.ctxs, self.hier = [], []
        for rank in range(self.nranks):
            ctx = slab.Context(0)
            ctx.set_process_grid(grid, rank)
            self.ctxs.append(ctx)
            self.hier.append(ctx.build_hierarchy(local_dims, levels))
        self.global_dims = tuple(l * p for l, p in zip(local_dims, grid))

    def levels(self, depth):
        out = list(self.hier)
        for _ in range(depth):
            out = [h.coarser for h in out]
        return out

    def exchange(self, levels, vecs, color=-1):
        """deliver every rank's packed boundary values to the peers' ghost ranges"""
        messages = []
        for rank, (lvl, v) in enumerate(zip(levels, vecs)):
            for direction in range(27):
                send, _recv, peer = lvl.halo_info(direction, color)
                if peer >= 0 and send > 0:
                    messages.append((peer, 26 - direction, lvl.halo_pack(v, direction, color)))
        for peer, direction, payload in messages:
            levels[peer].halo_unpack(vecs[peer], direction, color, payload)

    def scatter(self, levels, global_values):
        """global natural-order array -> one vector per rank (ghost tails filled by an exchange)"""
        vecs = []
        gd = levels[0].decomp()["global"]
        g = np.asarray(global_values).reshape(gd[2], gd[1], gd[0])
        for ctx, lvl in zip(self.ctxs, levels):
            o = lvl.decomp()["offset"]
            l = lvl.dims
            block = g[o[2]:o[2] + l[2], o[1]:o[1] + l[1], o[0]:o[0] + l[0]]
            vecs.append(ctx.DenseVector(np.ascontiguousarray(block).ravel()))
        self.exchange(levels, vecs)
        return vecs

    def gather(self, levels, vecs):
        gd = levels[0].decomp()["global"]
        g = np.empty((gd[2], gd[1], gd[0]))
        for lvl, v in zip(levels, vecs):
            o = lvl.decomp()["offset"]
            l = lvl.dims
            g[o[2]:o[2] + l[2], o[1]:o[1] + l[1], o[0]:o[0] + l[0]] = v.values().reshape(l[2], l[1], l[0])
        return g.ravel()

    def zeros(self, levels):
        return [ctx.DenseVector(lvl.n(), 0.0) for ctx, lvl in zip(self.ctxs, levels)]

    # ---- lockstep drivers (mirror smoother.hpp / multigrid.hpp call by call)
    def color_step(self, levels, k, z, r):
        for lvl, zz, rr in zip(levels, z, r):
            self.slab.rbgs_color_step(lvl, k, zz, rr)
        self.exchange(levels, z, k)

    def symmetric(self, levels, z, r):
        for k in list(range(8)) + list(range(7, -1, -1)):
            self.color_step(levels, k, z, r)

    def vcycle(self, depth, z, r):
        slab = self.slab
        levels = self.levels(depth)
        self.symmetric(levels, z, r)
        if levels[0].coarser is None:
            return
        f = self.zeros(levels)
        for lvl, ff, zz in zip(levels, f, z):
            slab.mxv(ff, lvl.A, zz)          # ghosts of z are current after the last colour step
        for ff, rr in zip(f, r):
            slab.waxpby(ff, 1.0, rr, -1.0, ff)
        coarse = self.levels(depth + 1)
        r_c = [slab.restrict_vector(lvl, ff) for lvl, ff in zip(levels, f)]
        z_c = self.zeros(coarse)
        self.vcycle(depth + 1, z_c, r_c)
        for lvl, zz, zc in zip(levels, z, z_c):
            slab.refine_and_add(lvl, zz, zc)
        self.symmetric(levels, z, r)


GRIDS = [((2, 1, 1), (8, 8, 8), 3), ((2, 2, 1), (8, 8, 8), 2), ((2, 2, 2), (4, 4, 4), 2), ((2, 2, 2), (12, 12, 12), 3),
         ((1, 3, 2), (6, 4, 8), 2)]


@pytest.mark.parametrize("grid,local,levels", GRIDS)
def test_local_matrices_are_the_rows_of_the_global_matrix(slab, oracle, grid, local, levels):
    w = World(slab, grid, local, levels)
    depth = levels - 1  # check the coarsest level too (odd local dims / odd offsets for 12^3 x 3 levels)
    for d in (0, depth):
        lv = w.levels(d)
        gd = lv[0].decomp()["global"]
        gro, gco, gva = oracle.build_matrix(*gd)
        ldims = lv[0].dims
        for rank, lvl in enumerate(lv):
            o = lvl.decomp()["offset"]
            ro, co, va = lvl.A.csr()
            assert lvl.A.nnz() == int(ro[-1])
            for i in range(0, lvl.n(), max(1, lvl.n() // 150)):
                ix, iy, iz = i % ldims[0], (i // ldims[0]) % ldims[1], i // (ldims[0] * ldims[1])
                gi = (o[0] + ix) + gd[0] * ((o[1] + iy) + gd[1] * (o[2] + iz))
                gcols = gco[int(gro[gi]):int(gro[gi + 1])].astype(np.int64)
                want = [slab.plan_local_index(ldims, grid, rank, int(c % gd[0]), int((c // gd[0]) % gd[1]),
                                              int(c // (gd[0] * gd[1]))) for c in gcols]
                assert list(co[int(ro[i]):int(ro[i + 1])].astype(np.int64)) == want
                assert np.array_equal(va[int(ro[i]):int(ro[i + 1])], gva[int(gro[gi]):int(gro[gi + 1])])


@pytest.mark.parametrize("grid,local,levels", GRIDS)
def test_distributed_spmv_and_sweeps_equal_global_bitwise(slab, ctx, grid, local, levels):
    w = World(slab, grid, local, 1)
    lv = w.levels(0)
    n_global = int(np.prod(w.global_dims))
    single = ctx.build_hierarchy(w.global_dims, 1)
    xg, _ = ctx.random_vector(n_global, 21)
    rg, _ = ctx.random_vector(n_global, 22)
    yg = ctx.DenseVector(n_global)
    slab.mxv(yg, single.A, xg)
    x = w.scatter(lv, xg.values())
    y = w.zeros(lv)
    for lvl, yy, xx in zip(lv, y, x):
        slab.mxv(yy, lvl.A, xx)
    assert np.array_equal(w.gather(lv, y), yg.values())
    # colour sizes and per-colour nnz add up to the global ones
    for k in range(8):
        assert sum(l.color_info(k)[0] for l in lv) == single.color_info(k)[0]
        assert sum(l.color_info(k)[1] for l in lv) == single.color_info(k)[1]
    zg = xg.copy()
    slab.rbgs_symmetric(single, zg, rg)
    z = w.scatter(lv, xg.values())
    r = w.scatter(lv, rg.values())
    w.symmetric(lv, z, r)
    assert np.array_equal(w.gather(lv, z), zg.values())


@pytest.mark.parametrize("overlap", [1, 0])
@pytest.mark.parametrize("grid,local,levels", GRIDS[:4])
def test_distributed_vcycle_equals_global_bitwise(slab, ctx, grid, local, levels, overlap):
    """overlap=1: every colour step runs as boundary rows (position list) + interior rows (skip flags),
    the shape whose halo messages overlap the interior on real ranks; overlap=0: one launch per step."""
    slab.set_tuning("halo_overlap", overlap)
    try:
        _vcycle_case(slab, ctx, grid, local, levels)
    finally:
        slab.set_tuning("halo_overlap", 1)


def _vcycle_case(slab, ctx, grid, local, levels):
    w = World(slab, grid, local, levels)
    n_global = int(np.prod(w.global_dims))
    single = ctx.build_hierarchy(w.global_dims, levels)
    rg, _ = ctx.random_vector(n_global, 31)
    zg = ctx.DenseVector(n_global, 0.0)
    slab.mg_vcycle(single, zg, rg)
    lv = w.levels(0)
    r = w.scatter(lv, rg.values())
    z = w.zeros(lv)
    w.vcycle(0, z, r)
    assert np.array_equal(w.gather(lv, z), zg.values())


def test_distributed_cg_history_matches_global(slab, ctx):
    """Scripted PCG (cg.hpp:95-132) over a 2x2x2 grid; dots are sums of per-rank dots."""
    grid, local, levels = (2, 2, 2), (8, 8, 8), 3
    w = World(slab, grid, local, levels)
    lv = w.levels(0)
    n_global = int(np.prod(w.global_dims))
    single = ctx.build_hierarchy(w.global_dims, levels)
    ones = ctx.DenseVector(n_global, 1.0)
    bg = ctx.DenseVector(n_global)
    slab.mxv(bg, single.A, ones)
    iters = 8
    ref = slab.cg_solve(single, bg, ctx.DenseVector(n_global, 0.0), slab.CGConfig(max_iters=iters, fixed_iterations=iters))

    def gdot(a, b):
        return sum(slab.dot(x, y) for x, y in zip(a, b))

    b = w.scatter(lv, bg.values())
    x = w.zeros(lv)
    r = [v.copy() for v in b]          # r = b - A*0
    p = w.zeros(lv)
    q = w.zeros(lv)
    hist = [np.sqrt(gdot(r, r))]
    rho_prev = 0.0
    for it in range(1, iters + 1):
        z = w.zeros(lv)
        w.vcycle(0, z, r)
        rho = gdot(r, z)
        for pp, zz in zip(p, z):
            if it == 1:
                slab.waxpby(pp, 1.0, zz, 0.0, zz)
            else:
                slab.waxpby(pp, 1.0, zz, rho / rho_prev, pp)
        w.exchange(lv, p)
        for lvl, qq, pp in zip(lv, q, p):
            slab.mxv(qq, lvl.A, pp)
        alpha = rho / gdot(p, q)
        for xx, pp, rr, qq in zip(x, p, r, q):
            slab.waxpby(xx, 1.0, xx, alpha, pp)
            slab.waxpby(rr, 1.0, rr, -alpha, qq)
        rho_prev = rho
        hist.append(np.sqrt(gdot(r, r)))
    got, want = np.array(hist), np.array(ref.residual_history)
    assert np.max(np.abs(got - want) / want) <= 1e-10
    assert np.max(np.abs(w.gather(lv, x) - ref.solution.values())) <= 1e-12


def test_halo_plan_counts_and_errors(slab):
    w = World(slab, (2, 2, 2), (4, 4, 4), 1)
    lvl = w.levels(0)[0]  # rank 0 sits in the low corner: 3 faces, 3 edges, 1 corner
    info = w.ctxs[0].dist_info()
    assert info["grid"] == (2, 2, 2) and info["nranks"] == 8 and not info["has_comm"]
    peers = {d: lvl.halo_info(d)[2] for d in range(27)}
    assert sorted(p for p in peers.values() if p >= 0) == [1, 2, 3, 4, 5, 6, 7]
    assert lvl.halo_info(14)[:2] == (16, 16)   # +x face: 4x4 points each way
    assert lvl.halo_info(26)[:2] == (1, 1)     # +x+y+z corner
    assert lvl.decomp()["n_ghost"] == 3 * 16 + 3 * 4 + 1
    assert sum(lvl.halo_info(14, c)[0] for c in range(8)) == 16
    with pytest.raises(slab.InvalidArgument):
        lvl.halo_info(27)
    single = slab.Context(0).build_hierarchy((4, 4, 4), 1)
    with pytest.raises(slab.InvalidArgument):
        single.halo_info(14)


def test_single_rank_nccl_communicator_is_transparent(slab, ctx):
    """The NCCL plumbing itself on one GPU: a 1x1x1 process grid with a real communicator (unique id,
    ncclCommInitRank, allreduce of the dots captured in the iteration graph) must reproduce the plain
    single-process solve bit for bit."""
    n = 16
    plain = ctx.build_hierarchy((n, n, n), 4)
    ones = ctx.DenseVector(plain.n(), 1.0)
    b = ctx.DenseVector(plain.n())
    slab.mxv(b, plain.A, ones)
    cfg = slab.CGConfig(max_iters=12, fixed_iterations=12)
    want = slab.cg_solve(plain, b, ctx.DenseVector(plain.n(), 0.0), cfg)

    dctx = slab.Context(0)
    dctx.set_process_grid((1, 1, 1), 0)
    dctx.init_nccl(slab.nccl_unique_id())
    assert dctx.dist_info()["has_comm"]
    h = dctx.build_hierarchy((n, n, n), 4)
    db = dctx.DenseVector(b.values())
    got = slab.cg_solve(h, db, dctx.DenseVector(h.n(), 0.0), cfg)
    assert got.residual_history == want.residual_history
    assert np.array_equal(got.solution.values(), want.solution.values())
    assert slab.dot(db, db) == slab.dot(b, b)
    # On a communicator a fixed-iteration solve sends r'r together with the next iteration's r'z (one allreduce of two
    # doubles) and writes an iteration's history entry one iteration late: same numbers, in both dot modes, with and
    # without the iteration graph; a tolerance-driven solve keeps the immediate reductions.
    for mode in (slab.DOT_TREE, slab.DOT_EXACT):
        ctx.dot_mode = dctx.dot_mode = mode
        try:
            want_m = slab.cg_solve(plain, b, ctx.DenseVector(plain.n(), 0.0), cfg)
            got_m = slab.cg_solve(h, db, dctx.DenseVector(h.n(), 0.0), cfg)
            dctx.set_graphs(False)
            eager = slab.cg_solve(h, db, dctx.DenseVector(h.n(), 0.0), cfg)
            dctx.set_graphs(True)
            tol = slab.CGConfig(max_iters=40, rtol=1e-9)
            want_t = slab.cg_solve(plain, b, ctx.DenseVector(plain.n(), 0.0), tol)
            got_t = slab.cg_solve(h, db, dctx.DenseVector(h.n(), 0.0), tol)
        finally:
            ctx.dot_mode = dctx.dot_mode = slab.DOT_EXACT
        assert len(got_m.residual_history) == 13 and eager.residual_history == got_m.residual_history
        assert got_t.converged and got_t.iterations == want_t.iterations
        if mode == slab.DOT_EXACT:
            assert got_m.residual_history == want_m.residual_history
            assert np.array_equal(got_m.solution.values(), want_m.solution.values())
            assert got_t.residual_history == want_t.residual_history
        else:  # tree dots: the product's fused dot has another tree shape without the slab-staged kernel
            w = np.array(want_m.residual_history)
            assert np.max(np.abs(np.array(got_m.residual_history) - w) / w) <= 1e-10
            w = np.array(want_t.residual_history)
            assert np.max(np.abs(np.array(got_t.residual_history) - w) / w) <= 1e-10


def test_full_size_two_rank_vcycle_equals_global_bitwise(slab, ctx):
    """BASELINE.json configs[3] on its 2x1x1 process grid at the real size: two ranks of 104^3 (global 208x104x104,
    4 levels down to 13^3 per rank) in lockstep on one device. The fine-level launches are large enough for the
    dictionary-coded kernels by themselves; rows next to the cut carry ghost columns outside the dictionary and are
    read from the plain arrays; boundary rows run first from a position list, interior rows with skip flags."""
    rank0 = slab.Context(0)
    rank0.set_process_grid((2, 1, 1), 0)
    info = rank0.build_hierarchy((104, 104, 104), 1).format_info()
    # the x = 103 face looks across the cut: its rows (104 x 104, in four of the eight colours) cannot all be coded
    assert info["packed"] == 1 and 0 < info["escaped_rows"] <= 104 * 104
    _vcycle_case(slab, ctx, (2, 1, 1), (104, 104, 104), 4)


def test_full_size_eight_rank_vcycle_equals_global_bitwise(slab, ctx, kernel_family):
    """BASELINE.json configs[3] on its 2x2x2 process grid at the real size: eight ranks of 104^3 (global 208^3,
    4 levels, odd 13^3 boxes with odd offsets at the coarsest level) in lockstep on one device."""
    if kernel_family != "default-kernels":
        pytest.skip("one pass at this size is enough: the default thresholds already select the coded kernels")
    _vcycle_case(slab, ctx, (2, 2, 2), (104, 104, 104), 4)


@pytest.mark.parametrize("grid,local", [((2, 1, 1), (8, 8, 8)), ((2, 2, 2), (12, 12, 12)), ((1, 3, 2), (6, 4, 8)),
                                         ((2, 1, 1), (104, 104, 104))])
def test_sweep_turnaround_on_decomposed_levels(slab, ctx, grid, local):
    """What the library's own symmetric sweep does on a decomposed level: colours 0..6 forward, colour 7 twice in
    ONE launch with a single halo message after the second update, colours 6..0 backward. Must equal the global
    forward-then-backward sweep bit for bit (the rows of a colour never read that colour's ghost copies, so the
    intermediate values need not travel)."""
    w = World(slab, grid, local, 1)
    lv = w.levels(0)
    n_global = int(np.prod(w.global_dims))
    single = ctx.build_hierarchy(w.global_dims, 1)
    zg, _ = ctx.random_vector(n_global, 41)
    rg, _ = ctx.random_vector(n_global, 42)
    z = w.scatter(lv, zg.values())
    r = w.scatter(lv, rg.values())
    slab.rbgs_forward(single, zg, rg)
    slab.rbgs_backward(single, zg, rg)
    for k in range(7):
        w.color_step(lv, k, z, r)
    for lvl, zz, rr in zip(lv, z, r):
        slab.rbgs_color_step_twice(lvl, 7, zz, rr)
    w.exchange(lv, z, 7)
    for k in range(6, -1, -1):
        w.color_step(lv, k, z, r)
    assert np.array_equal(w.gather(lv, z), zg.values())
