"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads either ``oracle/libslab_oracle.so`` (the plain-C restatement, kind
"port") or ``oracle/_ref/libslab_ref.so`` (the reference's own headers behind
the same C interface, kind "reference").  Only tests/, ``__graft_entry__.smoke``
and the ``cpu_baseline`` / ``--impl reference`` legs of bench.py may import this
module; the product package ``paper_2304_08232_b200`` never does.

The method names follow the reference's free functions (operations.hpp,
smoother.hpp, multigrid.hpp, cg.hpp, problem.hpp).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "libslab_oracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libslab_ref.so")

OK, DIMENSION_MISMATCH, INVALID_ARGUMENT, SOLVER_BREAKDOWN = 0, 1, 2, 3


class OracleError(RuntimeError):
    pass


class DimensionMismatch(OracleError):
    pass


class InvalidArgument(OracleError):
    pass


class SolverBreakdown(OracleError):
    pass


_ERRORS = {DIMENSION_MISMATCH: DimensionMismatch, INVALID_ARGUMENT: InvalidArgument, SOLVER_BREAKDOWN: SolverBreakdown}

_u64 = C.c_uint64
_f64 = C.c_double
_pu64 = C.POINTER(C.c_uint64)
_pf64 = C.POINTER(C.c_double)


class _CgConfig(C.Structure):
    _fields_ = [
        ("max_iters", C.c_uint64),
        ("rtol", C.c_double),
        ("use_preconditioner", C.c_int),
        ("has_fixed_iterations", C.c_int),
        ("fixed_iterations", C.c_uint64),
        ("sweeps", C.c_uint64),
    ]


def build(ref: bool = True) -> None:
    """Compile the oracle libraries (make -C oracle)."""
    target = ["all"] if ref else ["libslab_oracle.so"]
    subprocess.run(["make", "-C", _HERE, *target], check=True, stdout=subprocess.DEVNULL)


def _f(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _u(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _pf(a: np.ndarray):
    return a.ctypes.data_as(_pf64)


def _pu(a: np.ndarray):
    return a.ctypes.data_as(_pu64)


@dataclass
class CGResult:
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False
    solution: np.ndarray | None = None


class Level:
    """One ProblemLevel (problem.hpp:220-277); ``coarser`` walks the chain."""

    def __init__(self, lib: "Oracle", handle, owner: bool):
        self._o = lib
        self._h = handle
        self._owner = owner
        self._coarser = None

    def __del__(self):
        if getattr(self, "_owner", False) and self._h:
            self._o._lib.so_level_destroy(self._h)
            self._h = None

    @property
    def n(self) -> int:
        return int(self._o._lib.so_level_n(self._h))

    @property
    def nnz(self) -> int:
        return int(self._o._lib.so_level_nnz(self._h))

    @property
    def dims(self):
        d = (C.c_uint64 * 3)()
        self._o._lib.so_level_dims(self._h, d)
        return tuple(int(v) for v in d)

    @property
    def num_colors(self) -> int:
        return int(self._o._lib.so_level_num_colors(self._h))

    def color_members(self, k: int) -> np.ndarray:
        size = int(self._o._lib.so_level_color_size(self._h, k))
        out = np.empty(size, dtype=np.uint64)
        self._o._lib.so_level_color_members(self._h, k, _pu(out))
        return out

    def color_nnz(self, k: int) -> int:
        return int(self._o._lib.so_level_color_nnz(self._h, k))

    def csr(self):
        ro = np.empty(self.n + 1, dtype=np.uint64)
        co = np.empty(self.nnz, dtype=np.uint64)
        va = np.empty(self.nnz, dtype=np.float64)
        self._o._lib.so_level_csr(self._h, _pu(ro), _pu(co), _pf(va))
        return ro, co, va

    def diag(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.float64)
        self._o._lib.so_level_diag(self._h, _pf(out))
        return out

    @property
    def coarser(self):
        if self._coarser is None:
            h = self._o._lib.so_level_coarser(self._h)
            if h:
                self._coarser = Level(self._o, h, owner=False)
                self._coarser._keepalive = self
        return self._coarser

    @property
    def nnz_visited(self) -> int:
        return int(self._o._lib.so_level_nnz_visited(self._h))

    def reset_stats(self) -> None:
        self._o._lib.so_level_reset_stats(self._h)

    def depth(self) -> int:
        return 1 + (self.coarser.depth() if self.coarser is not None else 0)


class Oracle:
    def __init__(self, kind: str = "port"):
        path = {"port": PORT_PATH, "reference": REF_PATH}[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} is not built (run make -C oracle)")
        lib = C.CDLL(path)
        self._lib = lib
        lib.so_kind.restype = C.c_char_p
        lib.so_get_threads.restype = C.c_int
        lib.so_set_threads.argtypes = [C.c_int]
        lib.so_stencil_nnz.restype = _u64
        lib.so_stencil_nnz.argtypes = [_u64] * 3
        lib.so_build_stencil.argtypes = [_u64, _u64, _u64, _pu64, _pu64, _pf64]
        lib.so_build_restriction_cols.argtypes = [_u64, _u64, _u64, _pu64]
        lib.so_lcg_fill.restype = _u64
        lib.so_lcg_fill.argtypes = [_u64, _pf64, _u64]
        lib.so_lcg_next.restype = _u64
        lib.so_lcg_next.argtypes = [_u64]
        lib.so_dot.restype = _f64
        lib.so_dot.argtypes = [_pf64, _pf64, _u64]
        lib.so_waxpby.restype = None
        lib.so_waxpby.argtypes = [_pf64, _f64, _pf64, _f64, _pf64, _u64]
        lib.so_mxv_csr.restype = None
        lib.so_mxv_csr.argtypes = [_pf64, _u64, _pu64, _pu64, _pf64, _pf64]
        lib.so_mxv_csr_masked.restype = None
        lib.so_mxv_csr_masked.argtypes = [_pf64, _pu64, _u64, _pu64, _pu64, _pf64, _pf64]
        lib.so_mxv_csr_transpose.restype = None
        lib.so_mxv_csr_transpose.argtypes = [_pf64, _u64, _u64, _pu64, _pu64, _pf64, _pf64]
        lib.so_mxv_csr_transpose_masked.restype = None
        lib.so_mxv_csr_transpose_masked.argtypes = [_pf64, _pu64, _u64, _u64, _u64, _pu64, _pu64, _pf64, _pf64]
        lib.so_hierarchy_create.argtypes = [_u64, _u64, _u64, _u64, C.POINTER(C.c_void_p)]
        lib.so_level_from_csr.argtypes = [_u64, _pu64, _pu64, _pf64, C.POINTER(C.c_void_p)]
        lib.so_level_destroy.restype = None
        lib.so_level_destroy.argtypes = [C.c_void_p]
        lib.so_level_coarser.restype = C.c_void_p
        lib.so_level_coarser.argtypes = [C.c_void_p]
        for name in ("so_level_n", "so_level_nnz", "so_level_num_colors", "so_level_nnz_visited"):
            getattr(lib, name).restype = _u64
            getattr(lib, name).argtypes = [C.c_void_p]
        lib.so_level_dims.restype = None
        lib.so_level_dims.argtypes = [C.c_void_p, C.POINTER(C.c_uint64 * 3)]
        lib.so_level_color_size.restype = _u64
        lib.so_level_color_size.argtypes = [C.c_void_p, _u64]
        lib.so_level_color_nnz.restype = _u64
        lib.so_level_color_nnz.argtypes = [C.c_void_p, _u64]
        lib.so_level_color_members.restype = None
        lib.so_level_color_members.argtypes = [C.c_void_p, _u64, _pu64]
        lib.so_level_csr.restype = None
        lib.so_level_csr.argtypes = [C.c_void_p, _pu64, _pu64, _pf64]
        lib.so_level_diag.restype = None
        lib.so_level_diag.argtypes = [C.c_void_p, _pf64]
        lib.so_level_reset_stats.restype = None
        lib.so_level_reset_stats.argtypes = [C.c_void_p]
        lib.so_level_mxv.argtypes = [C.c_void_p, _pf64, _pf64]
        lib.so_rbgs_color_step.argtypes = [C.c_void_p, _u64, _pf64, _pf64]
        lib.so_rbgs_forward.argtypes = [C.c_void_p, _pf64, _pf64]
        lib.so_rbgs_backward.argtypes = [C.c_void_p, _pf64, _pf64]
        lib.so_rbgs_symmetric.argtypes = [C.c_void_p, _pf64, _pf64, _u64]
        lib.so_restrict_vector.argtypes = [C.c_void_p, _pf64, _pf64]
        lib.so_refine_and_add.argtypes = [C.c_void_p, _pf64, _pf64]
        lib.so_mg_vcycle.argtypes = [C.c_void_p, _pf64, _pf64, _u64]
        lib.so_cg_solve.argtypes = [C.c_void_p, _pf64, _pf64, C.POINTER(_CgConfig), _pf64, _pf64, _pu64,
                                    C.POINTER(C.c_int)]
        lib.so_residual_norm.argtypes = [C.c_void_p, _pf64, _pf64, _pf64]

    # ------------------------------------------------------------------
    @property
    def kind(self) -> str:
        return self._lib.so_kind().decode()

    def set_threads(self, threads: int) -> None:
        self._lib.so_set_threads(int(threads))

    @property
    def threads(self) -> int:
        return int(self._lib.so_get_threads())

    @staticmethod
    def _check(rc: int, what: str) -> None:
        if rc != OK:
            raise _ERRORS.get(rc, OracleError)(f"{what}: status {rc}")

    # -- problem.hpp -----------------------------------------------------
    def stencil_nnz(self, nx, ny, nz) -> int:
        return int(self._lib.so_stencil_nnz(nx, ny, nz))

    def build_matrix(self, nx, ny, nz):
        if min(nx, ny, nz) < 2:
            raise InvalidArgument("grid dimensions must all be at least 2")
        n = nx * ny * nz
        nnz = self.stencil_nnz(nx, ny, nz)
        ro = np.empty(n + 1, dtype=np.uint64)
        co = np.empty(nnz, dtype=np.uint64)
        va = np.empty(nnz, dtype=np.float64)
        self._check(self._lib.so_build_stencil(nx, ny, nz, _pu(ro), _pu(co), _pf(va)), "build_matrix")
        return ro, co, va

    def build_restriction_cols(self, nx, ny, nz) -> np.ndarray:
        if min(nx, ny, nz) < 2 or nx % 2 or ny % 2 or nz % 2:
            raise InvalidArgument("build_restriction: dims must be even and >= 2")
        out = np.empty((nx // 2) * (ny // 2) * (nz // 2), dtype=np.uint64)
        self._check(self._lib.so_build_restriction_cols(nx, ny, nz, _pu(out)), "build_restriction")
        return out

    def build_hierarchy(self, nx, ny, nz, levels) -> Level:
        h = C.c_void_p()
        self._check(self._lib.so_hierarchy_create(nx, ny, nz, levels, C.byref(h)), "build_hierarchy")
        return Level(self, h, owner=True)

    def level_from_csr(self, ro, co, va) -> Level:
        ro, co, va = _u(ro), _u(co), _f(va)
        h = C.c_void_p()
        self._check(self._lib.so_level_from_csr(len(ro) - 1, _pu(ro), _pu(co), _pf(va), C.byref(h)), "ProblemLevel")
        return Level(self, h, owner=True)

    # -- rng.hpp ---------------------------------------------------------
    def random_vector(self, n: int, seed: int):
        """Returns (vector, state after n draws) — random_vector(n, Lcg64(seed))."""
        out = np.empty(n, dtype=np.float64)
        state = int(self._lib.so_lcg_fill(seed, _pf(out), n))
        return out, state

    def lcg_next(self, state: int) -> int:
        return int(self._lib.so_lcg_next(state))

    # -- operations.hpp --------------------------------------------------
    def dot(self, x, y) -> float:
        x, y = _f(x), _f(y)
        if x.size != y.size:
            raise DimensionMismatch("dot: vector lengths differ")
        return float(self._lib.so_dot(_pf(x), _pf(y), x.size))

    def waxpby(self, alpha, x, beta, y) -> np.ndarray:
        x, y = _f(x), _f(y)
        if x.size != y.size:
            raise DimensionMismatch("waxpby: vector lengths differ")
        w = np.empty_like(x)
        self._lib.so_waxpby(_pf(w), alpha, _pf(x), beta, _pf(y), x.size)
        return w

    def mxv(self, csr, x, transpose: bool = False, ncols: int | None = None, mask=None, y=None) -> np.ndarray:
        ro, co, va = _u(csr[0]), _u(csr[1]), _f(csr[2])
        nrows = ro.size - 1
        x = _f(x)
        if ncols is None:
            ncols = nrows
        out_len, in_len = (ncols, nrows) if transpose else (nrows, ncols)
        if x.size != in_len:
            raise DimensionMismatch("mxv: operand sizes do not match the matrix")
        if mask is None:
            out = np.empty(out_len, dtype=np.float64)
            if transpose:
                self._lib.so_mxv_csr_transpose(_pf(out), nrows, ncols, _pu(ro), _pu(co), _pf(va), _pf(x))
            else:
                self._lib.so_mxv_csr(_pf(out), nrows, _pu(ro), _pu(co), _pf(va), _pf(x))
            return out
        members = _u(mask)
        out = _f(y).copy()
        if out.size != out_len:
            raise DimensionMismatch("mxv: output length")
        if transpose:
            self._lib.so_mxv_csr_transpose_masked(_pf(out), _pu(members), members.size, nrows, ncols, _pu(ro), _pu(co),
                                                  _pf(va), _pf(x))
        else:
            self._lib.so_mxv_csr_masked(_pf(out), _pu(members), members.size, _pu(ro), _pu(co), _pf(va), _pf(x))
        return out

    def level_mxv(self, level: Level, x) -> np.ndarray:
        x = _f(x)
        y = np.empty(level.n, dtype=np.float64)
        self._check(self._lib.so_level_mxv(level._h, _pf(y), _pf(x)), "mxv")
        return y

    # -- smoother.hpp ------------------------------------------------------
    def _zr(self, level, z, r):
        z, r = _f(z).copy(), _f(r)
        if z.size != level.n or r.size != level.n:
            raise DimensionMismatch("smoother: vector lengths differ from the level size")
        return z, r

    def rbgs_color_step(self, level, k, z, r):
        z, r = self._zr(level, z, r)
        self._check(self._lib.so_rbgs_color_step(level._h, k, _pf(z), _pf(r)), "rbgs_color_step")
        return z

    def rbgs_forward(self, level, z, r):
        z, r = self._zr(level, z, r)
        self._check(self._lib.so_rbgs_forward(level._h, _pf(z), _pf(r)), "rbgs_forward")
        return z

    def rbgs_backward(self, level, z, r):
        z, r = self._zr(level, z, r)
        self._check(self._lib.so_rbgs_backward(level._h, _pf(z), _pf(r)), "rbgs_backward")
        return z

    def rbgs_symmetric(self, level, z, r, sweeps: int = 1):
        z, r = self._zr(level, z, r)
        self._check(self._lib.so_rbgs_symmetric(level._h, _pf(z), _pf(r), sweeps), "rbgs_symmetric")
        return z

    # -- multigrid.hpp -----------------------------------------------------
    def restrict_vector(self, level, v_fine):
        v = _f(v_fine)
        if level.coarser is None:
            raise InvalidArgument("restrict_vector: the coarsest level has no restriction operator")
        if v.size != level.n:
            raise DimensionMismatch("restrict_vector")
        out = np.empty(level.coarser.n, dtype=np.float64)
        self._check(self._lib.so_restrict_vector(level._h, _pf(v), _pf(out)), "restrict_vector")
        return out

    def refine_and_add(self, level, z, z_c):
        if level.coarser is None:
            raise InvalidArgument("refine_and_add: the coarsest level has no restriction operator")
        z, z_c = _f(z).copy(), _f(z_c)
        if z.size != level.n or z_c.size != level.coarser.n:
            raise DimensionMismatch("refine_and_add")
        self._check(self._lib.so_refine_and_add(level._h, _pf(z), _pf(z_c)), "refine_and_add")
        return z

    def mg_vcycle(self, level, z, r, sweeps: int = 1):
        z, r = _f(z).copy(), _f(r)
        if z.size != level.n or r.size != level.n:
            raise DimensionMismatch("mg_vcycle: vector lengths differ from the level size")
        self._check(self._lib.so_mg_vcycle(level._h, _pf(z), _pf(r), sweeps), "mg_vcycle")
        return z

    # -- cg.hpp ------------------------------------------------------------
    def cg_solve(self, hierarchy, b, x0, max_iters=500, rtol=1e-6, use_preconditioner=True, fixed_iterations=None,
                 sweeps=1) -> CGResult:
        b, x0 = _f(b), _f(x0)
        if b.size != hierarchy.n or x0.size != hierarchy.n:
            raise DimensionMismatch("cg_solve: vector lengths differ from the system size")
        cfg = _CgConfig(max_iters, rtol, int(use_preconditioner), int(fixed_iterations is not None),
                        int(fixed_iterations or 0), sweeps)
        x = np.empty_like(b)
        hist = np.zeros(max(int(max_iters), 1) + 1, dtype=np.float64)
        iters = C.c_uint64(0)
        conv = C.c_int(0)
        rc = self._lib.so_cg_solve(hierarchy._h, _pf(b), _pf(x0), C.byref(cfg), _pf(x), _pf(hist), C.byref(iters),
                                   C.byref(conv))
        self._check(rc, "cg_solve")
        k = int(iters.value)
        return CGResult(k, [float(v) for v in hist[: k + 1]], bool(conv.value), x)

    def residual_norm(self, level, x, b) -> float:
        out = C.c_double(0.0)
        x, b = _f(x), _f(b)
        self._check(self._lib.so_residual_norm(level._h, _pf(x), _pf(b), C.byref(out)), "residual_norm")
        return float(out.value)


def available_kinds():
    kinds = []
    if os.path.exists(PORT_PATH):
        kinds.append("port")
    if os.path.exists(REF_PATH):
        kinds.append("reference")
    return kinds
