"""ctypes binding of include/slab_b200.h plus a host-side mirror of the reference's operator API.

The reference ("slab") is a header-only C++ library; its natural host language is C++ and the
C++ facade lives in include/slab_b200.hpp. This module is the same mirror for Python callers
(tests/, bench.py): same free-function names, argument order and error taxonomy as
/root/reference/proj/include/slab/*.hpp, every call going through the C ABI into the CUDA
library. There is no CPU path here: if libslab_b200.so is missing or no sm_100 GPU is visible,
loading / context creation raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslab_b200.so")

# ---------------------------------------------------------------- errors (error.hpp:25-42)


class Error(RuntimeError):
    """slab::Error"""


class DimensionMismatch(Error):
    """slab::DimensionMismatch"""


class InvalidArgument(Error):
    """slab::InvalidArgument"""


class SolverBreakdown(Error):
    """slab::SolverBreakdown"""


class CudaError(Error):
    """CUDA / NCCL runtime failure, or no usable GPU (there is no CPU fallback)."""


_STATUS = {1: DimensionMismatch, 2: InvalidArgument, 3: SolverBreakdown, 4: CudaError}

DESC_NONE, DESC_STRUCTURAL, DESC_TRANSPOSE = 0, 1, 2
DOT_EXACT, DOT_TREE = 0, 1


@dataclass(frozen=True)
class Descriptor:  # descriptor.hpp:26-31
    structural: bool = False
    transpose_matrix: bool = False

    @property
    def flags(self) -> int:
        return (DESC_STRUCTURAL if self.structural else 0) | (DESC_TRANSPOSE if self.transpose_matrix else 0)


class descriptors:  # descriptor.hpp:33-38
    none = Descriptor()
    structural = Descriptor(True, False)
    transpose_matrix = Descriptor(False, True)
    structural_transpose = Descriptor(True, True)


class _CgConfig(C.Structure):
    _fields_ = [
        ("max_iters", C.c_uint64),
        ("rtol", C.c_double),
        ("use_preconditioner", C.c_int),
        ("has_fixed_iterations", C.c_int),
        ("fixed_iterations", C.c_uint64),
        ("sweeps", C.c_uint64),
    ]


class _CgResult(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("converged", C.c_int), ("solve_ms", C.c_double)]


class FormatInfo(C.Structure):  # slab_format_info
    _fields_ = [("packed", C.c_int32), ("width_class", C.c_int32), ("dict_size", C.c_int32), ("stride", C.c_int32),
                ("escaped_rows", C.c_int64), ("plain_bytes", C.c_uint64), ("packed_bytes", C.c_uint64),
                ("mask_bytes", C.c_uint64), ("plane_phases", C.c_int32), ("reserved", C.c_int32)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class _LevelStats(C.Structure):
    _fields_ = [("smoother_ns", C.c_uint64), ("transfer_ns", C.c_uint64), ("mg_ns", C.c_uint64),
                ("nnz_visited", C.c_uint64)]


_u64 = C.c_uint64
_vp = C.c_void_p
_pu64 = C.POINTER(C.c_uint64)
_pf64 = C.POINTER(C.c_double)
_pvp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); the full export list of include/slab_b200.h
SIGNATURES = {
    "slab_abi_version": (C.c_int, []),
    "slab_last_error": (C.c_char_p, []),
    "slab_status_name": (C.c_char_p, [C.c_int]),
    "slab_launch_count": (_u64, []),
    "slab_set_programmatic_launch": (C.c_int, [C.c_int]),
    "slab_set_tuning": (C.c_int, [C.c_char_p, C.c_int64]),
    "slab_ctx_create": (C.c_int, [C.c_int, _pvp]),
    "slab_ctx_destroy": (C.c_int, [_vp]),
    "slab_ctx_sync": (C.c_int, [_vp]),
    "slab_ctx_set_dot_mode": (C.c_int, [_vp, C.c_int]),
    "slab_ctx_get_dot_mode": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "slab_ctx_set_graphs": (C.c_int, [_vp, C.c_int]),
    "slab_ctx_set_fused_transfers": (C.c_int, [_vp, C.c_int]),
    "slab_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "slab_ctx_timer_start": (C.c_int, [_vp]),
    "slab_ctx_timer_stop": (C.c_int, [_vp, _pf64]),
    "slab_ctx_device_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), _pu64]),
    "slab_vec_create": (C.c_int, [_vp, _u64, C.c_double, _pvp]),
    "slab_vec_destroy": (C.c_int, [_vp]),
    "slab_vec_size": (C.c_int, [_vp, _pu64]),
    "slab_vec_upload": (C.c_int, [_vp, _vp, _u64]),
    "slab_vec_download": (C.c_int, [_vp, _vp, _u64]),
    "slab_vec_copy": (C.c_int, [_vp, _vp]),
    "slab_vec_fill_lcg": (C.c_int, [_vp, _u64, _pu64]),
    "slab_set_all": (C.c_int, [_vp, C.c_double]),
    "slab_dot": (C.c_int, [_vp, _vp, _pf64]),
    "slab_waxpby": (C.c_int, [_vp, C.c_double, _vp, C.c_double, _vp]),
    "slab_mat_create_csr": (C.c_int, [_vp, _u64, _u64, _vp, _vp, _vp, _pvp]),
    "slab_mat_create_stencil27": (C.c_int, [_vp, _u64, _u64, _u64, _pvp]),
    "slab_mat_create_restriction": (C.c_int, [_vp, _u64, _u64, _u64, _pvp]),
    "slab_mat_destroy": (C.c_int, [_vp]),
    "slab_mat_shape": (C.c_int, [_vp, _pu64, _pu64, _pu64]),
    "slab_mat_download_csr": (C.c_int, [_vp, _vp, _vp, _vp]),
    "slab_mat_device_bytes": (C.c_int, [_vp, _pu64]),
    "slab_mat_format_info": (C.c_int, [_vp, _vp]),
    "slab_level_format_info": (C.c_int, [_vp, _vp]),
    "slab_mask_create": (C.c_int, [_vp, _u64, _vp, _u64, _pvp]),
    "slab_mask_destroy": (C.c_int, [_vp]),
    "slab_mask_info": (C.c_int, [_vp, _pu64, _pu64]),
    "slab_mxv": (C.c_int, [_vp, _vp, _vp, C.c_uint]),
    "slab_mxv_masked": (C.c_int, [_vp, _vp, _vp, _vp, C.c_uint]),
    "slab_hierarchy_create": (C.c_int, [_vp, _u64, _u64, _u64, _u64, _pvp]),
    "slab_level_create_csr": (C.c_int, [_vp, _u64, _vp, _vp, _vp, _pvp]),
    "slab_level_destroy": (C.c_int, [_vp]),
    "slab_level_coarser": (C.c_int, [_vp, _pvp]),
    "slab_level_matrix": (C.c_int, [_vp, _pvp]),
    "slab_level_restriction": (C.c_int, [_vp, _pvp]),
    "slab_level_diag": (C.c_int, [_vp, _pvp]),
    "slab_level_info": (C.c_int, [_vp, C.POINTER(C.c_uint64 * 3), _pu64, _pu64, _pu64, _pu64]),
    "slab_level_color_info": (C.c_int, [_vp, _u64, _pu64, _pu64]),
    "slab_level_color_members": (C.c_int, [_vp, _u64, _vp]),
    "slab_level_stats_get": (C.c_int, [_vp, C.POINTER(_LevelStats)]),
    "slab_level_stats_reset": (C.c_int, [_vp]),
    "slab_rbgs_color_step": (C.c_int, [_vp, _u64, _vp, _vp]),
    "slab_rbgs_color_step_twice": (C.c_int, [_vp, _u64, _vp, _vp]),
    "slab_rbgs_forward": (C.c_int, [_vp, _vp, _vp]),
    "slab_rbgs_backward": (C.c_int, [_vp, _vp, _vp]),
    "slab_rbgs_symmetric": (C.c_int, [_vp, _vp, _vp, _u64]),
    "slab_restrict_vector": (C.c_int, [_vp, _vp, _vp]),
    "slab_refine_and_add": (C.c_int, [_vp, _vp, _vp]),
    "slab_mg_vcycle": (C.c_int, [_vp, _vp, _vp, _u64]),
    "slab_cg_config_default": (None, [C.POINTER(_CgConfig)]),
    "slab_cg_solve": (C.c_int, [_vp, _vp, _vp, C.POINTER(_CgConfig), _vp, _vp, C.POINTER(_CgResult)]),
    "slab_cg_solve_host": (C.c_int, [_vp, _vp, _vp, _u64, C.POINTER(_CgConfig), _vp, _vp, C.POINTER(_CgResult)]),
    "slab_residual_norm": (C.c_int, [_vp, _vp, _vp, _pf64]),
    "slab_ctx_set_process_grid": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int]),
    "slab_nccl_unique_id": (C.c_int, [_vp]),
    "slab_ctx_init_nccl": (C.c_int, [_vp, _vp]),
    "slab_ctx_dist_info": (C.c_int, [_vp, C.POINTER(C.c_int * 3), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), _pu64]),
    "slab_level_decomp": (C.c_int, [_vp, C.POINTER(C.c_uint64 * 3), C.POINTER(C.c_uint64 * 3), _pu64]),
    "slab_level_halo_info": (C.c_int, [_vp, C.c_int, C.c_int, _pu64, _pu64, C.POINTER(C.c_int)]),
    "slab_level_halo_pack": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "slab_level_halo_unpack": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp]),
    "slab_plan_query": (C.c_int, [C.POINTER(C.c_uint64 * 3), C.POINTER(C.c_uint64 * 3), _u64, C.c_int, C.c_int, _pu64,
                                  _pu64, _pu64, _pu64, C.POINTER(C.c_int64), _pu64, _vp]),
    "slab_plan_local_index": (C.c_int, [C.POINTER(C.c_uint64 * 3), C.POINTER(C.c_uint64 * 3), _u64, _u64, _u64, _u64,
                                        C.POINTER(C.c_int64)]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """dlopen the CUDA library and type every export. Raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_2304_08232_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (restype, argtypes) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.slab_last_error().decode(errors="replace")
        raise _STATUS.get(rc, Error)(msg)


def set_programmatic_launch(enabled: bool) -> None:
    _check(load_library().slab_set_programmatic_launch(int(enabled)))


def set_tuning(key: str, value: int) -> None:
    """Performance knobs that never change results (see slab_set_tuning in include/slab_b200.h)."""
    _check(load_library().slab_set_tuning(key.encode(), int(value)))


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(load_library().slab_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def plan_query(local_dims, grid, rank: int, direction: int, color: int) -> dict:
    """Host-only halo plan of one rank for (direction, colour); needs no GPU."""
    lib = load_library()
    ld = (C.c_uint64 * 3)(*[int(v) for v in local_dims])
    pg = (C.c_uint64 * 3)(*[int(v) for v in grid])
    nl, ng, sc, rc, gb = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    peer = C.c_int64()
    _check(lib.slab_plan_query(C.byref(ld), C.byref(pg), rank, direction, color, C.byref(nl), C.byref(ng), C.byref(sc),
                               C.byref(rc), C.byref(peer), C.byref(gb), None))
    idx = np.empty(sc.value, dtype=np.uint64)
    _check(lib.slab_plan_query(C.byref(ld), C.byref(pg), rank, direction, color, None, None, None, None, None, None,
                               _ptr(idx)))
    return {"n_local": nl.value, "n_ghost": ng.value, "send_count": sc.value, "recv_count": rc.value,
            "peer": peer.value, "ghost_base": gb.value, "send_indices": idx}


def plan_local_index(local_dims, grid, rank: int, X: int, Y: int, Z: int) -> int:
    ld = (C.c_uint64 * 3)(*[int(v) for v in local_dims])
    pg = (C.c_uint64 * 3)(*[int(v) for v in grid])
    out = C.c_int64()
    _check(load_library().slab_plan_local_index(C.byref(ld), C.byref(pg), rank, X, Y, Z, C.byref(out)))
    return out.value


def launch_count() -> int:
    return int(load_library().slab_launch_count())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _u64a(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- context


class Context:
    """One device + one stream. All containers are created from a context."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = C.c_void_p()
        _check(lib.slab_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.slab_ctx_destroy(self._h)
            self._h = None

    # no __del__: containers keep raw pointers into the context, and at interpreter shutdown the
    # destruction order is arbitrary. A context is a stream plus a few KB; close() is explicit.

    def sync(self) -> None:
        _check(_lib.slab_ctx_sync(self._h))

    @property
    def dot_mode(self) -> int:
        m = C.c_int()
        _check(_lib.slab_ctx_get_dot_mode(self._h, C.byref(m)))
        return m.value

    @dot_mode.setter
    def dot_mode(self, mode: int) -> None:
        _check(_lib.slab_ctx_set_dot_mode(self._h, mode))

    def set_graphs(self, enabled: bool) -> None:
        _check(_lib.slab_ctx_set_graphs(self._h, int(enabled)))

    def set_fused_transfers(self, enabled: bool) -> None:
        _check(_lib.slab_ctx_set_fused_transfers(self._h, int(enabled)))

    def set_profiling(self, enabled: bool) -> None:
        """LevelStats times (smoother_ns, transfer_ns, mg_ns) are only filled while this is on."""
        _check(_lib.slab_ctx_set_profiling(self._h, int(enabled)))

    def timer_start(self) -> None:
        _check(_lib.slab_ctx_timer_start(self._h))

    def timer_stop(self) -> float:
        ms = C.c_double()
        _check(_lib.slab_ctx_timer_stop(self._h, C.byref(ms)))
        return ms.value

    def device_info(self) -> dict:
        sm, ma, mi, mem = C.c_int(), C.c_int(), C.c_int(), C.c_uint64()
        _check(_lib.slab_ctx_device_info(self._h, C.byref(sm), C.byref(ma), C.byref(mi), C.byref(mem)))
        return {"sm_count": sm.value, "cc": (ma.value, mi.value), "hbm_bytes": mem.value}

    # ---- 3D domain decomposition (one process per GPU)
    def set_process_grid(self, grid, rank: int) -> None:
        _check(_lib.slab_ctx_set_process_grid(self._h, int(grid[0]), int(grid[1]), int(grid[2]), int(rank)))

    def init_nccl(self, unique_id: bytes) -> None:
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        _check(_lib.slab_ctx_init_nccl(self._h, C.cast(buf, C.c_void_p)))

    def dist_info(self) -> dict:
        grid = (C.c_int * 3)()
        rank, nranks, comm, ex = C.c_int(), C.c_int(), C.c_int(), C.c_uint64()
        _check(_lib.slab_ctx_dist_info(self._h, C.byref(grid), C.byref(rank), C.byref(nranks), C.byref(comm),
                                       C.byref(ex)))
        return {"grid": tuple(grid), "rank": rank.value, "nranks": nranks.value, "has_comm": bool(comm.value),
                "exchanges": ex.value}

    # factories in the reference's vocabulary
    def DenseVector(self, length_or_values, value: float = 0.0) -> "DenseVector":
        return DenseVector(self, length_or_values, value)

    def build_matrix(self, dims) -> "SparseMatrix":  # problem.hpp:90-131
        h = C.c_void_p()
        _check(_lib.slab_mat_create_stencil27(self._h, *[int(d) for d in dims], C.byref(h)))
        return SparseMatrix(self, h)

    def build_restriction(self, dims) -> "SparseMatrix":  # problem.hpp:174-201
        h = C.c_void_p()
        _check(_lib.slab_mat_create_restriction(self._h, *[int(d) for d in dims], C.byref(h)))
        return SparseMatrix(self, h)

    def build_rhs(self, dims) -> "DenseVector":  # problem.hpp:134-137
        if min(dims) < 2:
            raise InvalidArgument("grid dimensions must all be at least 2")
        return DenseVector(self, int(np.prod([int(d) for d in dims])), 1.0)

    def build_hierarchy(self, dims, levels: int) -> "ProblemLevel":  # problem.hpp:284-319
        h = C.c_void_p()
        _check(_lib.slab_hierarchy_create(self._h, *[int(d) for d in dims], int(levels), C.byref(h)))
        return ProblemLevel(self, h, owner=True)

    def random_vector(self, n: int, seed: int):  # rng.hpp:59-65; returns (vector, lcg state after n draws)
        v = DenseVector(self, n)
        state = C.c_uint64()
        _check(_lib.slab_vec_fill_lcg(v._h, seed, C.byref(state)))
        return v, state.value


# ---------------------------------------------------------------- containers


class DenseVector:  # dense_vector.hpp:33-66
    def __init__(self, ctx: Context, length_or_values, value: float = 0.0):
        self.ctx = ctx
        h = C.c_void_p()
        if isinstance(length_or_values, (int, np.integer)):
            _check(_lib.slab_vec_create(ctx._h, int(length_or_values), float(value), C.byref(h)))
            self._h = h
        else:
            host = _f64(length_or_values)
            _check(_lib.slab_vec_create(ctx._h, host.size, 0.0, C.byref(h)))
            self._h = h
            _check(_lib.slab_vec_upload(self._h, _ptr(host), host.size))

    @classmethod
    def _borrow(cls, ctx: Context, handle, keepalive) -> "DenseVector":
        self = cls.__new__(cls)
        self.ctx = ctx
        self._h = handle
        self._borrowed = keepalive
        return self

    def __del__(self):
        if getattr(self, "_h", None) and not hasattr(self, "_borrowed"):
            _lib.slab_vec_destroy(self._h)
            self._h = None

    def size(self) -> int:
        n = C.c_uint64()
        _check(_lib.slab_vec_size(self._h, C.byref(n)))
        return n.value

    def __len__(self) -> int:
        return self.size()

    def values(self) -> np.ndarray:  # download, natural order
        out = np.empty(self.size(), dtype=np.float64)
        _check(_lib.slab_vec_download(self._h, _ptr(out), out.size))
        return out

    def assign(self, values) -> "DenseVector":
        host = _f64(values)
        _check(_lib.slab_vec_upload(self._h, _ptr(host), host.size))
        return self

    def copy(self) -> "DenseVector":
        out = DenseVector(self.ctx, self.size())
        _check(_lib.slab_vec_copy(out._h, self._h))
        return out

    def __eq__(self, other) -> bool:  # value equality like std::vector<double>::operator==
        if isinstance(other, DenseVector):
            other = other.values()
        other = np.asarray(other, dtype=np.float64)
        mine = self.values()
        return mine.shape == other.shape and bool(np.all(mine == other))

    __hash__ = None


class SparseMatrix:  # sparse_matrix.hpp:48-171
    def __init__(self, ctx: Context, handle, keepalive=None):
        self.ctx = ctx
        self._h = handle
        if keepalive is not None:
            self._borrowed = keepalive

    @classmethod
    def from_csr(cls, ctx: Context, nrows: int, ncols: int, row_offsets, col_indices, values) -> "SparseMatrix":
        ro, co, va = _u64a(row_offsets), _u64a(col_indices), _f64(values)
        if ro.size != nrows + 1 or (ro.size and ro[0] != 0):
            raise InvalidArgument("from_csr: row_offsets must have nrows+1 entries starting at 0")
        if int(ro[-1]) != co.size or co.size != va.size:
            raise InvalidArgument("from_csr: offsets, column and value arrays disagree on nnz")
        h = C.c_void_p()
        _check(_lib.slab_mat_create_csr(ctx._h, nrows, ncols, _ptr(ro), _ptr(co), _ptr(va), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_triplets(cls, ctx: Context, nrows: int, ncols: int, triplets) -> "SparseMatrix":
        """sparse_matrix.hpp:59-93 (sorting and duplicate rejection are host-side container logic)."""
        t = list(triplets)
        for (r, c, _v) in t:
            if r >= nrows or c >= ncols or r < 0 or c < 0:
                raise InvalidArgument(f"from_triplets: coordinate ({r}, {c}) out of range")
        t.sort(key=lambda e: (e[0], e[1]))
        for k in range(1, len(t)):
            if t[k][0] == t[k - 1][0] and t[k][1] == t[k - 1][1]:
                raise InvalidArgument(f"from_triplets: duplicate coordinate ({t[k][0]}, {t[k][1]})")
        ro = np.zeros(nrows + 1, dtype=np.uint64)
        for (r, _c, _v) in t:
            ro[r + 1] += 1
        ro = np.cumsum(ro, dtype=np.uint64)
        co = np.array([e[1] for e in t], dtype=np.uint64)
        va = np.array([e[2] for e in t], dtype=np.float64)
        return cls.from_csr(ctx, nrows, ncols, ro, co, va)

    def __del__(self):
        if getattr(self, "_h", None) and not hasattr(self, "_borrowed"):
            _lib.slab_mat_destroy(self._h)
            self._h = None

    def _shape(self):
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_lib.slab_mat_shape(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def nrows(self) -> int:
        return self._shape()[0]

    def ncols(self) -> int:
        return self._shape()[1]

    def nnz(self) -> int:
        return self._shape()[2]

    def csr(self):
        """(row_offsets, col_indices, values) converted back from the opaque device format."""
        nrows, _ncols, nnz = self._shape()
        ro = np.empty(nrows + 1, dtype=np.uint64)
        co = np.empty(max(nnz, 1), dtype=np.uint64)
        va = np.empty(max(nnz, 1), dtype=np.float64)
        _check(_lib.slab_mat_download_csr(self._h, _ptr(ro), _ptr(co), _ptr(va)))
        return ro, co[:nnz], va[:nnz]

    def device_bytes(self) -> int:
        b = C.c_uint64()
        _check(_lib.slab_mat_device_bytes(self._h, C.byref(b)))
        return b.value

    def format_info(self) -> dict:
        info = FormatInfo()
        _check(_lib.slab_mat_format_info(self._h, C.byref(info)))
        return info.as_dict()


class IndexMask:  # index_mask.hpp:35-73
    def __init__(self, ctx: Context, universe_size: int, members: Sequence[int]):
        self.ctx = ctx
        m = _u64a(members)
        h = C.c_void_p()
        _check(_lib.slab_mask_create(ctx._h, int(universe_size), _ptr(m), m.size, C.byref(h)))
        self._h = h
        self._members = m.copy()
        self._universe = int(universe_size)

    @classmethod
    def full(cls, ctx: Context, n: int) -> "IndexMask":
        return cls(ctx, n, np.arange(n, dtype=np.uint64))

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.slab_mask_destroy(self._h)
            self._h = None

    def universe_size(self) -> int:
        return self._universe

    def members(self) -> np.ndarray:
        return self._members

    def size(self) -> int:
        return int(self._members.size)

    def empty(self) -> bool:
        return self._members.size == 0


@dataclass
class LevelStats:  # problem.hpp:204-209
    smoother_ns: int = 0
    transfer_ns: int = 0
    mg_ns: int = 0
    nnz_visited: int = 0


class ProblemLevel:  # problem.hpp:220-277
    def __init__(self, ctx: Context, handle_or_matrix, owner: bool = True, keepalive=None):
        """ProblemLevel(ctx, (row_offsets, col_indices, values)) builds a standalone level around an
        arbitrary square CSR system (problem.hpp:253); hierarchies come from build_hierarchy."""
        self.ctx = ctx
        self._keepalive = keepalive
        if isinstance(handle_or_matrix, C.c_void_p):
            self._h = handle_or_matrix
            self._owner = owner
        else:
            ro, co, va = handle_or_matrix
            ro, co, va = _u64a(ro), _u64a(co), _f64(va)
            h = C.c_void_p()
            _check(_lib.slab_level_create_csr(ctx._h, ro.size - 1, _ptr(ro), _ptr(co), _ptr(va), C.byref(h)))
            self._h = h
            self._owner = True
        self._coarser = None

    def __del__(self):
        if getattr(self, "_owner", False) and getattr(self, "_h", None):
            _lib.slab_level_destroy(self._h)
            self._h = None

    def _info(self):
        dims = (C.c_uint64 * 3)()
        n, nnz, nc, depth = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(_lib.slab_level_info(self._h, C.byref(dims), C.byref(n), C.byref(nnz), C.byref(nc), C.byref(depth)))
        return tuple(int(d) for d in dims), n.value, nnz.value, nc.value, depth.value

    @property
    def dims(self):
        return self._info()[0]

    def n(self) -> int:
        return self._info()[1]

    @property
    def num_colors(self) -> int:
        return self._info()[3]

    def depth(self) -> int:
        return self._info()[4]

    def has_coarser(self) -> bool:
        return self.coarser is not None

    @property
    def coarser(self) -> Optional["ProblemLevel"]:
        if self._coarser is None:
            h = C.c_void_p()
            _check(_lib.slab_level_coarser(self._h, C.byref(h)))
            if h.value:
                self._coarser = ProblemLevel(self.ctx, h, owner=False, keepalive=self)
        return self._coarser

    @property
    def A(self) -> SparseMatrix:
        h = C.c_void_p()
        _check(_lib.slab_level_matrix(self._h, C.byref(h)))
        return SparseMatrix(self.ctx, h, keepalive=self)

    @property
    def restriction(self) -> Optional[SparseMatrix]:
        h = C.c_void_p()
        _check(_lib.slab_level_restriction(self._h, C.byref(h)))
        return SparseMatrix(self.ctx, h, keepalive=self) if h.value else None

    @property
    def a_diag(self) -> DenseVector:
        h = C.c_void_p()
        _check(_lib.slab_level_diag(self._h, C.byref(h)))
        return DenseVector._borrow(self.ctx, h, self)

    def color_members(self, k: int) -> np.ndarray:  # colors.masks[k].members()
        size, _nnz = self.color_info(k)
        out = np.empty(size, dtype=np.uint64)
        _check(_lib.slab_level_color_members(self._h, k, _ptr(out)))
        return out

    def color_info(self, k: int):
        size, cnnz = C.c_uint64(), C.c_uint64()
        _check(_lib.slab_level_color_info(self._h, k, C.byref(size), C.byref(cnnz)))
        return size.value, cnnz.value

    @property
    def color_nnz(self):
        return [self.color_info(k)[1] for k in range(self.num_colors)]

    @property
    def stats(self) -> LevelStats:
        s = _LevelStats()
        _check(_lib.slab_level_stats_get(self._h, C.byref(s)))
        return LevelStats(s.smoother_ns, s.transfer_ns, s.mg_ns, s.nnz_visited)

    def reset_stats(self) -> None:
        _check(_lib.slab_level_stats_reset(self._h))

    def format_info(self) -> dict:
        """format of the colour-major matrix copy the smoother reads"""
        info = FormatInfo()
        _check(_lib.slab_level_format_info(self._h, C.byref(info)))
        return info.as_dict()

    # ---- domain decomposition: manual halo access (tests, custom transports)
    def decomp(self) -> dict:
        g, o = (C.c_uint64 * 3)(), (C.c_uint64 * 3)()
        ng = C.c_uint64()
        _check(_lib.slab_level_decomp(self._h, C.byref(g), C.byref(o), C.byref(ng)))
        return {"global": tuple(int(v) for v in g), "offset": tuple(int(v) for v in o), "n_ghost": ng.value}

    def halo_info(self, direction: int, color: int = -1):
        s, r, p = C.c_uint64(), C.c_uint64(), C.c_int()
        _check(_lib.slab_level_halo_info(self._h, direction, color, C.byref(s), C.byref(r), C.byref(p)))
        return s.value, r.value, p.value

    def halo_pack(self, v: DenseVector, direction: int, color: int = -1) -> np.ndarray:
        count = self.halo_info(direction, color)[0]
        out = np.empty(count, dtype=np.float64)
        _check(_lib.slab_level_halo_pack(self._h, v._h, direction, color, _ptr(out)))
        return out

    def halo_unpack(self, v: DenseVector, direction: int, color: int, values: np.ndarray) -> None:
        values = _f64(values)
        if values.size != self.halo_info(direction, color)[1]:
            raise DimensionMismatch("halo_unpack: message length differs from the ghost range")
        _check(_lib.slab_level_halo_unpack(self._h, v._h, direction, color, _ptr(values)))


# ---------------------------------------------------------------- operations.hpp


def set_all(v: DenseVector, value: float) -> DenseVector:
    _check(_lib.slab_set_all(v._h, float(value)))
    return v


def dot(x: DenseVector, y: DenseVector) -> float:
    out = C.c_double()
    _check(_lib.slab_dot(x._h, y._h, C.byref(out)))
    return out.value


def waxpby(w: DenseVector, alpha: float, x: DenseVector, beta: float, y: DenseVector) -> DenseVector:
    _check(_lib.slab_waxpby(w._h, float(alpha), x._h, float(beta), y._h))
    return w


def mxv(y: DenseVector, *args) -> DenseVector:
    """mxv(y, A, x[, desc]) or mxv(y, mask, A, x[, desc]) — operations.hpp:213-230."""
    if isinstance(args[0], IndexMask):
        mask, A, x = args[0], args[1], args[2]
        desc = args[3] if len(args) > 3 else descriptors.none
        _check(_lib.slab_mxv_masked(y._h, mask._h, A._h, x._h, desc.flags))
    else:
        A, x = args[0], args[1]
        desc = args[2] if len(args) > 2 else descriptors.none
        _check(_lib.slab_mxv(y._h, A._h, x._h, desc.flags))
    return y


# ---------------------------------------------------------------- smoother.hpp / multigrid.hpp


@dataclass
class SmootherConfig:  # smoother.hpp:48-50
    sweeps: int = 1


def rbgs_color_step(level: ProblemLevel, k: int, z: DenseVector, r: DenseVector) -> DenseVector:
    _check(_lib.slab_rbgs_color_step(level._h, int(k), z._h, r._h))
    return z


def rbgs_color_step_twice(level: ProblemLevel, k: int, z: DenseVector, r: DenseVector) -> DenseVector:
    """the turnaround of a symmetric sweep: colour k updated twice in a row by one launch"""
    _check(_lib.slab_rbgs_color_step_twice(level._h, int(k), z._h, r._h))
    return z


def rbgs_forward(level: ProblemLevel, z: DenseVector, r: DenseVector) -> DenseVector:
    _check(_lib.slab_rbgs_forward(level._h, z._h, r._h))
    return z


def rbgs_backward(level: ProblemLevel, z: DenseVector, r: DenseVector) -> DenseVector:
    _check(_lib.slab_rbgs_backward(level._h, z._h, r._h))
    return z


def rbgs_symmetric(level: ProblemLevel, z: DenseVector, r: DenseVector, cfg: SmootherConfig = SmootherConfig()):
    if cfg.sweeps < 1:
        raise InvalidArgument("SmootherConfig: sweeps must be at least 1")
    _check(_lib.slab_rbgs_symmetric(level._h, z._h, r._h, int(cfg.sweeps)))
    return z


def restrict_vector(level: ProblemLevel, v_fine: DenseVector, out: Optional[DenseVector] = None) -> DenseVector:
    if out is None:  # allocating variant, multigrid.hpp:57-65
        R = level.restriction
        if R is None:
            raise InvalidArgument("restrict_vector: the coarsest level has no restriction operator")
        out = DenseVector(level.ctx, R.nrows())
    _check(_lib.slab_restrict_vector(level._h, v_fine._h, out._h))
    return out


def refine_and_add(level: ProblemLevel, z: DenseVector, z_c: DenseVector) -> DenseVector:
    _check(_lib.slab_refine_and_add(level._h, z._h, z_c._h))
    return z


def mg_vcycle(level: ProblemLevel, z: DenseVector, r: DenseVector, cfg: SmootherConfig = SmootherConfig()):
    if cfg.sweeps < 1:
        raise InvalidArgument("SmootherConfig: sweeps must be at least 1")
    _check(_lib.slab_mg_vcycle(level._h, z._h, r._h, int(cfg.sweeps)))
    return z


# ---------------------------------------------------------------- cg.hpp


@dataclass
class CGConfig:  # cg.hpp:41-48
    max_iters: int = 500
    rtol: float = 1e-6
    use_preconditioner: bool = True
    fixed_iterations: Optional[int] = None


@dataclass
class CGResult:  # cg.hpp:50-56
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False
    solution: object = None
    solve_ms: float = 0.0


def _c_config(cfg: CGConfig, scfg: SmootherConfig) -> _CgConfig:
    if cfg.max_iters < 0 or (cfg.fixed_iterations is not None and cfg.fixed_iterations < 0) or scfg.sweeps < 0:
        raise InvalidArgument("CGConfig: negative counts")
    return _CgConfig(int(cfg.max_iters), float(cfg.rtol), int(cfg.use_preconditioner),
                     int(cfg.fixed_iterations is not None), int(cfg.fixed_iterations or 0), int(scfg.sweeps))


def _history_len(cfg: CGConfig) -> int:
    return max(int(cfg.max_iters), 1) + 1


def cg_solve(hierarchy: ProblemLevel, b: DenseVector, x0: DenseVector, cfg: CGConfig = CGConfig(),
             smoother_cfg: SmootherConfig = SmootherConfig(), out: Optional[DenseVector] = None) -> CGResult:
    """cg.hpp:77-142. `out` optionally supplies the solution vector (the reference returns a fresh
    one); reusing it across calls lets the library replay its cached iteration graph."""
    cc = _c_config(cfg, smoother_cfg)
    hist = np.zeros(_history_len(cfg), dtype=np.float64)
    res = _CgResult()
    x = out if out is not None else DenseVector(hierarchy.ctx, hierarchy.n())
    _check(_lib.slab_cg_solve(hierarchy._h, b._h, x0._h, C.byref(cc), x._h, _ptr(hist), C.byref(res)))
    k = int(res.iterations)
    return CGResult(k, [float(v) for v in hist[: k + 1]], bool(res.converged), x, float(res.solve_ms))


def cg_solve_host(hierarchy: ProblemLevel, b: np.ndarray, x0: np.ndarray, cfg: CGConfig = CGConfig(),
                  smoother_cfg: SmootherConfig = SmootherConfig(), out: Optional[np.ndarray] = None) -> CGResult:
    """cg_solve with HOST buffers: upload b/x0, solve, download x — the end-to-end plugin call."""
    cc = _c_config(cfg, smoother_cfg)
    b, x0 = _f64(b), _f64(x0)
    n = hierarchy.n()
    if b.size != n or x0.size != n:
        raise DimensionMismatch("cg_solve: vector lengths differ from the system size")
    hist = np.zeros(_history_len(cfg), dtype=np.float64)
    res = _CgResult()
    if out is not None:
        # the library writes n doubles through this pointer: anything but a writable, contiguous float64 array of
        # exactly n elements would be written past its end or into a temporary copy
        if not isinstance(out, np.ndarray) or out.dtype != np.float64 or not out.flags["C_CONTIGUOUS"] or not out.flags["WRITEABLE"]:
            raise InvalidArgument("cg_solve_host: out must be a writable C-contiguous float64 numpy array")
        if out.size != n:
            raise DimensionMismatch("cg_solve_host: out must have as many elements as the system has rows")
    x = out if out is not None else np.empty(n, dtype=np.float64)
    _check(_lib.slab_cg_solve_host(hierarchy._h, _ptr(b), _ptr(x0), b.size, C.byref(cc), _ptr(x), _ptr(hist),
                                   C.byref(res)))
    k = int(res.iterations)
    return CGResult(k, [float(v) for v in hist[: k + 1]], bool(res.converged), x, float(res.solve_ms))


def residual_norm(A: SparseMatrix, x: DenseVector, b: DenseVector) -> float:
    out = C.c_double()
    _check(_lib.slab_residual_norm(A._h, x._h, b._h, C.byref(out)))
    return out.value
