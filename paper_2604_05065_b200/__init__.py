"""B200-native APLICUR hot path: Python host mirror of the reference solver API.

The product is ``_lib/libapc_b200.so`` (hand-written sm_100a kernels + C++
host orchestration behind the C-ABI in ``include/apc_b200.h``).  This module is
a thin ctypes binding that mirrors the reference's public names
(/root/reference/proj/include/aplicur/solver.hpp:29-120, 162, 396):
``SolverConfig``, ``SolveResult``, ``PhaseReport``, ``aplicur_solve``,
``plain_lsqr_solve``, plus the operator products of ``Matrix`` /
``AugmentedOperator`` (matrix.hpp:151-195, 365-392).

There is no CPU fallback: every compute call goes through the CUDA library
and fails loudly (``ApcError``) when no device or no library is available.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
import weakref
from pathlib import Path
from typing import Optional

import numpy as np

_PKG = Path(__file__).resolve().parent
_HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int64, C.c_void_p)
LIB_PATH = _PKG / "_lib" / "libapc_b200.so"
HEADER_PATHS = [_PKG.parent / "include" / "apc_b200.h"]

_i64 = C.c_int64
_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)

APC_OK = 0
APC_NO_DEVICE = 22

ERROR_KINDS = {  # aplicur::ErrorKind + 1 (error.hpp:10-20)
    1: "invalid_argument", 2: "dimension_mismatch", 3: "rank_deficient", 4: "singular",
    5: "not_positive", 6: "no_convergence", 7: "numerical_breakdown", 8: "not_applicable",
    9: "io", 20: "cuda", 21: "nccl", 22: "no_device",
}


class ApcError(RuntimeError):
    """aplicur::Error equivalent: ``kind`` (ErrorKind name) and ``index``."""

    def __init__(self, code: int, msg: str, index: int = -1):
        super().__init__(f"[{ERROR_KINDS.get(code, code)}] {msg}")
        self.code = code
        self.kind = ERROR_KINDS.get(code, str(code))
        self.index = index


class StopReason(enum.IntEnum):  # lsqr.hpp:17-24
    none = 0
    gradient_tol = 1
    dynamic_rate = 2
    dynamic_diff = 3
    iteration_cap = 4
    exact_zero_rhs = 5


class SolveStatus(enum.IntEnum):  # solver.hpp:90
    converged = 0
    rank_exhausted = 1
    breakdown = 2


class PrecondVariant(enum.IntEnum):  # solver.hpp:21
    svd = 0
    svd_free = 1


class CoreFactorKind(enum.IntEnum):  # cur.hpp:50
    qr = 0
    lu = 1


class SketchKind(enum.IntEnum):
    sparse_sign = 0
    gaussian = 1          # exact order: Y bit-identical to GaussianEmbedding::apply
    gaussian_dmma = 2     # opt-in FP64 tensor-core (DMMA) sketch: Y rounded differently


class _Config(C.Structure):
    _fields_ = [
        ("block", _i64), ("eps_cur", C.c_double), ("eps_lsqr", C.c_double),
        ("nu_prec", C.c_double), ("nu_lsqr", C.c_double), ("mu", C.c_double),
        ("variant", C.c_int32), ("core", C.c_int32), ("sketch_xi", _i64),
        ("probe_count", _i64), ("lsqr_cap", _i64), ("max_rank", _i64), ("seed", _u64),
        ("trace_sample_stride", _i64), ("outer_cap", _i64), ("sketch_kind", C.c_int32),
        ("reserved", C.c_int32),
    ]


class _RebuildInfo(C.Structure):  # apc_rebuild_info
    _fields_ = [("phase", C.c_int32), ("variant", C.c_int32), ("rank", C.c_int64),
                ("rows", C.POINTER(C.c_int64)), ("cols", C.POINTER(C.c_int64)), ("rho", C.c_double),
                ("sigma_hat", C.c_double), ("sigma_floor", C.c_double), ("sigma_cur", C.POINTER(C.c_double)),
                ("sigma_reg", C.POINTER(C.c_double)), ("n_sigma", C.c_int64)]


_REBUILD_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(_RebuildInfo))
_PHASE_END_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.c_int64)


class _Hooks(C.Structure):  # apc_hooks
    _fields_ = [("user", C.c_void_p), ("on_rebuild", _REBUILD_FN), ("on_phase_end", _PHASE_END_FN)]


class _Phase(C.Structure):
    _fields_ = [
        ("phase", C.c_int32), ("reason", C.c_int32), ("rank", _i64), ("rho", C.c_double),
        ("sigma_hat", C.c_double), ("mu", C.c_double), ("lsqr_iters", _i64),
        ("t_augment_ms", C.c_double), ("t_factor_ms", C.c_double), ("t_precond_ms", C.c_double),
        ("t_lsqr_ms", C.c_double), ("relres_at_end", C.c_double), ("t_lsqr_device_ms", C.c_double),
    ]


class _Trace(C.Structure):
    _fields_ = [
        ("phase", C.c_int32), ("pad", C.c_int32), ("iter", _i64), ("phibar", C.c_double),
        ("cvgrate", C.c_double), ("cvgdiff", C.c_double), ("matvecs", _u64),
        ("wall_ms", C.c_double), ("true_relres", C.c_double),
    ]


_lib = None


def _preload_nccl() -> None:
    """One NCCL per process: the library links libnccl.so.2 by soname.  When
    torch is in the same process it needs its bundled NCCL (newer symbols), so
    that copy is loaded first when present; whichever is loaded first then
    satisfies both."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        cand = Path(base) / "nccl" / "lib" / "libnccl.so.2"
        if cand.exists():
            try:
                C.CDLL(str(cand), mode=C.RTLD_GLOBAL)
            except OSError:
                pass
            return


def load_library(path: Optional[os.PathLike] = None) -> C.CDLL:
    """Load libapc_b200.so (in-tree build).  Raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # APC_LIB_PATH: an alternative build of the same library (kernel-variant
    # experiments, scripts/build_variant.py); the default is the in-tree build
    p = Path(path) if path else Path(os.environ.get("APC_LIB_PATH") or LIB_PATH)
    if not p.exists():
        raise ApcError(20, f"CUDA library missing: {p} (run __graft_entry__.build())")
    _preload_nccl()
    lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    vp = C.c_void_p
    sig = {
        "apc_abi_version": (C.c_int, []),
        "apc_last_error": (C.c_char_p, [_i64p]),
        "apc_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "apc_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, C.POINTER(vp)]),
        "apc_ctx_destroy": (C.c_int, [vp]),
        "apc_nccl_unique_id": (C.c_int, [vp]),
        "apc_ctx_create_host_comm": (C.c_int, [C.c_int, C.c_int, C.c_int, _HOST_ALLREDUCE, vp, C.POINTER(vp)]),
        "apc_ctx_stream": (vp, [vp]),
        "apc_ctx_launches": (_u64, [vp]),
        "apc_ctx_sync": (C.c_int, [vp]),
        "apc_mat_upload_dense": (C.c_int, [vp, _i64, _i64, _dp, _i64, _i64, C.POINTER(vp)]),
        "apc_mat_upload_csc": (C.c_int, [vp, _i64, _i64, _i64p, _i64p, _dp, _i64, _i64, C.POINTER(vp)]),
        "apc_mat_free": (C.c_int, [vp]),
        "apc_mat_info": (C.c_int, [vp, _i64p, _i64p, _i64p, C.POINTER(C.c_int), _i64p, _i64p]),
        "apc_op_apply_dev": (C.c_int, [vp, C.c_double, C.c_int, C.c_int, vp, vp]),
        "apc_op_pair_dev": (C.c_int, [vp, vp, vp, vp, C.POINTER(C.c_int)]),
        "apc_dgemm": (C.c_int, [vp, C.c_int, C.c_int, _i64, _i64, _i64, C.c_double, vp, _i64, vp, _i64, C.c_double,
                                vp, _i64]),
        "apc_dtrsm_right_upper": (C.c_int, [vp, _i64, _i64, vp, _i64, vp, _i64]),
        "apc_dpotrf_upper": (C.c_int, [vp, _i64, vp, _i64p]),
        "apc_dtrsm_rows": (C.c_int, [vp, _i64, vp, vp, _i64, C.c_int]),
        "apc_op_apply_host": (C.c_int, [vp, C.c_double, C.c_int, C.c_int, _dp, _dp]),
        "apc_partition_rows": (C.c_int, [_i64, _i64p, C.c_int, _i64p]),
        "apc_rng_fill": (C.c_int, [_u64, C.c_int, _u64, C.c_int, _u64, _i64, vp]),
        "apc_mix64": (_u64, [_u64]),
        "apc_rng_fill_device": (C.c_int, [vp, _u64, C.c_int, _u64, _i64, C.POINTER(_u64)]),
        "apc_problem_generate": (C.c_int, [C.c_int, _i64, _i64, _u64, C.POINTER(vp)]),
        "apc_problem_info": (C.c_int, [vp, _i64p, _i64p, C.POINTER(C.c_int), _i64p]),
        "apc_problem_dense": (vp, [vp]),
        "apc_problem_csc": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
        "apc_problem_b": (vp, [vp]),
        "apc_problem_free": (C.c_int, [vp]),
        "apc_config_default": (C.c_int, [C.POINTER(_Config)]),
        "apc_solve": (C.c_int, [vp, _dp, C.POINTER(_Config), C.c_int, C.POINTER(vp)]),
        "apc_solve_sharded": (C.c_int, [vp, vp, _dp, C.POINTER(_Config), C.c_int, C.POINTER(vp)]),
        "apc_result_free": (C.c_int, [vp]),
        "apc_result_summary": (C.c_int, [vp, C.POINTER(C.c_int), _dp, _dp, C.POINTER(_u64),
                                         C.POINTER(_u64), _i64p, _i64p, _i64p, _i64p]),
        "apc_result_x": (C.c_int, [vp, _dp]),
        "apc_result_indices": (C.c_int, [vp, _i64p, _i64p]),
        "apc_result_rho_history": (C.c_int, [vp, _dp]),
        "apc_result_phases": (C.c_int, [vp, C.POINTER(_Phase)]),
        "apc_result_phase_spectrum": (C.c_int, [vp, _i64, _dp, _i64p]),
        "apc_solve_hooked": (C.c_int, [vp, vp, _dp, C.POINTER(_Config), C.POINTER(_Hooks), C.POINTER(vp)]),
        "apc_result_trace": (C.c_int, [vp, C.POINTER(_Trace)]),
        "apc_result_timing": (C.c_int, [vp, _dp, _dp, _dp]),
        "apc_cur_create": (C.c_int, [vp, _i64, _u64, _i64, _i64, C.c_int, C.c_int, C.POINTER(vp)]),
        "apc_cur_free": (C.c_int, [vp]),
        "apc_cur_augment": (C.c_int, [vp, _i64p, C.POINTER(C.c_int)]),
        "apc_cur_refresh": (C.c_int, [vp]),
        "apc_cur_rollback_last_augment": (C.c_int, [vp]),
        "apc_cur_state": (C.c_int, [vp, _i64p, _dp, _i64p, _i64p]),
        "apc_cur_indices": (C.c_int, [vp, _i64p, _i64p]),
        "apc_cur_rho_history": (C.c_int, [vp, _dp]),
        "apc_cur_timing": (C.c_int, [vp, _dp, _dp]),
        "apc_cur_sketch": (C.c_int, [vp, _dp]),
        "apc_cur_residual": (C.c_int, [vp, _dp]),
        "apc_lupp": (C.c_int, [vp, _dp, _i64, _i64, _i64, _i64p, _dp, _i64p]),
        "apc_mm_write_csc": (C.c_int, [C.c_char_p, _i64, _i64, _i64p, _i64p, _dp]),
        "apc_mm_write_dense": (C.c_int, [C.c_char_p, _i64, _i64, _dp]),
        "apc_mm_read": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
        "apc_trace_csv_write": (C.c_int, [C.c_char_p, C.POINTER(_Trace), _i64, C.POINTER(_Phase), _i64, C.c_int32]),
        "apc_report_json_write": (C.c_int, [C.c_char_p, C.POINTER(_Config), C.c_int32, C.c_double, C.c_double,
                                            _u64, _u64, C.c_char_p, _i64p, _i64p, _i64, _dp, _i64,
                                            C.POINTER(_Phase), _i64, C.POINTER(_dp), _i64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(code: int) -> None:
    if code != APC_OK:
        idx = _i64(-1)
        msg = load_library().apc_last_error(C.byref(idx)).decode()
        raise ApcError(code, msg, idx.value)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def device_count() -> int:
    n = C.c_int(0)
    _check(load_library().apc_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------------------
# context / matrices
# ---------------------------------------------------------------------------
class Context:
    """One GPU (rank) worth of stream, scratch and communicator: NCCL (nccl_uid
    from rank 0), or host-staged collectives through ``host_allreduce(buf)``, a
    callable that replaces the float64 numpy array ``buf`` in place by its sum
    over the ranks, added in rank order (apc_ctx_create_host_comm)."""

    def __init__(self, device: int = 0, nranks: int = 1, rank: int = 0,
                 nccl_uid: Optional[bytes] = None, host_allreduce=None):
        lib = load_library()
        h = C.c_void_p()
        if host_allreduce is not None:
            def _cb(buf, count, _user):
                try:
                    host_allreduce(np.ctypeslib.as_array(buf, shape=(count,)))
                    return 0
                except Exception:  # reported as a comm error by the library
                    return 1
            self._host_cb = _HOST_ALLREDUCE(_cb)  # kept alive with the ctx
            _check(lib.apc_ctx_create_host_comm(device, nranks, rank, self._host_cb, None, C.byref(h)))
        else:
            uid = C.create_string_buffer(nccl_uid, 128) if nccl_uid else None
            _check(lib.apc_ctx_create(device, nranks, rank, uid, C.byref(h)))
        self.h = h
        self.device, self.nranks, self.rank = device, nranks, rank
        self._children = weakref.WeakSet()  # device objects freed before the ctx

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(load_library().apc_nccl_unique_id(buf))
        return buf.raw

    @property
    def stream(self) -> int:
        return load_library().apc_ctx_stream(self.h) or 0

    @property
    def launches(self) -> int:
        return int(load_library().apc_ctx_launches(self.h))

    def sync(self) -> None:
        _check(load_library().apc_ctx_sync(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            for c in list(self._children):
                c.close()
            load_library().apc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceMatrix:
    """Device-resident A (dense column-major, or CSR(A) + CSR(A^T) from CSC)."""

    def __init__(self, ctx: Context, h, m: int, n: int, sparse: bool, r0: int, r1: int, keep=None):
        self.ctx, self.h, self.m, self.n, self.sparse, self.r0, self.r1 = ctx, h, m, n, sparse, r0, r1
        self._keep = keep
        ctx._children.add(self)

    @classmethod
    def dense(cls, ctx: Context, a_colmajor: np.ndarray, m: int, n: int, r0: int = 0,
              r1: Optional[int] = None) -> "DeviceMatrix":
        a = np.ascontiguousarray(a_colmajor, dtype=np.float64).reshape(-1)
        assert a.size == m * n
        r1 = m if r1 is None else r1
        h = C.c_void_p()
        _check(load_library().apc_mat_upload_dense(ctx.h, m, n, _dptr(a), r0, r1, C.byref(h)))
        return cls(ctx, h, m, n, False, r0, r1)

    @classmethod
    def from_numpy(cls, ctx: Context, A: np.ndarray, **kw) -> "DeviceMatrix":
        m, n = A.shape
        return cls.dense(ctx, np.asfortranarray(A, dtype=np.float64).reshape(-1, order="F"), m, n, **kw)

    @classmethod
    def csc(cls, ctx: Context, m: int, n: int, colptr, rowidx, vals, r0: int = 0,
            r1: Optional[int] = None) -> "DeviceMatrix":
        cp = np.ascontiguousarray(colptr, dtype=np.int64)
        ri = np.ascontiguousarray(rowidx, dtype=np.int64)
        va = np.ascontiguousarray(vals, dtype=np.float64)
        r1 = m if r1 is None else r1
        h = C.c_void_p()
        _check(load_library().apc_mat_upload_csc(ctx.h, m, n, _iptr(cp), _iptr(ri), _dptr(va), r0, r1,
                                                 C.byref(h)))
        return cls(ctx, h, m, n, True, r0, r1)

    @classmethod
    def from_problem(cls, ctx: Context, p: "Problem", r0: int = 0, r1: Optional[int] = None):
        if p.sparse:
            return cls.csc(ctx, p.m, p.n, p.colptr, p.rowidx, p.vals, r0, r1)
        return cls.dense(ctx, p.dense, p.m, p.n, r0, r1)

    @property
    def mloc(self) -> int:
        return self.r1 - self.r0

    def apply(self, x: np.ndarray, mu: float = 0.0, augmented: bool = False,
              transpose: bool = False) -> np.ndarray:
        """y = A_mu x  (or A_mu^T x), host buffers (matrix.hpp:151-195, 377-392)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        tail = self.n if augmented else 0
        out = np.empty(self.n if transpose else self.mloc + tail)
        _check(load_library().apc_op_apply_host(self.h, mu, int(augmented), int(transpose),
                                                _dptr(x), _dptr(out)))
        return out

    def apply_dev(self, x_ptr: int, y_ptr: int, mu: float = 0.0, augmented: bool = False,
                  transpose: bool = False) -> None:
        _check(load_library().apc_op_apply_dev(self.h, mu, int(augmented), int(transpose),
                                               C.c_void_p(x_ptr), C.c_void_p(y_ptr)))

    def pair_dev(self, x_ptr: int, y_ptr: int, g_ptr: int) -> bool:
        """y = A x, g[0:n] = A^T y, g[n] = ||y||^2 on device pointers (the LSQR
        operator pair); True when the fused read-A-once kernel ran."""
        fused = C.c_int(0)
        _check(load_library().apc_op_pair_dev(self.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_void_p(g_ptr),
                                              C.byref(fused)))
        return bool(fused.value)

    def free(self) -> None:
        if getattr(self, "h", None):
            if getattr(self.ctx, "h", None):  # a closed ctx already freed it
                load_library().apc_mat_free(self.h)
            self.h = None

    close = free

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class CurState:
    """Device CurState (cur.hpp:200-371): single sketch, incremental augment /
    refresh with exact-order kernels (bit-identical indices and rho)."""

    def __init__(self, mat: DeviceMatrix, block: int, seed: int, xi: int = 8, probe_count: int = 10,
                 core: CoreFactorKind = CoreFactorKind.qr, sketch: SketchKind = SketchKind.sparse_sign):
        h = C.c_void_p()
        _check(load_library().apc_cur_create(mat.h, block, seed, xi, probe_count, int(core), int(sketch),
                                             C.byref(h)))
        self.h, self.mat = h, mat
        mat.ctx._children.add(self)

    def augment(self):
        added, ex = _i64(), C.c_int()
        _check(load_library().apc_cur_augment(self.h, C.byref(added), C.byref(ex)))
        return added.value, bool(ex.value)

    def refresh(self) -> None:
        _check(load_library().apc_cur_refresh(self.h))

    def rollback_last_augment(self) -> None:
        _check(load_library().apc_cur_rollback_last_augment(self.h))

    def _state(self):
        r, rho, s, nr = _i64(), C.c_double(), _i64(), _i64()
        load_library().apc_cur_state(self.h, C.byref(r), C.byref(rho), C.byref(s), C.byref(nr))
        return r.value, rho.value, s.value, nr.value

    def rank(self) -> int:
        return self._state()[0]

    def rho(self) -> float:
        return self._state()[1]

    def indices(self):
        r = self.rank()
        rows, cols = np.zeros(r, np.int64), np.zeros(r, np.int64)
        load_library().apc_cur_indices(self.h, _iptr(rows), _iptr(cols))
        return rows, cols

    def sketch_timing(self):
        """(host embedding generation ms, device sketch kernel ms)."""
        e, k = C.c_double(), C.c_double()
        load_library().apc_cur_timing(self.h, C.byref(e), C.byref(k))
        return e.value, k.value

    def rho_history(self) -> np.ndarray:
        out = np.zeros(self._state()[3])
        load_library().apc_cur_rho_history(self.h, _dptr(out))
        return out

    def sketch_matrix(self) -> np.ndarray:
        s = self._state()[2]
        y = np.zeros(s * self.mat.n)
        _check(load_library().apc_cur_sketch(self.h, _dptr(y)))
        return y.reshape(self.mat.n, s).T

    def sketch_residual(self) -> np.ndarray:
        s = self._state()[2]
        y = np.zeros(s * self.mat.n)
        _check(load_library().apc_cur_residual(self.h, _dptr(y)))
        return y.reshape(self.mat.n, s).T

    def close(self):
        if getattr(self, "h", None):
            if getattr(self.mat.ctx, "h", None):
                load_library().apc_cur_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lu_partial_pivot(ctx: Context, W: np.ndarray, max_pivots: int = -1):
    """Pivot order + magnitudes of partial-pivoting LU (dense_factor.hpp:119-157), on the GPU."""
    rows, cols = W.shape
    w = np.asfortranarray(W, dtype=np.float64).reshape(-1, order="F")
    k = min(rows, cols) if max_pivots < 0 else min(rows, cols, max_pivots)
    order, mags, ns = np.zeros(max(k, 1), np.int64), np.zeros(max(k, 1)), _i64()
    _check(load_library().apc_lupp(ctx.h, _dptr(w), rows, cols, max_pivots, _iptr(order), _dptr(mags),
                                   C.byref(ns)))
    return order[: ns.value], mags[: ns.value]


def partition_rows(m: int, nranks: int, row_nnz: Optional[np.ndarray] = None) -> np.ndarray:
    b = np.zeros(nranks + 1, dtype=np.int64)
    rn = None if row_nnz is None else np.ascontiguousarray(row_nnz, dtype=np.int64)
    _check(load_library().apc_partition_rows(m, None if rn is None else _iptr(rn), nranks, _iptr(b)))
    return b


def rng_fill(seed: int, kind: int, count: int, stream: int = -1, index: int = 0, bound: int = 0):
    out = np.empty(count, dtype=np.uint64 if kind in (0, 3) else np.float64)
    _check(load_library().apc_rng_fill(seed, stream, index, kind, bound, count, out.ctypes.data_as(C.c_void_p)))
    return out


# ---------------------------------------------------------------------------
# synthetic BASELINE problems
# ---------------------------------------------------------------------------
class Problem:
    """Host copy of a generated BASELINE input (same bytes for oracle and GPU)."""

    def __init__(self, config: int, m: int = 0, n: int = 0, seed: int = 0, _handle=None):
        lib = load_library()
        if _handle is None:
            h = C.c_void_p()
            _check(lib.apc_problem_generate(config, m, n, seed, C.byref(h)))
        else:
            h = _handle
        mm, nn, nz, sp = _i64(), _i64(), _i64(), C.c_int()
        lib.apc_problem_info(h, C.byref(mm), C.byref(nn), C.byref(sp), C.byref(nz))
        self.config, self.m, self.n, self.sparse, self.nnz = config, mm.value, nn.value, bool(sp.value), nz.value
        bp = lib.apc_problem_b(h)
        self.b = np.ctypeslib.as_array(C.cast(bp, _dp), shape=(self.m,)).copy()
        if self.sparse:
            cp, ri, va = C.c_void_p(), C.c_void_p(), C.c_void_p()
            lib.apc_problem_csc(h, C.byref(cp), C.byref(ri), C.byref(va))
            self.colptr = np.ctypeslib.as_array(C.cast(cp, _i64p), shape=(self.n + 1,)).copy()
            self.rowidx = np.ctypeslib.as_array(C.cast(ri, _i64p), shape=(self.nnz,)).copy()
            self.vals = np.ctypeslib.as_array(C.cast(va, _dp), shape=(self.nnz,)).copy()
            self.dense = None
        else:
            dp = lib.apc_problem_dense(h)
            self.dense = np.ctypeslib.as_array(C.cast(dp, _dp), shape=(self.m * self.n,)).copy()
        lib.apc_problem_free(h)

    def to_numpy(self) -> np.ndarray:
        if not self.sparse:
            return self.dense.reshape(self.n, self.m).T
        A = np.zeros((self.m, self.n))
        for j in range(self.n):
            A[self.rowidx[self.colptr[j]:self.colptr[j + 1]], j] = self.vals[self.colptr[j]:self.colptr[j + 1]]
        return A


# ---------------------------------------------------------------------------
# solver API (solver.hpp:29-120)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class SolverConfig:
    block: int = 0
    eps_cur: float = -1.0
    eps_lsqr: float = 1e-10
    nu_prec: float = 10.0
    nu_lsqr: float = 100.0
    mu: float = 0.0
    variant: PrecondVariant = PrecondVariant.svd
    sketch_xi: int = 8
    probe_count: int = 10
    lsqr_cap: int = 0
    max_rank: int = 0
    seed: int = 0
    core: CoreFactorKind = CoreFactorKind.qr
    trace_sample_stride: int = 1
    outer_cap: int = 100000
    sketch_kind: SketchKind = SketchKind.sparse_sign

    def _c(self) -> _Config:
        c = _Config()
        load_library().apc_config_default(C.byref(c))
        for f in dataclasses.fields(self):
            setattr(c, f.name, int(getattr(self, f.name)) if isinstance(getattr(self, f.name), enum.Enum)
                    else getattr(self, f.name))
        return c


@dataclasses.dataclass
class PhaseReport:
    phase: int
    rank: int
    rho: float
    sigma_hat: float
    mu: float
    lsqr_iters: int
    reason: StopReason
    t_augment_ms: float
    t_factor_ms: float
    t_precond_ms: float
    t_lsqr_ms: float
    relres_at_end: float
    t_lsqr_device_ms: float = 0.0
    precond_spectrum: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0))  # svd variant only


@dataclasses.dataclass
class SolveResult:
    x: np.ndarray
    phases: list
    trace: np.ndarray  # structured rows (phase, iter, phibar, cvgrate, cvgdiff, matvecs, wall_ms, true_relres)
    status: SolveStatus
    final_rho: float
    final_relres: float
    sketch_applications: int
    system_matvecs: int
    row_indices: np.ndarray
    col_indices: np.ndarray
    rho_history: np.ndarray
    total_ms: float = 0.0
    lsqr_ms: float = 0.0
    setup_ms: float = 0.0
    _raw_phases: object = None  # ctypes apc_phase_report array (for the report writers)

    @property
    def lsqr_iters(self) -> int:
        return int(sum(p.lsqr_iters for p in self.phases))

    def _phase_array(self):
        if self._raw_phases is not None:
            return self._raw_phases
        arr = (_Phase * max(1, len(self.phases)))()
        for k, p in enumerate(self.phases):
            arr[k] = _Phase(p.phase, int(p.reason), p.rank, p.rho, p.sigma_hat, p.mu, p.lsqr_iters, p.t_augment_ms,
                            p.t_factor_ms, p.t_precond_ms, p.t_lsqr_ms, p.relres_at_end, p.t_lsqr_device_ms)
        return arr

    def write_trace_csv(self, path) -> None:
        """report_io.hpp:28-47 -- one row per LSQR iteration, reason on each phase's last row."""
        rows = np.ascontiguousarray(self.trace)
        reason = int(self.phases[-1].reason) if self.phases else 0
        _check(load_library().apc_trace_csv_write(str(path).encode(), rows.ctypes.data_as(C.POINTER(_Trace)),
                                                  len(rows), self._phase_array(), len(self.phases), reason))

    def write_report_json(self, path, config: "SolverConfig", trace_path: str = "") -> None:
        """report_io.hpp:94-110 -- solve report (config, status, CUR indices, phases), atomic write."""
        c = config._c()
        ri = np.ascontiguousarray(self.row_indices, dtype=np.int64)
        ci = np.ascontiguousarray(self.col_indices, dtype=np.int64)
        rho = np.ascontiguousarray(self.rho_history, dtype=np.float64)
        specs = [np.ascontiguousarray(p.precond_spectrum, dtype=np.float64) for p in self.phases]
        sp = (_dp * max(1, len(specs)))(*[_dptr(a) for a in specs])
        nsp = np.array([a.size for a in specs] or [0], dtype=np.int64)
        _check(load_library().apc_report_json_write(
            str(path).encode(), C.byref(c), int(self.status), self.final_relres, self.final_rho,
            self.sketch_applications, self.system_matvecs, str(trace_path).encode(), _iptr(ri), _iptr(ci), len(ri),
            _dptr(rho), len(rho), self._phase_array(), len(self.phases), sp, _iptr(nsp)))


def _collect(h) -> SolveResult:
    lib = load_library()
    st, nph, ntr, rk, nrho = C.c_int(), _i64(), _i64(), _i64(), _i64()
    frho, frel = C.c_double(), C.c_double()
    sk, smv = _u64(), _u64()
    lib.apc_result_summary(h, C.byref(st), C.byref(frho), C.byref(frel), C.byref(sk), C.byref(smv),
                           C.byref(nph), C.byref(ntr), C.byref(rk), C.byref(nrho))
    # x length: ask via trace-free path -> use phases' knowledge: stored n in result
    phases = (_Phase * max(1, nph.value))()
    lib.apc_result_phases(h, phases)
    trace = (_Trace * max(1, ntr.value))()
    lib.apc_result_trace(h, trace)
    rows = np.zeros(rk.value, dtype=np.int64)
    cols = np.zeros(rk.value, dtype=np.int64)
    lib.apc_result_indices(h, _iptr(rows), _iptr(cols))
    rho = np.zeros(nrho.value)
    lib.apc_result_rho_history(h, _dptr(rho))
    tt, tl, ts = C.c_double(), C.c_double(), C.c_double()
    lib.apc_result_timing(h, C.byref(tt), C.byref(tl), C.byref(ts))
    tr = np.ctypeslib.as_array(trace)[: ntr.value].copy()
    specs = []
    for k in range(nph.value):
        ns = _i64()
        lib.apc_result_phase_spectrum(h, k, None, C.byref(ns))
        a = np.zeros(ns.value)
        lib.apc_result_phase_spectrum(h, k, _dptr(a), C.byref(ns))
        specs.append(a)
    ph = [PhaseReport(p.phase, p.rank, p.rho, p.sigma_hat, p.mu, p.lsqr_iters, StopReason(p.reason),
                      p.t_augment_ms, p.t_factor_ms, p.t_precond_ms, p.t_lsqr_ms, p.relres_at_end,
                      p.t_lsqr_device_ms, specs[k])
          for k, p in enumerate(phases[: nph.value])]
    return SolveResult(None, ph, tr, SolveStatus(st.value), frho.value, frel.value, sk.value, smv.value,
                       rows, cols, rho, tt.value, tl.value, ts.value, phases)


@dataclasses.dataclass
class CurStateView:
    """Host summary of the device CUR state handed to on_rebuild (cur.hpp:228-242)."""
    rank: int
    row_indices: np.ndarray
    col_indices: np.ndarray
    rho: float


@dataclasses.dataclass
class PreconditionerView:
    """Host summary of the device preconditioner (preconditioner.hpp:19-56)."""
    rank: int
    variant: PrecondVariant
    target_level: float
    smallest_cur_sigma: float
    cur_spectrum: np.ndarray  # svd variant only (else empty)
    regularized_spectrum: np.ndarray


@dataclasses.dataclass
class SolveHooks:
    """SolveHooks (solver.hpp:114-120): diagnostic observers.

    on_rebuild(cur: CurStateView, precond: PreconditionerView, phase) runs after
    each preconditioner build, before its LSQR phase; on_phase_end(phase, x)
    at the end of every phase with x so far."""
    on_rebuild: Optional[object] = None
    on_phase_end: Optional[object] = None


def _hook_struct(hooks: SolveHooks, errors: list):
    def rebuild(_user, info_p):
        if errors:
            return
        try:
            ri = info_p.contents
            k, ns = ri.rank, ri.n_sigma
            cv = CurStateView(k, np.ctypeslib.as_array(ri.rows, (k,)).copy() if k else np.zeros(0, np.int64),
                              np.ctypeslib.as_array(ri.cols, (k,)).copy() if k else np.zeros(0, np.int64), ri.rho)
            sc = np.ctypeslib.as_array(ri.sigma_cur, (ns,)).copy() if ns and ri.sigma_cur else np.zeros(0)
            sr = np.ctypeslib.as_array(ri.sigma_reg, (ns,)).copy() if ns and ri.sigma_reg else np.zeros(0)
            pv = PreconditionerView(k, PrecondVariant(ri.variant), ri.sigma_hat, ri.sigma_floor, sc, sr)
            hooks.on_rebuild(cv, pv, ri.phase)
        except BaseException as e:  # re-raised after the solve returns
            errors.append(e)

    def phase_end(_user, phase, x, n):
        if errors:
            return
        try:
            hooks.on_phase_end(int(phase), np.ctypeslib.as_array(x, (n,)).copy())
        except BaseException as e:
            errors.append(e)

    fr = _REBUILD_FN(rebuild) if hooks.on_rebuild else _REBUILD_FN()
    fp = _PHASE_END_FN(phase_end) if hooks.on_phase_end else _PHASE_END_FN()
    return _Hooks(None, fr, fp), (fr, fp)


def solve(mat: DeviceMatrix, b: np.ndarray, config: SolverConfig, plain: bool = False,
          full: Optional[DeviceMatrix] = None, hooks: Optional[SolveHooks] = None) -> SolveResult:
    """Run aplicur_solve (plain=False) or plain_lsqr_solve on a device-resident A.

    On a multi-rank context ``mat`` is this rank's row block (row-partitioned
    multi-GPU solve: one allreduce per LSQR iteration).  Root-only setup:
    rank 0 passes ``full``, the whole matrix, and the sketch, the CUR
    selection and every preconditioner build run there and are broadcast.
    Sharded setup: every rank passes ``full=None`` and no rank holds the whole
    matrix (carried sketch, row pivots over the shards, R rows from their
    owners; the same indices as one rank)."""
    lib = load_library()
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert b.size == mat.m
    c = config._c()
    h = C.c_void_p()
    errors: list = []
    if hooks is not None and not plain and (hooks.on_rebuild or hooks.on_phase_end):
        hs, _keep = _hook_struct(hooks, errors)
        _check(lib.apc_solve_hooked(None if full is None else full.h, mat.h, _dptr(b), C.byref(c), C.byref(hs),
                                    C.byref(h)))
    elif full is not None or mat.ctx.nranks > 1:
        _check(lib.apc_solve_sharded(None if full is None else full.h, mat.h, _dptr(b), C.byref(c), int(plain),
                                     C.byref(h)))
    else:
        _check(lib.apc_solve(mat.h, _dptr(b), C.byref(c), int(plain), C.byref(h)))
    try:
        res = _collect(h)
        x = np.zeros(mat.n)
        lib.apc_result_x(h, _dptr(x))
        res.x = x
    finally:
        lib.apc_result_free(h)
    if errors:
        raise errors[0]
    return res


def aplicur_solve(mat: DeviceMatrix, b: np.ndarray, config: SolverConfig,
                  full: Optional[DeviceMatrix] = None, hooks: Optional[SolveHooks] = None) -> SolveResult:
    """solver.hpp:162 -- adaptive CUR-preconditioned LSQR."""
    return solve(mat, b, config, plain=False, full=full, hooks=hooks)


def plain_lsqr_solve(mat: DeviceMatrix, b: np.ndarray, config: SolverConfig) -> SolveResult:
    """solver.hpp:396 -- unpreconditioned LSQR baseline."""
    return solve(mat, b, config, plain=True)


def read_matrix_market(path) -> Problem:
    """matrix_market.hpp:48-116 -- a host Problem (b = zeros(m)) from a Matrix Market file."""
    h = C.c_void_p()
    _check(load_library().apc_mm_read(str(path).encode(), C.byref(h)))
    return Problem(0, _handle=h)


def write_matrix_market(path, a) -> None:
    """matrix_market.hpp:18-46 -- coordinate (a sparse Problem, or (m, n, colptr, rowidx, vals))
    or array (a dense Problem, or a 2-D numpy array) with %.17g values."""
    lib = load_library()
    if isinstance(a, Problem):
        if a.sparse:
            cp, ri, va = (np.ascontiguousarray(x) for x in (a.colptr, a.rowidx, a.vals))
            _check(lib.apc_mm_write_csc(str(path).encode(), a.m, a.n, _iptr(cp), _iptr(ri), _dptr(va)))
        else:
            d = np.ascontiguousarray(a.dense, dtype=np.float64)
            _check(lib.apc_mm_write_dense(str(path).encode(), a.m, a.n, _dptr(d)))
    elif isinstance(a, tuple):
        m, n, cp, ri, va = a
        cp = np.ascontiguousarray(cp, dtype=np.int64)
        ri = np.ascontiguousarray(ri, dtype=np.int64)
        va = np.ascontiguousarray(va, dtype=np.float64)
        _check(lib.apc_mm_write_csc(str(path).encode(), m, n, _iptr(cp), _iptr(ri), _dptr(va)))
    else:
        A = np.asarray(a, dtype=np.float64)
        d = np.ascontiguousarray(A.T).reshape(-1)  # column-major
        _check(lib.apc_mm_write_dense(str(path).encode(), A.shape[0], A.shape[1], _dptr(d)))


__all__ = [
    "ApcError", "StopReason", "SolveStatus", "PrecondVariant", "CoreFactorKind", "SketchKind",
    "Context", "DeviceMatrix", "Problem", "SolverConfig", "SolveResult", "PhaseReport",
    "aplicur_solve", "plain_lsqr_solve", "solve", "load_library", "device_count",
    "partition_rows", "rng_fill", "LIB_PATH", "HEADER_PATHS", "CurState", "lu_partial_pivot",
    "read_matrix_market", "write_matrix_market",
]
