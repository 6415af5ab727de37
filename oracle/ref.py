"""ORACLE / TEST INFRASTRUCTURE ONLY -- ctypes binding to oracle/_ref/libaplicur_ref.so,
the unmodified APLICUR reference (/root/reference/proj/include) compiled by
oracle/Makefile.  Used by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference arm as the checker; never by the product path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libaplicur_ref.so"
REF_INC = Path("/root/reference/proj/include")

_i64, _u64, _i32 = C.c_int64, C.c_uint64, C.c_int32
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class RefProblem(C.Structure):
    _fields_ = [("m", _i64), ("n", _i64), ("sparse", _i32), ("dense", _dp), ("colptr", _i64p),
                ("rowidx", _i64p), ("vals", _dp)]


class RefConfig(C.Structure):
    _fields_ = [("block", _i64), ("eps_cur", C.c_double), ("eps_lsqr", C.c_double),
                ("nu_prec", C.c_double), ("nu_lsqr", C.c_double), ("mu", C.c_double),
                ("variant", _i32), ("sketch_xi", _i64), ("probe_count", _i64), ("lsqr_cap", _i64),
                ("max_rank", _i64), ("seed", _u64), ("core", _i32), ("trace_sample_stride", _i64),
                ("outer_cap", _i64)]


class RefOut(C.Structure):
    _fields_ = [("x", _dp), ("status", _i32), ("final_rho", C.c_double), ("final_relres", C.c_double),
                ("sketch_applications", _u64), ("system_matvecs", _u64),
                ("row_idx", _i64p), ("col_idx", _i64p), ("n_idx", _i64), ("cap_idx", _i64),
                ("rho_hist", _dp), ("n_rho", _i64), ("cap_rho", _i64),
                ("ph_rank", _i64p), ("ph_iters", _i64p), ("ph_reason", C.POINTER(_i32)),
                ("ph_rho", _dp), ("ph_sigma_hat", _dp), ("ph_relres", _dp), ("ph_t_lsqr_ms", _dp),
                ("ph_t_total_ms", _dp), ("n_ph", _i64), ("cap_ph", _i64),
                ("tr_phase", C.POINTER(_i32)), ("tr_iter", _i64p), ("tr_phibar", _dp),
                ("tr_matvecs", C.POINTER(_u64)), ("tr_relres", _dp), ("n_tr", _i64), ("cap_tr", _i64),
                ("wall_ms", C.c_double)]


def build() -> Optional[Path]:
    """Compile oracle/_ref from /root/reference when present (this container)."""
    if REF_INC.exists():
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB if LIB.exists() else None


_lib = None


def available() -> bool:
    return LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise FileNotFoundError(f"{LIB} missing: build it with `make -C oracle` where /root/reference exists")
        L = C.CDLL(str(LIB))
        vp = C.c_void_p
        P = C.POINTER(RefProblem)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng.argtypes = [_u64, _i32, _u64, _i32, _u64, _i64, vp]
        L.ref_mix64.restype = _u64
        L.ref_mix64.argtypes = [_u64]
        L.ref_matvec.argtypes = [P, C.c_double, _i32, _i32, _dp, _dp]
        L.ref_sparse_sign.argtypes = [_i64, _i64, _i64, _u64, _i64p, C.POINTER(C.c_int8), _dp]
        L.ref_sketch_sparse_sign.argtypes = [P, C.c_double, _i32, _i64, _i64, _u64, _dp]
        L.ref_gaussian_embedding.argtypes = [_i64, _i64, _u64, _dp]
        L.ref_sketch_gaussian.argtypes = [P, _i64, _u64, _dp]
        L.ref_lupp.argtypes = [_dp, _i64, _i64, _i64, _i64p, _dp, _i64p]
        L.ref_spectral_norm_estimate.argtypes = [_dp, _i64, _i64, _i64, _u64, _dp]
        L.ref_solve.argtypes = [P, _dp, C.POINTER(RefConfig), _i32, C.POINTER(RefOut)]
        L.ref_cur_steps.argtypes = [P, _i64, _u64, _i64, _i64, _i32, _i32, _i64, _dp, _i64p, _i64p,
                                    _i64p, _dp, _i64p, _dp]
        L.ref_time_op_pair.argtypes = [P, _i64, _dp]
        L.ref_generate.argtypes = [_i32, _i64, _i64, _u64, _i32, C.POINTER(C.c_void_p)]
        L.ref_gen_view.argtypes = [C.c_void_p, P, C.POINTER(_dp)]
        L.ref_gen_free.argtypes = [C.c_void_p]
        L.ref_gen_free.restype = None
        L.ref_solve_gen.argtypes = [C.c_void_p, _dp, C.POINTER(RefConfig), _i32, _i32, C.POINTER(RefOut)]
        L.ref_mm_write.argtypes = [P, C.c_char_p]
        L.ref_mm_read.argtypes = [C.c_char_p, _i64p, _i64p, C.POINTER(_i32), _i64p, _i64p, _i64p, _dp, _dp]
        _lib = L
    return _lib


def _chk(code: int):
    if code != 0:
        raise RuntimeError(f"reference error {code}: {lib().ref_last_error().decode()}")


class Problem:
    """Holds numpy buffers alive for a RefProblem view."""

    def __init__(self, m, n, dense=None, colptr=None, rowidx=None, vals=None):
        self.m, self.n = int(m), int(n)
        self.sparse = dense is None
        if self.sparse:
            self.colptr = np.ascontiguousarray(colptr, dtype=np.int64)
            self.rowidx = np.ascontiguousarray(rowidx, dtype=np.int64)
            self.vals = np.ascontiguousarray(vals, dtype=np.float64)
            self.c = RefProblem(self.m, self.n, 1, None, self.colptr.ctypes.data_as(_i64p),
                                self.rowidx.ctypes.data_as(_i64p), self.vals.ctypes.data_as(_dp))
        else:
            self.dense = np.ascontiguousarray(dense, dtype=np.float64).reshape(-1)
            self.c = RefProblem(self.m, self.n, 0, self.dense.ctypes.data_as(_dp), None, None, None)

    @classmethod
    def generate(cls, config: int, m: int = 0, n: int = 0, seed: int = 0, threads: int = 0) -> "Problem":
        """BASELINE input from the oracle's own generator (ref_harness.cpp
        ref_generate): arrays are views of memory the reference owns, so the
        process never maps the product library."""
        import os

        h = C.c_void_p()
        _chk(lib().ref_generate(config, m, n, seed, threads or os.cpu_count() or 1, C.byref(h)))
        view, bp = RefProblem(), _dp()
        _chk(lib().ref_gen_view(h, C.byref(view), C.byref(bp)))
        self = cls.__new__(cls)
        self.m, self.n, self.sparse, self.c, self._gen = view.m, view.n, bool(view.sparse), view, h
        self.config = config
        self.b = np.ctypeslib.as_array(bp, shape=(self.m,))
        if self.sparse:
            nnz = int(view.colptr[self.n])
            self.nnz = nnz
            self.colptr = np.ctypeslib.as_array(view.colptr, shape=(self.n + 1,))
            self.rowidx = np.ctypeslib.as_array(view.rowidx, shape=(nnz,))
            self.vals = np.ctypeslib.as_array(view.vals, shape=(nnz,))
        else:
            self.nnz = self.m * self.n
            self.dense = np.ctypeslib.as_array(view.dense, shape=(self.m * self.n,))
        return self

    def free(self) -> None:
        """Release a generated input (the numpy views die with it)."""
        h = getattr(self, "_gen", None)
        if h is not None:
            self._gen = None
            for k in ("b", "colptr", "rowidx", "vals", "dense"):
                self.__dict__.pop(k, None)
            lib().ref_gen_free(h)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @classmethod
    def from_apc(cls, p) -> "Problem":
        if p.sparse:
            return cls(p.m, p.n, colptr=p.colptr, rowidx=p.rowidx, vals=p.vals)
        return cls(p.m, p.n, dense=p.dense)

    @classmethod
    def from_numpy(cls, A: np.ndarray, sparse: bool = False) -> "Problem":
        m, n = A.shape
        if not sparse:
            return cls(m, n, dense=np.asfortranarray(A).reshape(-1, order="F"))
        colptr = [0]
        rows, vals = [], []
        for j in range(n):
            nz = np.nonzero(A[:, j])[0]
            rows.extend(nz.tolist())
            vals.extend(A[nz, j].tolist())
            colptr.append(len(rows))
        return cls(m, n, colptr=colptr, rowidx=rows, vals=vals)


def matvec(p: Problem, x, mu=0.0, augmented=False, transpose=False) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(p.n if transpose else p.m + (p.n if augmented else 0))
    _chk(lib().ref_matvec(C.byref(p.c), mu, int(augmented), int(transpose), x.ctypes.data_as(_dp),
                          out.ctypes.data_as(_dp)))
    return out


def rng(seed, kind, count, stream=-1, index=0, bound=0) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64 if kind in (0, 3) else np.float64)
    _chk(lib().ref_rng(seed, stream, index, kind, bound, count, out.ctypes.data_as(C.c_void_p)))
    return out


def mix64(x: int) -> int:
    return int(lib().ref_mix64(x))


def sparse_sign(s, m, xi, seed):
    x = min(xi, s)
    rows = np.empty(m * x, dtype=np.int64)
    signs = np.empty(m * x, dtype=np.int8)
    scale = C.c_double()
    _chk(lib().ref_sparse_sign(s, m, xi, seed, rows.ctypes.data_as(_i64p),
                               signs.ctypes.data_as(C.POINTER(C.c_int8)), C.byref(scale)))
    return rows, signs, scale.value


def sketch_sparse_sign(p: Problem, s, xi, emb_seed, mu=0.0, augmented=False) -> np.ndarray:
    y = np.empty(s * p.n)
    _chk(lib().ref_sketch_sparse_sign(C.byref(p.c), mu, int(augmented), s, xi, emb_seed, y.ctypes.data_as(_dp)))
    return y.reshape(p.n, s).T


def gaussian_embedding(s, m, emb_seed) -> np.ndarray:
    S = np.empty(s * m)
    _chk(lib().ref_gaussian_embedding(s, m, emb_seed, S.ctypes.data_as(_dp)))
    return S.reshape(m, s).T


def sketch_gaussian(p: Problem, s, emb_seed) -> np.ndarray:
    y = np.empty(s * p.n)
    _chk(lib().ref_sketch_gaussian(C.byref(p.c), s, emb_seed, y.ctypes.data_as(_dp)))
    return y.reshape(p.n, s).T


def lupp(W: np.ndarray, max_pivots=-1):
    rows, cols = W.shape
    w = np.asfortranarray(W, dtype=np.float64).reshape(-1, order="F")
    k = min(rows, cols) if max_pivots < 0 else min(rows, cols, max_pivots)
    order = np.empty(max(k, 1), dtype=np.int64)
    mags = np.empty(max(k, 1))
    ns = _i64()
    _chk(lib().ref_lupp(w.ctypes.data_as(_dp), rows, cols, max_pivots, order.ctypes.data_as(_i64p),
                        mags.ctypes.data_as(_dp), C.byref(ns)))
    return order[: ns.value], mags[: ns.value]


def spectral_norm_estimate(E: np.ndarray, r: int, seed: int) -> float:
    e = np.asfortranarray(E, dtype=np.float64).reshape(-1, order="F")
    out = C.c_double()
    _chk(lib().ref_spectral_norm_estimate(e.ctypes.data_as(_dp), E.shape[0], E.shape[1], r, seed, C.byref(out)))
    return out.value


@dataclasses.dataclass
class RefResult:
    x: np.ndarray
    status: int
    final_rho: float
    final_relres: float
    sketch_applications: int
    system_matvecs: int
    row_indices: np.ndarray
    col_indices: np.ndarray
    rho_history: np.ndarray
    phase_rank: np.ndarray
    phase_iters: np.ndarray
    phase_reason: np.ndarray
    phase_rho: np.ndarray
    phase_sigma_hat: np.ndarray
    phase_relres: np.ndarray
    phase_t_lsqr_ms: np.ndarray
    phase_t_total_ms: np.ndarray
    trace_phase: np.ndarray
    trace_iter: np.ndarray
    trace_phibar: np.ndarray
    trace_matvecs: np.ndarray
    trace_true_relres: np.ndarray
    wall_ms: float


def solve(p: Problem, b, cfg: dict, plain=False, cap_idx=20000, cap_rho=4096, cap_ph=4096,
          cap_tr=2_000_000, consume=False) -> RefResult:
    """Reference aplicur_solve (or plain_lsqr_solve).  For a Problem made by
    Problem.generate, b may be None (the generated b) and consume=True moves A
    into the solve (no second copy of a 20 GB matrix); the Problem is then
    spent."""
    c = RefConfig(block=0, eps_cur=-1.0, eps_lsqr=1e-10, nu_prec=10.0, nu_lsqr=100.0, mu=0.0, variant=0,
                  sketch_xi=8, probe_count=10, lsqr_cap=0, max_rank=0, seed=0, core=0,
                  trace_sample_stride=0, outer_cap=100000)
    for k, v in cfg.items():
        setattr(c, k, int(v) if isinstance(v, (bool, np.integer)) else v)
    gen = getattr(p, "_gen", None)
    if b is not None:
        b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(p.n)
    bufs = dict(
        row_idx=np.zeros(cap_idx, np.int64), col_idx=np.zeros(cap_idx, np.int64), rho_hist=np.zeros(cap_rho),
        ph_rank=np.zeros(cap_ph, np.int64), ph_iters=np.zeros(cap_ph, np.int64), ph_reason=np.zeros(cap_ph, np.int32),
        ph_rho=np.zeros(cap_ph), ph_sigma_hat=np.zeros(cap_ph), ph_relres=np.zeros(cap_ph),
        ph_t_lsqr_ms=np.zeros(cap_ph), ph_t_total_ms=np.zeros(cap_ph),
        tr_phase=np.zeros(cap_tr, np.int32), tr_iter=np.zeros(cap_tr, np.int64), tr_phibar=np.zeros(cap_tr),
        tr_matvecs=np.zeros(cap_tr, np.uint64), tr_relres=np.zeros(cap_tr))
    o = RefOut()
    o.x = x.ctypes.data_as(_dp)
    ftypes = dict(RefOut._fields_)
    for k, arr in bufs.items():
        setattr(o, k, arr.ctypes.data_as(ftypes[k]))
    o.cap_idx, o.cap_rho, o.cap_ph, o.cap_tr = cap_idx, cap_rho, cap_ph, cap_tr
    if gen is not None:
        if consume:
            for k in ("colptr", "rowidx", "vals", "dense"):
                p.__dict__.pop(k, None)
        _chk(lib().ref_solve_gen(gen, None if b is None else b.ctypes.data_as(_dp), C.byref(c), int(plain),
                                 int(consume), C.byref(o)))
    else:
        _chk(lib().ref_solve(C.byref(p.c), b.ctypes.data_as(_dp), C.byref(c), int(plain), C.byref(o)))
    ni, nr, nph, ntr = o.n_idx, o.n_rho, o.n_ph, min(o.n_tr, cap_tr)
    return RefResult(x, o.status, o.final_rho, o.final_relres, o.sketch_applications, o.system_matvecs,
                     bufs["row_idx"][:ni].copy(), bufs["col_idx"][:ni].copy(), bufs["rho_hist"][:nr].copy(),
                     bufs["ph_rank"][:nph].copy(), bufs["ph_iters"][:nph].copy(), bufs["ph_reason"][:nph].copy(),
                     bufs["ph_rho"][:nph].copy(), bufs["ph_sigma_hat"][:nph].copy(), bufs["ph_relres"][:nph].copy(),
                     bufs["ph_t_lsqr_ms"][:nph].copy(), bufs["ph_t_total_ms"][:nph].copy(),
                     bufs["tr_phase"][:ntr].copy(), bufs["tr_iter"][:ntr].copy(), bufs["tr_phibar"][:ntr].copy(),
                     bufs["tr_matvecs"][:ntr].copy(), bufs["tr_relres"][:ntr].copy(), o.wall_ms)


def cur_steps(p: Problem, block, seed, steps, xi=8, probes=10, core=0, gaussian=False):
    """Reference CurState init/augment/refresh sequence (cur.hpp:209-315)."""
    s = int(np.ceil(1.1 * block))
    y = np.empty(s * p.n)
    eres = np.empty(s * p.n)
    added = np.zeros(steps, np.int64)
    cap = min(p.m, p.n) + block
    ii = np.zeros(cap, np.int64)
    jj = np.zeros(cap, np.int64)
    rho = np.zeros(steps)
    nd = _i64()
    _chk(lib().ref_cur_steps(C.byref(p.c), block, seed, xi, probes, core, int(gaussian), steps,
                             y.ctypes.data_as(_dp), added.ctypes.data_as(_i64p), ii.ctypes.data_as(_i64p),
                             jj.ctypes.data_as(_i64p), rho.ctypes.data_as(_dp), C.byref(nd),
                             eres.ctypes.data_as(_dp)))
    k = nd.value
    rank = int(sum(a for a in added[:k] if a > 0))
    return dict(Y=y.reshape(p.n, s).T, eres=eres.reshape(p.n, s).T, added=added[:k], I=ii[:rank],
                J=jj[:rank], rho=rho[:k])


def time_op_pair(p: Problem, iters: int) -> float:
    out = C.c_double()
    _chk(lib().ref_time_op_pair(C.byref(p.c), iters, C.byref(out)))
    return out.value


def mm_write(p: "Problem", path) -> None:
    """Reference write_matrix_market (matrix_market.hpp:18-46)."""
    _chk(lib().ref_mm_write(C.byref(p.c), str(path).encode()))


def mm_read(path) -> dict:
    """Reference read_matrix_market (matrix_market.hpp:48-116): CSC or dense arrays."""
    m, n, nz, sp = _i64(), _i64(), _i64(), _i32()
    _chk(lib().ref_mm_read(str(path).encode(), C.byref(m), C.byref(n), C.byref(sp), C.byref(nz), None, None, None,
                           None))
    out = dict(m=m.value, n=n.value, sparse=bool(sp.value))
    if sp.value:
        cp = np.zeros(n.value + 1, dtype=np.int64)
        ri = np.zeros(nz.value, dtype=np.int64)
        va = np.zeros(nz.value)
        _chk(lib().ref_mm_read(str(path).encode(), C.byref(m), C.byref(n), C.byref(sp), C.byref(nz),
                               cp.ctypes.data_as(_i64p), ri.ctypes.data_as(_i64p), va.ctypes.data_as(_dp), None))
        out.update(colptr=cp, rowidx=ri, vals=va)
    else:
        d = np.zeros(m.value * n.value)
        _chk(lib().ref_mm_read(str(path).encode(), C.byref(m), C.byref(n), C.byref(sp), C.byref(nz), None, None, None,
                               d.ctypes.data_as(_dp)))
        out.update(dense=d)
    return out
