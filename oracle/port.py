"""ORACLE / TEST INFRASTRUCTURE ONLY -- a plain-Python restatement of the APLICUR
reference arithmetic on the hot path, pinned bit-for-bit against the golden
vectors produced by the unmodified reference (tests/golden/, oracle/make_golden.py).

Only tests/ (and smoke()/bench cpu_baseline) may import this module; the
product path never does.  Pure-Python loops: small cases only.  Every routine
keeps the reference's operation order (IEEE doubles, no FMA), so results are
bit-identical, not merely close.  Each function cites the reference it restates.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

_M64 = (1 << 64) - 1
_libm = ctypes.CDLL("libm.so.6")
_libm.hypot.restype = ctypes.c_double
_libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
_libm.log.restype = ctypes.c_double
_libm.log.argtypes = [ctypes.c_double]
_libm.cos.restype = ctypes.c_double
_libm.cos.argtypes = [ctypes.c_double]


# ---------------------------------------------------------------------------
# rng.hpp:12-78
# ---------------------------------------------------------------------------
def mix64(x: int) -> int:
    """splitmix64 (rng.hpp:15-20)."""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


class MT19937_64:
    """std::mt19937_64 (the C++ standard's parameters)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _M64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _M64
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


class Rng:
    """Rng (rng.hpp:38-78)."""

    def __init__(self, seed: int, stream: int | None = None, index: int = 0):
        if stream is None:
            self.g = MT19937_64(mix64(seed))
        else:
            s = mix64((mix64(seed ^ ((0x51ED2701A3C5E1BD * stream) & _M64)) + index) & _M64)
            self.g = MT19937_64(s)

    def next_u64(self) -> int:
        return self.g()

    def uniform(self) -> float:
        return float(self.g() >> 11) * 2.0 ** -53

    def gaussian(self) -> float:
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * _libm.log(u1)) * _libm.cos(6.283185307179586476925286766559 * u2)

    def below(self, n: int) -> int:
        limit = _M64 - (_M64 % n)
        while True:
            x = self.g()
            if x < limit:
                return x % n

    def sign(self) -> float:
        return 1.0 if (self.g() & 1) else -1.0


# ---------------------------------------------------------------------------
# sketch.hpp:18-111, 209-223
# ---------------------------------------------------------------------------
def sparse_sign(s: int, m: int, xi: int, seed: int):
    """SparseSignEmbedding ctor (sketch.hpp:20-50): Floyd sampling, sorted rows, signs."""
    x = min(xi, s)
    rng = Rng(seed)
    rows = np.zeros(m * x, np.int64)
    signs = np.zeros(m * x, np.int8)
    for c in range(m):
        pick = []
        for t in range(s - x, s):
            r = rng.below(t + 1)
            pick.append(t if r in pick else r)
        pick.sort()
        for q in range(x):
            rows[c * x + q] = pick[q]
            signs[c * x + q] = 1 if rng.sign() > 0 else -1
    return rows, signs, 1.0 / math.sqrt(float(x))


def sketch_dense(A: np.ndarray, s: int, rows, signs, scale: float) -> np.ndarray:
    """SparseSignEmbedding::apply, dense A (sketch.hpp:81-93)."""
    m, n = A.shape
    x = len(rows) // m
    Y = np.zeros((s, n))
    for j in range(n):
        y = [0.0] * s
        for k in range(m):
            v = float(A[k, j])
            if v == 0.0:
                continue
            sv = scale * v
            for q in range(x):
                y[rows[k * x + q]] += sv * float(signs[k * x + q])
        Y[:, j] = y
    return Y


def sketch_augmented_dense(A: np.ndarray, mu: float, s: int, rows, signs, scale: float) -> np.ndarray:
    """apply_to_augmented (sketch.hpp:115-162): top block, then mu * scale * sign tail."""
    m, n = A.shape
    x = len(rows) // (m + n)
    Y = sketch_dense(A, s, rows[: m * x], signs[: m * x], scale)
    if mu != 0.0:
        for j in range(n):
            c = m + j
            for q in range(x):
                Y[rows[c * x + q], j] += mu * scale * float(signs[c * x + q])
    return Y


def spectral_norm_estimate(E: np.ndarray, r: int, rng: Rng) -> float:
    """sketch.hpp:209-223 (unnormalised Gaussian probes, dense matvec chains)."""
    s, n = E.shape
    best = 0.0
    for _ in range(r):
        w = [rng.gaussian() for _ in range(n)]
        ew = matvec_dense(E, w)
        nrm2 = 0.0
        for v in ew:
            nrm2 += v * v
        best = max(best, math.sqrt(nrm2))
    return 10.0 * math.sqrt(2.0 / 3.14159265358979323846) * best


# ---------------------------------------------------------------------------
# matrix.hpp:151-195, 365-392
# ---------------------------------------------------------------------------
def matvec_dense(A: np.ndarray, x) -> list:
    """Matrix::matvec dense (matrix.hpp:156-162): column axpy, skipping x_j == 0."""
    m, n = A.shape
    y = [0.0] * m
    for j in range(n):
        xj = float(x[j])
        if xj == 0.0:
            continue
        col = A[:, j]
        for i in range(m):
            y[i] += xj * float(col[i])
    return y


def matvec_t_dense(A: np.ndarray, x) -> list:
    """Matrix::matvec_transpose dense (matrix.hpp:179-185): per-column dots."""
    m, n = A.shape
    out = []
    for j in range(n):
        s = 0.0
        col = A[:, j]
        for i in range(m):
            s += float(col[i]) * float(x[i])
        out.append(s)
    return out


def matvec_csc(m, colptr, rowidx, vals, x) -> list:
    """Matrix::matvec CSC scatter (matrix.hpp:163-171)."""
    y = [0.0] * m
    for j in range(len(colptr) - 1):
        xj = float(x[j])
        if xj == 0.0:
            continue
        for k in range(colptr[j], colptr[j + 1]):
            y[rowidx[k]] += xj * float(vals[k])
    return y


def matvec_t_csc(colptr, rowidx, vals, x) -> list:
    """Matrix::matvec_transpose CSC gather (matrix.hpp:186-193)."""
    out = []
    for j in range(len(colptr) - 1):
        s = 0.0
        for k in range(colptr[j], colptr[j + 1]):
            s += float(vals[k]) * float(x[rowidx[k]])
        out.append(s)
    return out


# ---------------------------------------------------------------------------
# dense_factor.hpp:119-157
# ---------------------------------------------------------------------------
def lu_partial_pivot(W: np.ndarray, max_pivots: int = -1):
    """Right-looking partial-pivot order; ties -> lowest original row; no FMA."""
    m, n = W.shape
    steps = min(m, n) if max_pivots < 0 else min(m, n, max_pivots)
    w = [[float(W[i, j]) for j in range(n)] for i in range(m)]
    perm = list(range(m))
    order, mags = [], []
    for k in range(steps):
        best, best_mag, best_orig = k, -1.0, 1 << 62
        for i in range(k, m):
            mag = abs(w[perm[i]][k])
            if mag > best_mag or (mag == best_mag and perm[i] < best_orig):
                best, best_mag, best_orig = i, mag, perm[i]
        perm[k], perm[best] = perm[best], perm[k]
        prow = perm[k]
        order.append(prow)
        mags.append(best_mag)
        pval = w[prow][k]
        if pval == 0.0:
            continue
        for i in range(k + 1, m):
            r = perm[i]
            f = w[r][k] / pval
            if f == 0.0:
                continue
            for j in range(k, n):
                w[r][j] -= f * w[prow][j]
    return np.array(order, np.int64), np.array(mags)


# ---------------------------------------------------------------------------
# lsqr.hpp:84-207 (plain operator, observer-free)
# ---------------------------------------------------------------------------
def lsqr(fwd, adj, m: int, n: int, rhs, eps: float, cap: int, nu: float = math.inf, floor: float = 0.0):
    """lsqr_solve: returns (y, phibar trace, reason, matvec counts)."""

    def norm2(v):
        s = 0.0
        for x in v:
            s += x * x
        return math.sqrt(s)

    u = [float(x) for x in rhs]
    beta = norm2(u)
    trace = [beta]
    y = [0.0] * n
    if beta == 0.0:
        return y, trace, 5
    u = [x / beta for x in u]
    v = adj(u)
    alpha = norm2(v)
    if alpha == 0.0:
        return y, trace, 1
    v = [x / alpha for x in v]
    w = list(v)
    phibar, rhobar, opnorm2, cvgrate1 = beta, alpha, alpha * alpha, 0.0
    for j in range(1, cap + 1):
        t = fwd(v)
        t = [t[i] - alpha * u[i] for i in range(m)]
        u = t
        beta = norm2(u)
        if beta > 0.0:
            u = [x / beta for x in u]
        t = adj(u)
        t = [t[i] - beta * v[i] for i in range(n)]
        v = t
        alpha = norm2(v)
        if alpha > 0.0:
            v = [x / alpha for x in v]
        opnorm2 += alpha * alpha + beta * beta
        rho = _libm.hypot(rhobar, beta)
        c, s = rhobar / rho, beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar_prev = phibar
        phibar = s * phibar
        t1, t2 = phi / rho, -theta / rho
        for i in range(n):
            y[i] += t1 * w[i]
            w[i] = v[i] + t2 * w[i]
        cvgrate = _libm.log(phibar_prev / phibar) if (phibar > 0.0 and phibar_prev > 0.0) else math.inf
        cvgdiff = phibar_prev - phibar
        if j == 1:
            cvgrate1 = cvgrate
        trace.append(phibar)
        grad = phibar * alpha * abs(c)
        ynorm = norm2(y)
        if grad <= eps * math.sqrt(opnorm2) * phibar or phibar <= eps * (math.sqrt(opnorm2) * ynorm + trace[0]) \
                or phibar == 0.0:
            return y, trace, 1
        if j >= 2 and not math.isinf(nu):
            if floor > 0.0 and cvgdiff < floor:
                return y, trace, 3
            if cvgrate <= 0.0 or cvgrate1 / cvgrate > nu:
                return y, trace, 2
    return y, trace, 4


def plain_lsqr_csc(m, n, colptr, rowidx, vals, b, mu, eps, cap):
    """plain_lsqr_solve (solver.hpp:396-448) on [A; mu I] (mu > 0) or A."""
    if mu > 0.0:
        fwd = lambda x: matvec_csc(m, colptr, rowidx, vals, x) + [mu * xi for xi in x]  # noqa: E731

        def adj(u):
            g = matvec_t_csc(colptr, rowidx, vals, u[:m])
            return [g[i] + mu * u[m + i] for i in range(n)]

        rhs = list(b) + [0.0] * n
        return lsqr(fwd, adj, m + n, n, rhs, eps, cap)
    return lsqr(lambda x: matvec_csc(m, colptr, rowidx, vals, x), lambda u: matvec_t_csc(colptr, rowidx, vals, u),
                m, n, list(b), eps, cap)
