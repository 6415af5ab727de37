"""The preconditioner construction's dense kernels (csrc/blas.cu, no cuBLAS):
DMMA GEMM with either operand transposed and the fixed-order split over k
(the tall-skinny Q^T E and E^T E of QrAccumulator::append,
preconditioner.hpp:435-476), and the blocked right upper-triangular solve
(E <- E R^{-1}), against numpy in float64 (rounding-level tolerance; the
products are deterministic run to run)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.asfortranarray(a).reshape(-1, order="F").copy()).cuda()


@pytest.mark.parametrize("ta,tb,m,n,k", [(False, False, 1000, 250, 1000), (True, False, 300, 120, 50000),
                                         (True, False, 7, 5, 3), (False, True, 97, 65, 33),
                                         (True, True, 130, 70, 900), (False, False, 50000, 250, 300)])
def test_dgemm_matches_numpy(apc, ctx, ta, tb, m, n, k):
    import ctypes as C

    rng = np.random.default_rng(m + n + k)
    A = rng.standard_normal((k, m) if ta else (m, k))
    B = rng.standard_normal((n, k) if tb else (k, n))
    C0 = rng.standard_normal((m, n))
    dA, dB, dC = _dev(A), _dev(B), _dev(C0)
    torch.cuda.synchronize()
    lib = apc.load_library()
    assert lib.apc_dgemm(ctx.h, int(ta), int(tb), m, n, k, 0.5, C.c_void_p(dA.data_ptr()), A.shape[0],
                         C.c_void_p(dB.data_ptr()), B.shape[0], -2.0, C.c_void_p(dC.data_ptr()), m) == 0
    got = dC.cpu().numpy().reshape(n, m).T
    want = 0.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 2.0 * C0
    scale = 0.5 * (np.abs(A.T if ta else A) @ np.abs(B.T if tb else B)) + 2.0 * np.abs(C0)
    assert np.max(np.abs(got - want) / scale) <= 4 * k * 2.0 ** -53
    # deterministic rerun
    dC2 = _dev(C0)
    lib.apc_dgemm(ctx.h, int(ta), int(tb), m, n, k, 0.5, C.c_void_p(dA.data_ptr()), A.shape[0],
                  C.c_void_p(dB.data_ptr()), B.shape[0], -2.0, C.c_void_p(dC2.data_ptr()), m)
    assert torch.equal(dC, dC2)


@pytest.mark.parametrize("m,n", [(5000, 250), (300, 33), (70000, 100), (10, 1)])
def test_dtrsm_right_upper(apc, ctx, m, n):
    import ctypes as C

    rng = np.random.default_rng(m + n)
    T = np.triu(rng.standard_normal((n, n))) + np.diag(np.full(n, 3.0 + n ** 0.5))
    B = rng.standard_normal((m, n))
    dT, dB = _dev(T), _dev(B)
    torch.cuda.synchronize()
    assert apc.load_library().apc_dtrsm_right_upper(ctx.h, m, n, C.c_void_p(dT.data_ptr()), n,
                                                     C.c_void_p(dB.data_ptr()), m) == 0
    X = dB.cpu().numpy().reshape(n, m).T
    assert np.allclose(X @ T, B, rtol=0, atol=1e-11 * np.abs(B).max())


@pytest.mark.parametrize("k", [1, 7, 64, 65, 250, 1000])
def test_dpotrf_upper_matches_numpy(apc, ctx, k):
    """Blocked device Cholesky (dense_small.cu) vs numpy: T upper, T^T T = G,
    lower part zeroed; a non-positive pivot is reported with its column."""
    import ctypes as C

    rng = np.random.default_rng(k)
    X = rng.standard_normal((2 * k + 3, k))
    G = X.T @ X
    d = _dev(G)
    bad = C.c_int64(7)
    lib = apc.load_library()
    assert lib.apc_dpotrf_upper(ctx.h, k, C.c_void_p(d.data_ptr()), C.byref(bad)) == 0
    assert bad.value == -1
    T = d.cpu().numpy().reshape(k, k).T
    assert np.all(np.tril(T, -1) == 0.0) and np.all(np.diag(T) > 0)
    want = np.linalg.cholesky(G).T
    assert np.max(np.abs(T - want)) <= 1e-10 * np.max(np.abs(want))
    if k >= 3:  # make column 2 dependent on columns 0, 1: pivot 2 is (numerically) not positive
        X[:, 2] = X[:, 0] - X[:, 1]
        G2 = X.T @ X
        G2[2, 2] -= 1e-3 * abs(G2[2, 2])
        d2 = _dev(G2)
        assert lib.apc_dpotrf_upper(ctx.h, k, C.c_void_p(d2.data_ptr()), C.byref(bad)) == 0
        assert bad.value == 2


@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("k,ncols", [(1, 3), (50, 50), (500, 37), (1000, 1000)])
def test_dtrsm_rows_matches_numpy(apc, ctx, k, ncols, transpose):
    """X <- T^{-1} X / T^{-T} X for every column (tri_solve, dense_factor.hpp:406-424)."""
    import ctypes as C

    rng = np.random.default_rng(k + ncols)
    T = np.triu(rng.standard_normal((k, k))) + 4.0 * np.eye(k)
    X = rng.standard_normal((k, ncols))
    dT = _dev(T)
    dX = torch.from_numpy(np.ascontiguousarray(X).reshape(-1).copy()).cuda()  # row-major k x ncols
    lib = apc.load_library()
    assert lib.apc_dtrsm_rows(ctx.h, k, C.c_void_p(dT.data_ptr()), C.c_void_p(dX.data_ptr()), ncols,
                              int(transpose)) == 0
    got = dX.cpu().numpy().reshape(k, ncols)
    M = T.T if transpose else T
    assert np.max(np.abs(M @ got - X)) <= 1e-10 * (np.abs(M) @ np.abs(got) + np.abs(X)).max()
    T[k // 2, k // 2] = 0.0
    dT = _dev(T)
    assert lib.apc_dtrsm_rows(ctx.h, k, C.c_void_p(dT.data_ptr()), C.c_void_p(dX.data_ptr()), ncols,
                              int(transpose)) == 4  # APC_SINGULAR
