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
