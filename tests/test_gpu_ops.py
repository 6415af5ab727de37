"""GPU parity of the operator products A*x, A^T*u, [A; mu I]*x, [A; mu I]^T*u
against the reference Matrix / AugmentedOperator (matrix.hpp:151-195, 365-392).

The device sums in a different (fixed) order than the reference's sequential
loops, so the gate is the componentwise summation-error bound
|y_gpu - y_ref|_i <= 2 k 2^-53 (|A| |x|)_i (k = inner length), plus
bit-identical reruns and the adjoint identity (test_matrix.cpp:123-136)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -53


def _bound(Aabs, xabs, k):
    return 2.0 * k * EPS * (Aabs @ xabs) + 1e-300


def _check(y, yref, bound):
    err = np.abs(y - yref)
    assert np.all(err <= bound), float(np.max(err / bound))


CASES = [
    ("dense", 1, 400, 50), ("dense", 1, 4000, 500), ("dense", 3, 3000, 700), ("dense", 4, 2000, 1999),
    ("sparse", 2, 20000, 2000), ("sparse", 2, 200000, 20000), ("sparse", 5, 200000, 20000),
]


@pytest.mark.parametrize("kind,cfg,m,n", CASES)
@pytest.mark.parametrize("mu", [0.0, 0.37])
def test_operator_products_vs_reference(apc, ref, ctx, kind, cfg, m, n, mu):
    p = apc.Problem(cfg, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    rp = ref.Problem.from_apc(p)
    rng = np.random.default_rng(m + n)
    x = rng.standard_normal(n)
    u = rng.standard_normal(m + n)
    aug = mu > 0
    Aabs = None
    if m * n <= 4e7:
        Aabs = np.abs(p.to_numpy())
    y = A.apply(x, mu, aug, False)
    yr = ref.matvec(rp, x, mu, aug, False)
    uu = u if aug else u[:m]
    g = A.apply(uu, mu, aug, True)
    gr = ref.matvec(rp, uu, mu, aug, True)
    if Aabs is not None:
        kf = (Aabs != 0).sum(axis=1).max() if p.sparse else n
        kt = (Aabs != 0).sum(axis=0).max() if p.sparse else m
        _check(y[:m], yr[:m], _bound(Aabs, np.abs(x), kf))
        _check(g, gr, _bound(Aabs.T, np.abs(uu[:m]), kt + 1) + (2 * EPS * mu * np.abs(uu[m:]) if aug else 0))
    else:
        assert np.allclose(y, yr, rtol=1e-10, atol=1e-12 * np.abs(yr).max())
        assert np.allclose(g, gr, rtol=1e-10, atol=1e-12 * np.abs(gr).max())
    if aug:
        assert np.array_equal(y[m:], mu * x)  # tail rows are exact
    # bit-identical reruns (fixed reduction order)
    assert np.array_equal(A.apply(x, mu, aug, False), y)
    assert np.array_equal(A.apply(uu, mu, aug, True), g)
    # adjoint identity <A_mu x, u> = <x, A_mu^T u>
    lhs, rhs = float(y @ uu), float(x @ g)
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs), 1.0)


def test_empty_and_degenerate_shapes(apc, ref, ctx):
    # zero columns present, a fully empty row, 1 x 1
    colptr = np.array([0, 2, 2, 3], dtype=np.int64)
    rowidx = np.array([0, 2, 2], dtype=np.int64)
    vals = np.array([1.5, -2.0, 4.0])
    A = apc.DeviceMatrix.csc(ctx, 4, 3, colptr, rowidx, vals)
    x = np.array([1.0, 2.0, 3.0])
    assert np.array_equal(A.apply(x), np.array([1.5, 0.0, 10.0, 0.0]))
    assert np.array_equal(A.apply(np.array([1.0, 1.0, 1.0, 1.0]), transpose=True), np.array([-0.5, 0.0, 4.0]))
    B = apc.DeviceMatrix.dense(ctx, np.array([3.0]), 1, 1)
    assert B.apply(np.array([2.0]))[0] == 6.0
    with pytest.raises(apc.ApcError):
        apc.DeviceMatrix.csc(ctx, 2, 1, np.array([0, 2]), np.array([1, 0]), np.array([1.0, 2.0]))


def test_long_rows_split_units(apc, ref, ctx):
    # one column with far more nonzeros than a work unit (fix-up path)
    m, n = 300000, 3
    rows = np.arange(0, m, 2, dtype=np.int64)
    colptr = np.array([0, rows.size, rows.size + 1, rows.size + 2], dtype=np.int64)
    rowidx = np.concatenate([rows, [5, 7]]).astype(np.int64)
    vals = np.concatenate([np.linspace(-1, 1, rows.size), [2.0, 3.0]])
    A = apc.DeviceMatrix.csc(ctx, m, n, colptr, rowidx, vals)
    rp = ref.Problem(m, n, colptr=colptr, rowidx=rowidx, vals=vals)
    u = np.random.default_rng(1).standard_normal(m)
    g = A.apply(u, transpose=True)
    gr = ref.matvec(rp, u, transpose=True)
    assert np.allclose(g, gr, rtol=1e-12, atol=1e-12)
