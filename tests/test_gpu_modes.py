"""The LSQR driver's execution modes agree: persistent cooperative kernel
(default for L2-resident sparse systems), CUDA graph with a conditional WHILE
node, host-polled graph batches (the multi-rank path, here without NCCL),
eager launches; and the sharded entry point (apc_solve_sharded) on one rank."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KNOBS = dict(mu=1e-3, eps_lsqr=1e-10, block=8, seed=3, max_rank=40, trace_sample_stride=0)


@pytest.fixture
def problem(apc, ctx):
    p = apc.Problem(2, 4000, 400)
    return p, apc.DeviceMatrix.from_problem(ctx, p)


@pytest.mark.parametrize("mode", ["while", "batch", "eager"])
def test_modes_agree_with_persistent(apc, problem, mode):
    p, A = problem
    base = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
    os.environ["APC_LSQR_MODE"] = mode
    try:
        other = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
    finally:
        del os.environ["APC_LSQR_MODE"]
    assert np.array_equal(base.row_indices, other.row_indices)
    assert abs(base.lsqr_iters - other.lsqr_iters) <= max(3, 0.05 * base.lsqr_iters)
    assert abs(base.final_relres - other.final_relres) <= 1e-3 * base.final_relres


def test_sharded_entry_single_rank(apc, ctx, problem):
    p, A = problem
    full = apc.DeviceMatrix.from_problem(ctx, p)
    g1 = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
    g2 = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS), full=full)
    assert np.array_equal(g1.row_indices, g2.row_indices)
    assert np.array_equal(g1.x, g2.x)


def test_row_shard_operator_products(apc, ref, ctx, problem):
    # a shard's A*x is the corresponding block of rows; its A^T u is the partial sum
    p, A = problem
    r0, r1 = 1000, 2500
    S = apc.DeviceMatrix.from_problem(ctx, p, r0, r1)
    x = np.random.default_rng(0).standard_normal(p.n)
    np.testing.assert_allclose(S.apply(x), A.apply(x)[r0:r1], rtol=1e-12, atol=1e-14)
    u = np.random.default_rng(1).standard_normal(r1 - r0)
    full_u = np.zeros(p.m)
    full_u[r0:r1] = u
    np.testing.assert_allclose(S.apply(u, transpose=True), A.apply(full_u, transpose=True), rtol=1e-11,
                               atol=1e-13)
