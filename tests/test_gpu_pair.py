"""The fused dense operator pair (dense_pair.cu: u = A z - alpha u/beta, ||u||^2
and A^T u with A read from HBM once) against the two-pass kernels, the numpy
product, and the reference solver when the LSQR loop runs on it.
Reference: Matrix::matvec / matvec_transpose (matrix.hpp:151-195) as
lsqr_solve calls them back to back (lsqr.hpp:139-150)."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture
def forced_pair():
    """APC_DENSE_PAIR=1: the fused path on every shape the kernel supports
    (by default only matrices of 64 MB or more take it); read once per matrix."""
    old = {k: os.environ.get(k) for k in ("APC_DENSE_PAIR", "APC_DP_RB", "APC_DP_GROUPS", "APC_DP_STAGES")}
    os.environ["APC_DENSE_PAIR"] = "1"
    yield os.environ
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _pair(ctx, A, x, m, n):
    dev = torch.device("cuda:0")
    xd = torch.from_numpy(x).to(dev)
    y = torch.zeros(m, dtype=torch.float64, device=dev)
    g = torch.zeros(n + 1, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    fused = A.pair_dev(xd.data_ptr(), y.data_ptr(), g.data_ptr())
    ctx.sync()
    return fused, y.cpu().numpy(), g.cpu().numpy()


SHAPES = [(5, 3), (50, 37), (64, 148), (400, 50), (4000, 500), (777, 9000), (10007, 4001), (2048, 20011)]


@pytest.mark.parametrize("m,n", SHAPES)
@pytest.mark.parametrize("knobs", [{}, {"APC_DP_GROUPS": "1"}, {"APC_DP_GROUPS": "2", "APC_DP_RB": "2"},
                                   {"APC_DP_STAGES": "3", "APC_DP_RB": "8"}])
def test_fused_pair_matches_numpy(apc, ctx, forced_pair, m, n, knobs):
    forced_pair.update(knobs)
    rng = np.random.default_rng(m * 131 + n)
    Ah = rng.standard_normal((m, n))
    x = rng.standard_normal(n)
    A = apc.DeviceMatrix.from_numpy(ctx, Ah)
    fused, y, g = _pair(ctx, A, x, m, n)
    assert fused, "the fused kernel did not run"
    yr = Ah @ x
    gr = Ah.T @ yr
    # componentwise bound of a length-n (resp. m) fp64 dot product in any order
    assert np.all(np.abs(y - yr) <= 4 * n * np.finfo(float).eps * (np.abs(Ah) @ np.abs(x)) + 1e-300)
    assert np.all(np.abs(g[:n] - gr) <= 8 * (m + n) * np.finfo(float).eps * (np.abs(Ah).T @ (np.abs(Ah) @ np.abs(x))))
    assert abs(g[n] - yr @ yr) <= 1e-13 * (yr @ yr)
    # reruns are bit-identical, and the counters re-arm between launches
    for _ in range(2):
        f2, y2, g2 = _pair(ctx, A, x, m, n)
        assert f2 and np.array_equal(y, y2) and np.array_equal(g, g2)
    A.free()


def test_small_matrices_keep_the_two_pass_kernels(apc, ctx):
    rng = np.random.default_rng(3)
    Ah = rng.standard_normal((300, 40))
    x = rng.standard_normal(40)
    A = apc.DeviceMatrix.from_numpy(ctx, Ah)
    fused, y, g = _pair(ctx, A, x, 300, 40)
    assert not fused
    assert np.array_equal(y, A.apply(x))
    assert np.allclose(g[:40], Ah.T @ (Ah @ x), rtol=1e-12, atol=1e-12)
    assert abs(g[40] - y @ y) <= 1e-13 * (y @ y)
    A.free()


def test_auto_rule_by_size_and_width(apc, ctx):
    """Without APC_DENSE_PAIR: 64 MB or more AND tiles of 16 KB or more take the
    fused kernel (10000 x 3000), a narrow matrix of the same bytes does not
    (30000 x 1000: its 7 KB tiles lose to the two streaming passes)."""
    assert "APC_DENSE_PAIR" not in os.environ
    rng = np.random.default_rng(11)
    for (m, n, want) in [(10000, 3000, True), (30000, 1000, False)]:
        Ah = rng.standard_normal((m, n))
        x = rng.standard_normal(n)
        A = apc.DeviceMatrix.from_numpy(ctx, Ah)
        fused, y, g = _pair(ctx, A, x, m, n)
        assert fused == want, (m, n, fused)
        yr = Ah @ x
        assert np.allclose(y, yr, rtol=0, atol=1e-11 * np.abs(yr).max())
        assert np.allclose(g[:n], Ah.T @ yr, rtol=0, atol=1e-11 * np.abs(Ah.T @ yr).max())
        A.free()


def test_sparse_matrix_runs_the_two_products(apc, ctx):
    p = apc.Problem(2, 4000, 400)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    x = np.random.default_rng(5).standard_normal(p.n)
    fused, y, g = _pair(ctx, A, x, p.m, p.n)
    assert not fused
    yr = A.apply(x)
    assert np.array_equal(y, yr)
    assert np.allclose(g[:p.n], A.apply(yr, transpose=True), rtol=1e-12, atol=1e-300)
    A.free()


@pytest.mark.parametrize("cfg,m,n,knobs", [
    (1, 4000, 500, dict(mu=0.0, eps_lsqr=1e-8, block=20, seed=1, max_rank=100)),
    (3, 3000, 300, dict(mu=1e-4, eps_lsqr=1e-8, block=10, seed=1, max_rank=60)),
    (1, 400, 50, dict(mu=0.05, eps_lsqr=1e-10, block=5, seed=1, variant=1)),
])
def test_solve_on_the_fused_pair_matches_reference(apc, ref, ctx, forced_pair, cfg, m, n, knobs):
    """The whole adaptive solve with every LSQR iteration on the fused kernel:
    indices bit-exact, iteration count within 5%, x within 1e-6 (the bars of
    test_gpu_solver.py)."""
    p = apc.Problem(cfg, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    L0 = ctx.launches
    g = apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs))
    fused_launches = ctx.launches - L0
    r = ref.solve(ref.Problem.from_apc(p), p.b, dict(knobs, trace_sample_stride=0))
    assert np.array_equal(g.row_indices, r.row_indices)
    assert np.array_equal(g.col_indices, r.col_indices)
    assert [ph.rank for ph in g.phases] == list(r.phase_rank)
    it_g, it_r = g.lsqr_iters, int(r.phase_iters.sum())
    assert abs(it_g - it_r) <= max(3, 0.05 * it_r), (it_g, it_r)
    assert g.phases[-1].reason == r.phase_reason[-1]
    rel = np.linalg.norm(g.x - r.x) / np.linalg.norm(r.x)
    bp = np.nextafter(p.b, np.inf)
    r2 = ref.solve(ref.Problem.from_apc(p), bp, dict(knobs, trace_sample_stride=0))
    self_sens = np.linalg.norm(r2.x - r.x) / np.linalg.norm(r.x)
    if r.phase_reason[-1] == apc.StopReason.gradient_tol:
        assert rel <= max(1e-6, 10.0 * self_sens), (rel, self_sens)
    else:
        assert g.final_relres <= r.final_relres * (1.0 + 1e-3)
    # and the path really was the fused one: the two-pass solve launches one
    # more kernel per iteration
    os.environ["APC_DENSE_PAIR"] = "0"
    A2 = apc.DeviceMatrix.from_problem(ctx, p)
    L1 = ctx.launches
    g2 = apc.aplicur_solve(A2, p.b, apc.SolverConfig(**knobs))
    two_pass_launches = ctx.launches - L1
    assert two_pass_launches >= fused_launches + min(g.lsqr_iters, g2.lsqr_iters) // 2
    assert np.array_equal(g2.row_indices, g.row_indices)
    A.free()
    A2.free()
