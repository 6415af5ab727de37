"""Device LSQR (graph-captured, device-side stop rules) against the reference
plain_lsqr_solve / lsqr_solve (solver.hpp:396-448, lsqr.hpp:84-207)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plain(apc, ref, ctx, p, **cfg):
    A = apc.DeviceMatrix.from_problem(ctx, p)
    g = apc.plain_lsqr_solve(A, p.b, apc.SolverConfig(**cfg))
    r = ref.solve(ref.Problem.from_apc(p), p.b, dict(cfg, trace_sample_stride=0), plain=True)
    return g, r


@pytest.mark.parametrize("cfg,m,n,mu,eps", [
    (1, 400, 50, 0.0, 1e-8),
    (1, 4000, 500, 0.0, 1e-8),
    (2, 20000, 2000, 1e-6, 1e-8),
    (2, 20000, 2000, 0.3, 1e-10),
    (3, 3000, 300, 1e-4, 1e-8),
])
def test_plain_lsqr_matches_reference(apc, ref, ctx, cfg, m, n, mu, eps):
    p = apc.Problem(cfg, m, n)
    cap = 600
    g, r = _plain(apc, ref, ctx, p, mu=mu, eps_lsqr=eps, lsqr_cap=cap)
    it_g, it_r = g.phases[0].lsqr_iters, int(r.phase_iters[0])
    assert abs(it_g - it_r) <= max(1, 0.05 * it_r), (it_g, it_r)
    assert g.phases[0].reason == r.phase_reason[0]
    # trace: phibar agrees early (rounding differences grow with j)
    k = min(len(g.trace), len(r.trace_phibar), 20)
    np.testing.assert_allclose(g.trace["phibar"][:k], r.trace_phibar[:k], rtol=1e-9)
    assert list(g.trace["matvecs"][: min(10, k)]) == list(r.trace_matvecs[: min(10, k)])
    # solution and residual
    if it_g == it_r and r.phase_reason[0] == 1:
        rel = np.linalg.norm(g.x - r.x) / np.linalg.norm(r.x)
        assert rel <= 1e-6, rel
    assert abs(g.final_relres - r.final_relres) <= 1e-6 * max(1.0, r.final_relres)
    assert g.system_matvecs == r.system_matvecs or it_g != it_r


def test_counts_and_cap(apc, ref, ctx):
    # 7 forced iterations: 7 forward + 8 transpose = 15 products (test_lsqr.cpp:69-82)
    p = apc.Problem(1, 60, 20)
    g, r = _plain(apc, ref, ctx, p, eps_lsqr=1e-300, lsqr_cap=7)
    assert g.phases[0].reason == apc.StopReason.iteration_cap
    assert g.system_matvecs == 15 == r.system_matvecs
    assert g.trace["matvecs"][-1] == 15
    np.testing.assert_allclose(g.x, r.x, rtol=1e-10, atol=1e-14)


def test_zero_rhs_returns_immediately(apc, ctx):
    p = apc.Problem(1, 50, 10)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    g = apc.plain_lsqr_solve(A, np.zeros(50), apc.SolverConfig())
    assert g.phases[0].reason == apc.StopReason.exact_zero_rhs
    assert len(g.trace) == 1 and np.all(g.x == 0.0)


def test_identity_converges_immediately(apc, ctx):
    n = 6
    A = apc.DeviceMatrix.from_numpy(ctx, np.eye(n))
    b = np.random.default_rng(1).standard_normal(n)
    g = apc.plain_lsqr_solve(A, b, apc.SolverConfig())
    assert g.phases[0].reason == apc.StopReason.gradient_tol
    assert g.trace["iter"][-1] <= 2
    np.testing.assert_allclose(g.x, b, rtol=1e-12)


def test_phibar_nonincreasing_and_rerun_identical(apc, ctx):
    p = apc.Problem(2, 20000, 2000)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    cfg = apc.SolverConfig(mu=1e-6, eps_lsqr=1e-12, lsqr_cap=300)
    g1 = apc.plain_lsqr_solve(A, p.b, cfg)
    g2 = apc.plain_lsqr_solve(A, p.b, cfg)
    ph = g1.trace["phibar"]
    assert np.all(np.diff(ph) <= 1e-12 * ph[0])
    assert np.array_equal(g1.x, g2.x)
    assert np.array_equal(g1.trace["phibar"], g2.trace["phibar"])


def test_matches_dense_least_squares(apc, ctx):
    rng = np.random.default_rng(3)
    A0 = rng.standard_normal((30, 20))
    b = rng.standard_normal(30)
    A = apc.DeviceMatrix.from_numpy(ctx, A0)
    g = apc.plain_lsqr_solve(A, b, apc.SolverConfig(eps_lsqr=1e-14, lsqr_cap=500))
    xref = np.linalg.lstsq(A0, b, rcond=None)[0]
    ra, rb = np.linalg.norm(A0 @ g.x - b), np.linalg.norm(A0 @ xref - b)
    assert ra <= (1 + 1e-8) * rb + 1e-8 * np.linalg.norm(b)
