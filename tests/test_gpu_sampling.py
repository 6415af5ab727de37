"""True-residual sampling of the solver observers (solver.hpp:222-236 for
aplicur_solve, :418-427 for plain_lsqr_solve): with trace_sample_stride = k
every trace row with iter >= 1 and iter % k == 0 carries
||A_mu x_j - [b; 0]|| / ||b||, x_j = x + P^{-1} y_j (plain: y_j), computed on
the device inside the iteration graph; the other rows stay NaN.  Values are
compared with the reference's observer on the same (phase, iter) rows."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # cfg, m, n, knobs, stride
    (1, 400, 50, dict(mu=0.0, eps_lsqr=1e-8, block=5, seed=1), 1),            # dense, explicit basis
    (2, 4000, 400, dict(mu=1e-3, eps_lsqr=1e-10, block=8, seed=3, max_rank=40), 1),  # sparse, implicit, mu tail
    (3, 3000, 300, dict(mu=1e-4, eps_lsqr=1e-8, block=10, seed=1, max_rank=60), 3),  # dense, mu tail
    (2, 4000, 400, dict(mu=1e-3, eps_lsqr=1e-10, block=8, seed=3, max_rank=40, variant=1), 2),  # svd-free
]


def _rows(trace_phase, trace_iter, relres):
    return {(int(p), int(i)): float(r) for p, i, r in zip(trace_phase, trace_iter, relres)}


def _check_mask(phase, it, rr, stride):
    for p, i, r in zip(phase, it, rr):
        if i >= 1 and i % stride == 0:
            assert np.isfinite(r), (p, i)
        else:
            assert np.isnan(r), (p, i)


def _worst(a_rows, r_rows):
    common = [k for k in r_rows if k in a_rows and np.isfinite(r_rows[k])]
    assert common
    return max(abs(a_rows[k] - r_rows[k]) / r_rows[k] for k in common)


def _compare(g_rows, r_rows, ref_rerun):
    """Bar 1e-6, widened only to the reference's own sensitivity: the
    unmodified reference rerun on b perturbed by one ulp (long phases drift
    along the LSQR trajectory, as x does in test_gpu_solver)."""
    worst = _worst(g_rows, r_rows)
    if worst > 1e-6:
        self_sens = _worst(ref_rerun(), r_rows)
        assert worst <= 10.0 * self_sens, (worst, self_sens)


@pytest.mark.parametrize("cfg,m,n,knobs,stride", CASES)
def test_aplicur_true_relres_matches_reference(apc, ref, ctx, cfg, m, n, knobs, stride):
    p = apc.Problem(cfg, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    g = apc.aplicur_solve(A, p.b, apc.SolverConfig(trace_sample_stride=stride, **knobs))
    r = ref.solve(ref.Problem.from_apc(p), p.b, dict(knobs, trace_sample_stride=stride))
    tr = g.trace
    _check_mask(tr["phase"], tr["iter"], tr["true_relres"], stride)
    _check_mask(r.trace_phase, r.trace_iter, r.trace_true_relres, stride)
    g_rows = _rows(tr["phase"], tr["iter"], tr["true_relres"])
    r_rows = _rows(r.trace_phase, r.trace_iter, r.trace_true_relres)

    def rerun():
        r2 = ref.solve(ref.Problem.from_apc(p), np.nextafter(p.b, np.inf), dict(knobs, trace_sample_stride=stride))
        return _rows(r2.trace_phase, r2.trace_iter, r2.trace_true_relres)

    _compare(g_rows, r_rows, rerun)
    # the final phase's last row, when sampled, is the final residual
    last = tr[-1]
    if last["iter"] >= 1 and last["iter"] % stride == 0:
        assert last["true_relres"] == pytest.approx(g.final_relres, rel=1e-12)


def test_sampling_does_not_change_the_solve(apc, ctx, monkeypatch):
    # sampling forces the graph path; pin the unsampled run to it too (the
    # persistent kernel's reduction order differs from the graph path's)
    monkeypatch.setenv("APC_LSQR_MODE", "while")
    p = apc.Problem(2, 4000, 400)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    knobs = dict(mu=1e-3, eps_lsqr=1e-10, block=8, seed=3, max_rank=40)
    a = apc.aplicur_solve(A, p.b, apc.SolverConfig(trace_sample_stride=0, **knobs))
    b = apc.aplicur_solve(A, p.b, apc.SolverConfig(trace_sample_stride=1, **knobs))
    assert np.array_equal(a.x, b.x)
    assert [q.lsqr_iters for q in a.phases] == [q.lsqr_iters for q in b.phases]
    assert np.all(np.isnan(a.trace["true_relres"]))


@pytest.mark.parametrize("cfg,m,n,mu,stride", [(1, 400, 50, 0.0, 1), (2, 4000, 400, 1e-3, 2), (3, 2000, 200, 0.0, 5)])
def test_plain_true_relres_matches_reference(apc, ref, ctx, cfg, m, n, mu, stride):
    p = apc.Problem(cfg, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    knobs = dict(mu=mu, eps_lsqr=1e-8, lsqr_cap=300)
    g = apc.plain_lsqr_solve(A, p.b, apc.SolverConfig(trace_sample_stride=stride, **knobs))
    r = ref.solve(ref.Problem.from_apc(p), p.b, dict(knobs, trace_sample_stride=stride), plain=True)
    tr = g.trace
    _check_mask(tr["phase"], tr["iter"], tr["true_relres"], stride)

    def rerun():
        r2 = ref.solve(ref.Problem.from_apc(p), np.nextafter(p.b, np.inf), dict(knobs, trace_sample_stride=stride),
                       plain=True)
        return _rows(r2.trace_phase, r2.trace_iter, r2.trace_true_relres)

    _compare(_rows(tr["phase"], tr["iter"], tr["true_relres"]),
             _rows(r.trace_phase, r.trace_iter, r.trace_true_relres), rerun)


def test_python_hooks_and_spectrum(apc, ctx):
    """SolveHooks through the Python API and PhaseReport.precond_spectrum
    (svd variant: sqrt(sigma_cur^2 + mu^2), target level its last entry)."""
    p = apc.Problem(2, 4000, 400)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    knobs = dict(mu=1e-3, eps_lsqr=1e-10, block=8, seed=3, max_rank=40, trace_sample_stride=0)
    seen, ends = [], []
    hooks = apc.SolveHooks(on_rebuild=lambda cur, pc, ph: seen.append((cur, pc, ph)),
                           on_phase_end=lambda ph, x: ends.append((ph, x)))
    r = apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs), hooks=hooks)
    r0 = apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs))
    assert np.array_equal(r.x, r0.x)
    assert [s[2] for s in seen] == [q.phase for q in r.phases] == [e[0] for e in ends]
    assert np.array_equal(ends[-1][1], r.x)
    for (cur, pc, _), q in zip(seen, r.phases):
        assert cur.rank == pc.rank == q.rank
        assert np.array_equal(cur.row_indices, r.row_indices[: q.rank])
        assert np.array_equal(cur.col_indices, r.col_indices[: q.rank])
        assert cur.rho == q.rho and pc.target_level == q.sigma_hat
        assert np.array_equal(pc.regularized_spectrum, q.precond_spectrum)
        assert q.precond_spectrum.size == q.rank
        assert np.allclose(q.precond_spectrum, np.sqrt(pc.cur_spectrum ** 2 + 1e-6), rtol=1e-15)
        assert q.sigma_hat == q.precond_spectrum[-1]

    def boom(ph, x):
        raise RuntimeError("hook")

    with pytest.raises(RuntimeError, match="hook"):
        apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs), hooks=apc.SolveHooks(on_phase_end=boom))
