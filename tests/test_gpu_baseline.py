"""Full BASELINE-config solves on the GPU against golden results of the
unmodified reference run here (tests/golden/baseline_c*.npz, made by
oracle/make_golden.py): the north-star parity bar on configs C1 and C2."""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"

SOLVER = {
    1: dict(mu=0.0, block=20, eps_lsqr=1e-8, seed=1),
    2: dict(mu=1e-6, block=50, eps_lsqr=1e-8, max_rank=200, seed=1),
}


@pytest.mark.parametrize("cfg", [1, 2])
def test_baseline_config_parity(apc, ctx, cfg):
    f = GOLD / f"baseline_c{cfg}.npz"
    if not f.exists():
        pytest.skip("golden fixture missing")
    g = np.load(f)
    p = apc.Problem(cfg)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    r = apc.aplicur_solve(A, p.b, apc.SolverConfig(trace_sample_stride=0, **SOLVER[cfg]))
    # CUR indices and rho history: bit-exact
    assert np.array_equal(r.row_indices, g["row_indices"])
    assert np.array_equal(r.col_indices, g["col_indices"])
    assert np.array_equal(r.rho_history.view(np.uint64), g["rho_history"].view(np.uint64))
    assert int(r.status) == int(g["status"])
    assert [ph.rank for ph in r.phases] == list(g["phase_rank"])
    assert [int(ph.reason) for ph in r.phases] == list(g["phase_reason"])
    # iteration count to tolerance within +-5%
    it, itr = r.lsqr_iters, int(g["phase_iters"].sum())
    assert abs(it - itr) <= max(3, 0.05 * itr), (it, itr)
    # residual level and solution
    assert abs(r.final_relres - float(g["final_relres"])) <= 1e-6 * float(g["final_relres"])
    rel = np.linalg.norm(r.x - g["x"]) / np.linalg.norm(g["x"])
    bound = 1e-6
    fu = GOLD / f"baseline_c{cfg}_ulp.npz"
    if fu.exists():  # the reference's own sensitivity to a one-ulp change of b
        gu = np.load(fu)
        bound = max(bound, 10.0 * np.linalg.norm(gu["x"] - g["x"]) / np.linalg.norm(g["x"]))
    print(f"C{cfg}: iters {it} vs {itr}, x rel err {rel:.3e} (bound {bound:.3e}), "
          f"relres {r.final_relres:.12g} vs {float(g['final_relres']):.12g}, {r.total_ms:.0f} ms "
          f"vs reference {float(g['wall_s']):.1f} s")
    assert rel <= bound, (rel, bound)
