"""C5 solve with a small per-phase LSQR cap (profiling driver)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_05065_b200 as apc  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 50
ctx = apc.Context(0)
p = apc.Problem(5)
A = apc.DeviceMatrix.from_problem(ctx, p)
cfg = apc.SolverConfig(mu=1e-8, block=250, eps_lsqr=1e-8, eps_cur=3e-7, max_rank=500, seed=1, lsqr_cap=cap,
                       trace_sample_stride=0)
r = apc.aplicur_solve(A, p.b, cfg)
print("setup_ms", r.setup_ms, "lsqr_ms", r.lsqr_ms, "iters", r.lsqr_iters,
      [(ph.rank, ph.lsqr_iters, round(ph.t_augment_ms), round(ph.t_precond_ms), round(ph.t_lsqr_device_ms, 1))
       for ph in r.phases])
ctx.close()
