"""Short capped solve of a BASELINE config (profiling driver): prof_cfg.py CONFIG CAP [REPS]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_05065_b200 as apc  # noqa: E402

SOLVER = {
    1: dict(mu=0.0, block=20, eps_lsqr=1e-8, seed=1),
    2: dict(mu=1e-6, block=50, eps_lsqr=1e-8, max_rank=200, seed=1),
    3: dict(mu=1e-4, block=100, eps_lsqr=1e-8, eps_cur=3e-3, max_rank=1000, seed=1),
    4: dict(mu=0.0, block=250, eps_lsqr=1e-10, max_rank=250, seed=1),
    5: dict(mu=1e-8, block=250, eps_lsqr=1e-8, eps_cur=3e-7, max_rank=500, seed=1),
}
cfgid, cap = int(sys.argv[1]), int(sys.argv[2])
ctx = apc.Context(0)
p = apc.Problem(cfgid)
A = apc.DeviceMatrix.from_problem(ctx, p)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2  # the last solve is reported (the first pays one-time init)
for _ in range(reps):
    r = apc.aplicur_solve(A, p.b, apc.SolverConfig(lsqr_cap=cap, trace_sample_stride=0, **SOLVER[cfgid]))
print("setup_ms", r.setup_ms, "lsqr_ms", r.lsqr_ms, "iters", r.lsqr_iters,
      [(ph.rank, ph.lsqr_iters, round(ph.t_lsqr_device_ms, 1),
        round(ph.t_lsqr_device_ms * 1e3 / max(1, ph.lsqr_iters), 1)) for ph in r.phases], flush=True)
ctx.close()
