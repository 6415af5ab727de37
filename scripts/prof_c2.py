"""Short C2 solve for profiling: BASELINE C2 settings with a per-phase LSQR cap,
so an ncu launch list covers setup + a few hundred steady-state iterations."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_05065_b200 as apc  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cfgid = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = apc.Context(0)
p = apc.Problem(cfgid)
A = apc.DeviceMatrix.from_problem(ctx, p)
knobs = {2: dict(mu=1e-6, block=50, eps_lsqr=1e-8, max_rank=200, seed=1),
         1: dict(mu=0.0, block=20, eps_lsqr=1e-8, seed=1)}[cfgid]
cfg = apc.SolverConfig(lsqr_cap=cap, trace_sample_stride=0, **knobs)
for k in range(2):
    t = time.perf_counter()
    r = apc.aplicur_solve(A, p.b, cfg)
    dt = time.perf_counter() - t
    print(f"solve {k}: {dt*1e3:.1f} ms, setup {r.setup_ms:.1f} ms, lsqr {r.lsqr_ms:.1f} ms, iters {r.lsqr_iters}, "
          f"us/iter {r.lsqr_ms*1e3/max(1,r.lsqr_iters):.1f}, phases "
          f"{[(ph.rank, ph.lsqr_iters, round(ph.t_augment_ms,1), round(ph.t_factor_ms,1), round(ph.t_precond_ms,1), round(ph.t_lsqr_ms,1)) for ph in r.phases]}",
          flush=True)
ctx.close()
