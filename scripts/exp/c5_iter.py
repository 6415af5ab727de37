"""C5 LSQR iteration time (device ms / iteration of the rank-500 phase, lsqr_cap K)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_05065_b200 as apc  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
ctx = apc.Context(0)
p = apc.Problem(5)
A = apc.DeviceMatrix.from_problem(ctx, p)
cfg = apc.SolverConfig(mu=1e-8, block=250, eps_lsqr=1e-8, eps_cur=3e-7, max_rank=500, seed=1, lsqr_cap=cap,
                       trace_sample_stride=0)
for rep in range(2):
    r = apc.aplicur_solve(A, p.b, cfg)
    ph = r.phases[-1]
    print(f"{os.environ.get('TAG', '')} rep {rep}: setup {r.setup_ms:.0f} ms, last phase {ph.lsqr_iters} its, "
          f"{1e3 * ph.t_lsqr_device_ms / ph.lsqr_iters:.1f} us/it, relres {r.final_relres:.10g}", flush=True)
