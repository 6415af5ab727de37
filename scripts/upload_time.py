"""Upload / first-solve overheads of a fresh device matrix (C2): upload time,
solve on the fresh matrix, solve again on the same matrix."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_05065_b200 as apc  # noqa: E402

ctx = apc.Context(0)
p = apc.Problem(2)
cfg = apc.SolverConfig(mu=1e-6, block=50, eps_lsqr=1e-8, max_rank=200, seed=1, trace_sample_stride=0)
for k in range(3):
    t = time.perf_counter()
    A = apc.DeviceMatrix.from_problem(ctx, p)
    ctx.sync()
    t1 = time.perf_counter()
    r1 = apc.aplicur_solve(A, p.b, cfg)
    t2 = time.perf_counter()
    r2 = apc.aplicur_solve(A, p.b, cfg)
    t3 = time.perf_counter()
    print(f"upload {1e3 * (t1 - t):.1f} ms | fresh solve {1e3 * (t2 - t1):.1f} ms (setup {r1.setup_ms:.1f}, lsqr "
          f"{r1.lsqr_ms:.1f}, iters {r1.lsqr_iters}) | again {1e3 * (t3 - t2):.1f} ms (setup {r2.setup_ms:.1f}, "
          f"lsqr {r2.lsqr_ms:.1f}, iters {r2.lsqr_iters})", flush=True)
    A.free()
