"""Full aplicur_solve on BASELINE configs with the BASELINE.md solver settings;
prints time-to-tol and the per-phase split (augment / factor / precond / lsqr).
    python scripts/solve_configs.py c4 c5 c3 [--cap K]"""
import argparse
import json
import sys
import time
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

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["c4", "c5", "c3"])
ap.add_argument("--cap", type=int, default=0)
ap.add_argument("--gaussian", action="store_true")
args = ap.parse_args()
ctx = apc.Context(0)
for c in args.configs:
    k = int(c[1:])
    t0 = time.time()
    p = apc.Problem(k)
    gen = time.time() - t0
    A = apc.DeviceMatrix.from_problem(ctx, p)
    knobs = dict(SOLVER[k], trace_sample_stride=0, lsqr_cap=args.cap)
    if args.gaussian and not p.sparse:
        knobs["sketch_kind"] = apc.SketchKind.gaussian
    t0 = time.time()
    r = apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs))
    wall = time.time() - t0
    out = dict(config=c, gen_s=gen, time_to_tol_s=wall, total_ms=r.total_ms, setup_ms=r.setup_ms, lsqr_ms=r.lsqr_ms,
               iters=r.lsqr_iters, iter_per_s=r.lsqr_iters / max(r.lsqr_ms / 1e3, 1e-9), status=int(r.status),
               rank=len(r.row_indices), final_relres=r.final_relres, rho=r.rho_history.tolist(),
               phases=[dict(rank=ph.rank, iters=ph.lsqr_iters, reason=int(ph.reason), aug_ms=ph.t_augment_ms,
                            fac_ms=ph.t_factor_ms, pre_ms=ph.t_precond_ms, lsqr_ms=ph.t_lsqr_ms,
                            relres=ph.relres_at_end) for ph in r.phases])
    print(json.dumps(out), flush=True)
    A.free()
    del p
ctx.close()
