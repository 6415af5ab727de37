"""Capped-parity mode of SURVEY.md 8(c)(3) for the configs whose full reference
solve does not finish on the host: the GPU solver and the unmodified reference
(oracle/_ref) run the same aplicur_solve with the same knobs plus
lsqr_cap = K, so both execute the same bounded algorithm.  Compared: CUR row /
column indices (bit-exact), rho history, per-phase ranks, stop reasons and
iteration counts, the phibar trace, final x and relres.

    python scripts/capped_parity.py [--cap K] c3 c4
One JSON object per config on stdout (and gpurun_out/capped_<c>.json)."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2604_05065_b200 as apc  # noqa: E402
from oracle import ref  # noqa: E402  (test infrastructure: the checker)

SOLVER = {
    1: dict(mu=0.0, block=20, eps_lsqr=1e-8, seed=1),
    2: dict(mu=1e-6, block=50, eps_lsqr=1e-8, max_rank=200, seed=1),
    3: dict(mu=1e-4, block=100, eps_lsqr=1e-8, eps_cur=3e-3, max_rank=1000, seed=1),
    4: dict(mu=0.0, block=250, eps_lsqr=1e-10, max_rank=250, seed=1),
    5: dict(mu=1e-8, block=250, eps_lsqr=1e-8, eps_cur=3e-7, max_rank=500, seed=1),
}


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    if a.shape != b.shape:
        return None
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return float(d / n) if n > 0 else float(d)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c4", "c3"])
    ap.add_argument("--cap", type=int, default=10)
    args = ap.parse_args()
    ctx = apc.Context(0)
    out_dir = ROOT / "gpurun_out"
    out_dir.mkdir(exist_ok=True)
    for c in args.configs:
        k = int(c[1:])
        knobs = dict(SOLVER[k], trace_sample_stride=0, lsqr_cap=args.cap)
        t0 = time.time()
        p = apc.Problem(k)
        gen_s = time.time() - t0
        A = apc.DeviceMatrix.from_problem(ctx, p)
        t0 = time.time()
        g = apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs))
        gpu_s = time.time() - t0
        A.free()
        rp = ref.Problem.from_apc(p)
        t0 = time.time()
        r = ref.solve(rp, p.b, knobs)
        ref_s = time.time() - t0
        g_rank = np.array([ph.rank for ph in g.phases])
        g_iters = np.array([ph.lsqr_iters for ph in g.phases])
        g_reason = np.array([int(ph.reason) for ph in g.phases])
        gtr = g.trace
        res = dict(
            config=c, cap=args.cap, gen_s=gen_s, gpu_s=gpu_s, ref_s=ref_s,
            row_indices_equal=bool(np.array_equal(g.row_indices, r.row_indices)),
            col_indices_equal=bool(np.array_equal(g.col_indices, r.col_indices)),
            rank=int(len(g.row_indices)), ref_rank=int(len(r.row_indices)),
            rho_history_equal=bool(np.array_equal(g.rho_history, r.rho_history)),
            rho_history_rel=rel(g.rho_history, r.rho_history),
            phase_ranks_equal=bool(np.array_equal(g_rank, r.phase_rank)),
            phase_iters=g_iters.tolist(), ref_phase_iters=r.phase_iters.tolist(),
            phase_reasons=g_reason.tolist(), ref_phase_reasons=r.phase_reason.tolist(),
            phibar_rel=rel(gtr["phibar"], r.trace_phibar) if len(gtr) == len(r.trace_phibar) else None,
            x_rel=rel(g.x, r.x), relres=float(g.final_relres), ref_relres=float(r.final_relres),
            status=int(g.status), ref_status=int(r.status))
        print(json.dumps(res), flush=True)
        (out_dir / f"capped_{c}.json").write_text(json.dumps(res, indent=1))
        del rp, p
    ctx.close()


if __name__ == "__main__":
    main()
