"""Plain LSQR on C5 under APC_NSPACE=0/1: phibar of the first iterations (debug)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_05065_b200 as apc  # noqa: E402

ctx = apc.Context(0)
p = apc.Problem(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
A = apc.DeviceMatrix.from_problem(ctx, p)
for mu in (1e-8, 0.0):
    rp = apc.plain_lsqr_solve(A, p.b, apc.SolverConfig(mu=mu, eps_lsqr=1e-8, lsqr_cap=6))
    ph = np.asarray(rp.trace["phibar"])
    print(os.environ.get("APC_NSPACE"), "mu", mu, " ".join(f"{v:.17g}" for v in ph), "x0", repr(rp.x[:3]), flush=True)
