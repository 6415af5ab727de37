"""Print the device's capped-parity trace beside the reference fixture's
(tests/golden/capped_cK_k200.npz): per-phase phibar, its decrease, and the
one-ulp rerun's, to see where the two trajectories part.

    python scripts/exp/capped_trace.py 3
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_2604_05065_b200 as apc  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = np.load(ROOT / f"tests/golden/capped_c{k}_k200.npz")
gu = np.load(ROOT / f"tests/golden/capped_c{k}_k200_ulp.npz")
meta = json.loads(str(g["meta"]))
ctx = apc.Context(0)
p = apc.Problem(k)
A = apc.DeviceMatrix.from_problem(ctx, p)
r = apc.aplicur_solve(A, p.b, apc.SolverConfig(**meta["knobs"]))
print("iters", [ph.lsqr_iters for ph in r.phases], "ref", g["phase_iters"].tolist(), "ulp", gu["phase_iters"].tolist())
print("sigma_hat", [ph.sigma_hat for ph in r.phases], "ref", g["phase_sigma_hat"].tolist())
for ph in r.phases:
    print("phase", ph.phase, ph.rank, ph.reason, "spectrum tail", ph.precond_spectrum[-3:])
tp, tb = np.asarray(r.trace["phase"]), np.asarray(r.trace["phibar"])
ph0 = np.unique(g["trace_phase"])[0]
pr = g["trace_phibar"][g["trace_phase"] == ph0]
pu = gu["trace_phibar"][: int(gu["phase_iters"][0]) + 1]
pg = tb[tp == np.unique(tp)[0]]
for i in range(1, max(len(pr), len(pg), len(pu))):
    f = lambda a: f"{a[i]:.12e} {a[i-1]-a[i]:.6e}" if i < len(a) else "-"
    rel = abs(pg[i] - pr[i]) / abs(pr[i]) if i < min(len(pg), len(pr)) else float("nan")
    print(i, "gpu", f(pg), "| ref", f(pr), "| ulp", f(pu), f"| rel {rel:.2e}")
