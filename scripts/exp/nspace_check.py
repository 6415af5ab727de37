"""Fused n-space kernel vs the unfused kernels (APC_NSPACE=0/1 set by the
caller): run a capped C5 solve (or plain LSQR on a config) and dump x + trace.

    APC_NSPACE=1 python scripts/exp/nspace_check.py 5 300 out.npz
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_05065_b200 as apc  # noqa: E402

cfg, cap, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
ctx = apc.Context(0)
p = apc.Problem(cfg)
A = apc.DeviceMatrix.from_problem(ctx, p)
knobs = {5: dict(mu=1e-8, block=250, eps_lsqr=1e-8, eps_cur=3e-7, max_rank=500, seed=1),
         2: dict(mu=1e-6, block=50, eps_lsqr=1e-8, eps_cur=3e-5, max_rank=200, seed=1)}[cfg]
r = apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs, lsqr_cap=cap, trace_sample_stride=0))
rp = apc.plain_lsqr_solve(A, p.b, apc.SolverConfig(mu=knobs["mu"], eps_lsqr=1e-8, lsqr_cap=cap))
np.savez(out, x=r.x, phibar=np.asarray(r.trace["phibar"]), xp=rp.x, phibar_p=np.asarray(rp.trace["phibar"]),
         iters=[ph.lsqr_iters for ph in r.phases])
ph = r.phases[-1]
print(f"{out}: iters {[q.lsqr_iters for q in r.phases]}, last phase {1e3 * ph.t_lsqr_device_ms / max(1, ph.lsqr_iters):.1f} "
      f"us/it; plain {rp.lsqr_iters} its {1e3 * rp.phases[-1].t_lsqr_device_ms / max(1, rp.lsqr_iters):.1f} us/it, "
      f"launches {ctx.launches}", flush=True)
