"""Reference (oracle/_ref) per-iteration cost on C5, alone on the host: the
plain LSQR iterations of plain_lsqr_solve on [A; mu I] (lsqr_cap = K), the
input of bench.py's extrapolated reference time-to-tol.  Prints one JSON line."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import ref  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 10
t0 = time.time()
p = ref.Problem.generate(5, threads=os.cpu_count() or 1)
gen = time.time() - t0
knobs = dict(mu=1e-8, block=250, eps_lsqr=1e-8, eps_cur=3e-7, max_rank=500, seed=1, trace_sample_stride=0,
             lsqr_cap=cap)
t0 = time.time()
r = ref.solve(p, None, knobs, plain=True)
wall = time.time() - t0
it = int(np.sum(r.phase_iters))
print(json.dumps(dict(gen_s=gen, wall_s=wall, iters=it, s_per_iter=float(np.sum(r.phase_t_lsqr_ms)) / 1e3 / it,
                      nproc=os.cpu_count(), cap=cap)))
