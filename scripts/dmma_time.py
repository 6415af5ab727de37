"""Gaussian sketch Y = S A on BASELINE C1/C3/C4: exact-order kernel vs the
opt-in DMMA kernel (CUDA events around the sketch launch, reported by the
library), TFLOP/s = 2 s m n / t against the FP64 peak.
    python scripts/dmma_time.py [c1 c3 c4]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_05065_b200 as apc  # noqa: E402

BLOCK = {1: 20, 3: 100, 4: 250}
ctx = apc.Context(0)
for c in sys.argv[1:] or ["c1", "c3", "c4"]:
    k = int(c[1:])
    t0 = time.time()
    p = apc.Problem(k)
    gen = time.time() - t0
    A = apc.DeviceMatrix.from_problem(ctx, p)
    s = int(np.ceil(1.1 * BLOCK[k]))
    out = dict(config=c, s=s, m=p.m, n=p.n, gen_s=gen, flops=2.0 * s * p.m * p.n)
    Y = {}
    for kind in (apc.SketchKind.gaussian, apc.SketchKind.gaussian_dmma):
        best = None
        for _ in range(3):
            cur = apc.CurState(A, BLOCK[k], seed=1, sketch=kind)
            emb, ker = cur.sketch_timing()
            best = ker if best is None else min(best, ker)
        Y[kind] = cur.sketch_matrix()
        out[kind.name] = dict(kernel_ms=best, embed_ms=emb, tflops=out["flops"] / (best * 1e-3) / 1e12)
    out["dmma_vs_exact_maxrel"] = float(np.max(np.abs(Y[2] - Y[1])) / np.max(np.abs(Y[1])))
    print(json.dumps(out), flush=True)
    A.free()
ctx.close()
