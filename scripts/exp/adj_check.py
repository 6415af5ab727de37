"""Check: C5-shaped adjoint through the tail stream vs the units path (bit-identical
is not expected: different summation grouping; compare to 1e-13 relative) and timing."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_05065_b200 as apc  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = apc.Context(0)
p = apc.Problem(cfg)
A = apc.DeviceMatrix.from_problem(ctx, p)
rng = np.random.default_rng(1)
u = rng.standard_normal(p.m)
g = A.apply(u, transpose=True)
# exact-ish reference: CSC column dots in long double via numpy float128
cp, ri, va = p.colptr, p.rowidx, p.vals
prod = va * u[ri]
ref = np.add.reduceat(prod, cp[:-1]) if p.nnz else np.zeros(p.n)
ref[np.diff(cp) == 0] = 0.0
scale = np.add.reduceat(np.abs(prod), cp[:-1])
scale[np.diff(cp) == 0] = 0.0
err = np.abs(g - ref) / np.maximum(scale, 1e-300)
print(f"tail_seg={os.environ.get('APC_TAIL_SEG', '1')}: max componentwise err {err.max():.3e} "
      f"(bound ~ nnz_col * 2^-53), nan {np.isnan(g).sum()}", flush=True)
g2 = A.apply(u, transpose=True)
print("rerun bit-identical:", np.array_equal(g, g2))
