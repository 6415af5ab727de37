"""Minimal operator-pair driver for ncu: <config> -> upload, 2 warm pairs, 1 pair.
    ncu ... -k regex:"csr_|dense_" -s 4 -c 2 python scripts/ncu_ops.py 5"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_05065_b200 as apc  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ctx = apc.Context(0)
p = apc.Problem(cfg, m, n)
A = apc.DeviceMatrix.from_problem(ctx, p)
x = torch.randn(p.n, dtype=torch.float64, device="cuda")
y = torch.empty(p.m, dtype=torch.float64, device="cuda")
g = torch.empty(p.n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for _ in range(3):
    A.apply_dev(x.data_ptr(), y.data_ptr())
    A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
ctx.sync()
print("ok", p.m, p.n, p.nnz)
ctx.close()
