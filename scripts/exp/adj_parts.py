"""Experiment: live time of the C5 adjoint's parts (APC_ADJ_MASK set per run by the caller)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_05065_b200 as apc  # noqa: E402

ctx = apc.Context(0)
p = apc.Problem(5)
A = apc.DeviceMatrix.from_problem(ctx, p)
dev = torch.device("cuda:0")
x = torch.randn(p.n, dtype=torch.float64, device=dev)
y = torch.empty(p.m, dtype=torch.float64, device=dev)
g = torch.empty(p.n, dtype=torch.float64, device=dev)
s = torch.cuda.ExternalStream(ctx.stream)
torch.cuda.synchronize()
for _ in range(3):
    A.apply_dev(x.data_ptr(), y.data_ptr())
    A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
ctx.sync()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
R = 20
ev[0].record(s)
for _ in range(R):
    A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
ev[1].record(s)
for _ in range(R):
    A.apply_dev(x.data_ptr(), y.data_ptr())
    A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
ev[2].record(s)
ctx.sync()
print(f"mask {os.environ.get('APC_ADJ_MASK', 'all')}: adj back-to-back {ev[0].elapsed_time(ev[1]) / R * 1e3:.1f} us, "
      f"pair interleaved {ev[1].elapsed_time(ev[2]) / R * 1e3:.1f} us", flush=True)
