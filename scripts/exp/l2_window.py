"""Experiment: C5 operator pair with an L2 persisting access-policy window on
u (the A*v output / A^T*u input, 64 MB) versus none."""
import sys
from pathlib import Path

import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_05065_b200 as apc  # noqa: E402


def pair(ctx, A, x, y, g, reps=20):
    s = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        A.apply_dev(x.data_ptr(), y.data_ptr())
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ctx.sync()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(s)
    for _ in range(reps):
        A.apply_dev(x.data_ptr(), y.data_ptr())
    ev[1].record(s)
    for _ in range(reps):
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ev[2].record(s)
    for _ in range(reps):  # interleaved, as in LSQR
        A.apply_dev(x.data_ptr(), y.data_ptr())
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ev[3].record(s)
    ctx.sync()
    return [ev[i].elapsed_time(ev[i + 1]) / reps * 1e3 for i in range(3)]


def set_window(stream, ptr, nbytes, ratio):
    v = rt.cudaStreamAttrValue()
    w = v.accessPolicyWindow
    w.base_ptr = ptr
    w.num_bytes = nbytes
    w.hitRatio = ratio
    w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
    w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    v.accessPolicyWindow = w
    err, = rt.cudaStreamSetAttribute(stream, rt.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, v)
    return err


ctx = apc.Context(0)
err, prop = rt.cudaGetDeviceProperties(0)
print("l2", prop.l2CacheSize, "persistingL2CacheMaxSize", prop.persistingL2CacheMaxSize,
      "accessPolicyMaxWindowSize", prop.accessPolicyMaxWindowSize, flush=True)
p = apc.Problem(5)
A = apc.DeviceMatrix.from_problem(ctx, p)
dev = torch.device("cuda:0")
x = torch.randn(p.n, dtype=torch.float64, device=dev)
y = torch.empty(p.m, dtype=torch.float64, device=dev)
g = torch.empty(p.n, dtype=torch.float64, device=dev)
torch.cuda.synchronize()
print("none      fwd/adj/pair us", pair(ctx, A, x, y, g), flush=True)
print("setlimit", rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize))
for ratio in (1.0, 0.75, 0.5):
    nb = min(8 * p.m, prop.accessPolicyMaxWindowSize)
    print("window", set_window(ctx.stream, y.data_ptr(), nb, ratio), nb, ratio)
    print(f"u window {ratio}: fwd/adj/pair us", pair(ctx, A, x, y, g), flush=True)
    rt.cudaCtxResetPersistingL2Cache()
set_window(ctx.stream, 0, 0, 0.0)
print("reset      fwd/adj/pair us", pair(ctx, A, x, y, g), flush=True)
