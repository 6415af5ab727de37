"""Fused dense operator pair (dense_pair.cu) against the two-pass kernels:
correctness (y, g, ||y||^2 within rounding; two runs bit-identical) and time.

    python scripts/pair_bench.py small        # forced on small shapes (APC_DENSE_PAIR=1)
    python scripts/pair_bench.py c3 [c4]      # BASELINE dense configs (auto)
    python scripts/pair_bench.py rand M N
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(apc, ctx, A, m, n, tag, iters=10):
    dev = torch.device("cuda:0")
    torch.manual_seed(1)
    x = torch.randn(n, dtype=torch.float64, device=dev)
    y0 = torch.empty(m, dtype=torch.float64, device=dev)
    g0 = torch.empty(n, dtype=torch.float64, device=dev)
    y1 = torch.zeros(m, dtype=torch.float64, device=dev)
    g1 = torch.zeros(n + 1, dtype=torch.float64, device=dev)
    y2 = torch.zeros(m, dtype=torch.float64, device=dev)
    g2 = torch.zeros(n + 1, dtype=torch.float64, device=dev)
    s = torch.cuda.ExternalStream(ctx.stream)
    torch.cuda.synchronize()
    A.apply_dev(x.data_ptr(), y0.data_ptr())
    A.apply_dev(y0.data_ptr(), g0.data_ptr(), transpose=True)
    fused = A.pair_dev(x.data_ptr(), y1.data_ptr(), g1.data_ptr())
    A.pair_dev(x.data_ptr(), y2.data_ptr(), g2.data_ptr())
    ctx.sync()
    ey = float((y1 - y0).abs().max() / y0.abs().max())
    eg = float((g1[:n] - g0).abs().max() / g0.abs().max())
    en = float(abs(g1[n] - (y0 * y0).sum()) / (y0 * y0).sum())
    same = bool(torch.equal(y1, y2) and torch.equal(g1, g2))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(s)
    for _ in range(iters):
        A.apply_dev(x.data_ptr(), y0.data_ptr())
        A.apply_dev(y0.data_ptr(), g0.data_ptr(), transpose=True)
    ev[1].record(s)
    for _ in range(iters):
        A.pair_dev(x.data_ptr(), y1.data_ptr(), g1.data_ptr())
    ev[2].record(s)
    ctx.sync()
    t2 = ev[0].elapsed_time(ev[1]) / iters
    t1 = ev[1].elapsed_time(ev[2]) / iters
    byts = 16.0 * m * n + 16.0 * (m + n)
    out = dict(tag=tag, m=m, n=n, fused=fused, err_y=ey, err_g=eg, err_norm=en, rerun_identical=same,
               two_pass_ms=t2, fused_ms=t1, two_pass_GBps=byts / t2 / 1e6, fused_GBps_algorithmic=byts / t1 / 1e6,
               fused_GBps_read_once=(8.0 * m * n + 16.0 * (m + n)) / t1 / 1e6, speedup=t2 / t1,
               env={k: v for k, v in os.environ.items() if k.startswith("APC_D")})
    print(json.dumps(out), flush=True)
    assert os.environ.get('APC_DP_DEBUG') or (ey < 1e-12 and eg < 1e-12 and en < 1e-12 and same), out
    return out


def main():
    args = sys.argv[1:] or ["small"]
    if args[0] in ("small", "rand"):
        os.environ.setdefault("APC_DENSE_PAIR", "1")
    import paper_2604_05065_b200 as apc

    ctx = apc.Context(0)
    if args[0] == "small":
        rng = np.random.default_rng(0)
        for (m, n) in [(3000, 2500), (10007, 4001), (777, 9000), (20000, 12345), (4096, 40000)]:
            Ah = np.asfortranarray(rng.standard_normal((m, n)))
            A = apc.DeviceMatrix.from_numpy(ctx, Ah)
            run(apc, ctx, A, m, n, f"rand{m}x{n}", iters=5)
            A.free()
    elif args[0] == "rand":
        m, n = int(args[1]), int(args[2])
        dev = torch.device("cuda:0")
        Ad = torch.randn(n, m, dtype=torch.float64, device=dev)  # column-major m x n
        A = apc.DeviceMatrix.from_numpy(ctx, Ad.cpu().numpy().T)
        del Ad
        run(apc, ctx, A, m, n, f"rand{m}x{n}")
        A.free()
    elif args[0] == "sweep":
        p = apc.Problem(int(args[1][1:]))
        combos = [dict(), dict(APC_DP_RB="8")]
        for c in combos:
            for k in ("APC_DP_GROUPS", "APC_DP_RB", "APC_DP_STAGES", "APC_DP_DEBUG"):
                os.environ.pop(k, None)
            os.environ.update(c)
            A = apc.DeviceMatrix.from_problem(ctx, p)
            try:
                run(apc, ctx, A, p.m, p.n, args[1])
            except Exception as e:
                print("failed", c, e, flush=True)
            A.free()
    else:
        for w in args:
            p = apc.Problem(int(w[1:]))
            A = apc.DeviceMatrix.from_problem(ctx, p)
            run(apc, ctx, A, p.m, p.n, w)
            A.free()
    ctx.close()


if __name__ == "__main__":
    main()
