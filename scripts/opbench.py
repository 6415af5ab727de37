"""Operator-pair bandwidth probe: A*v + A^T*u on device buffers, timed with CUDA
events on the library stream.  Prints GB/s against the algorithmic bytes of
SURVEY.md 8(d) (dense 16mn + 16(m+n); CSR 24 nnz + 4(m+1) + 4(n+1) + 16(m+n))."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_05065_b200 as apc  # noqa: E402


def bench(ctx, A, m, n, nnz, sparse, iters=20):
    dev = torch.device("cuda:0")
    x = torch.randn(n, dtype=torch.float64, device=dev)
    y = torch.empty(m, dtype=torch.float64, device=dev)
    g = torch.empty(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    s = torch.cuda.ExternalStream(ctx.stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for _ in range(3):
        A.apply_dev(x.data_ptr(), y.data_ptr())
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ctx.sync()
    with torch.cuda.stream(s):
        ev[0].record(s)
        for _ in range(iters):
            A.apply_dev(x.data_ptr(), y.data_ptr())
        ev[1].record(s)
        for _ in range(iters):
            A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
        ev[2].record(s)
    ctx.sync()
    tf = ev[0].elapsed_time(ev[1]) / iters
    ta = ev[1].elapsed_time(ev[2]) / iters
    if sparse:
        bf = 12 * nnz + 4 * (m + 1) + 8 * (m + n)
        ba = 12 * nnz + 4 * (n + 1) + 8 * (m + n)
    else:
        bf = ba = 8 * m * n + 8 * (m + n)
    return dict(fwd_ms=tf, adj_ms=ta, fwd_GBps=bf / tf / 1e6, adj_GBps=ba / ta / 1e6,
                pair_GBps=(bf + ba) / (tf + ta) / 1e6)


def main():
    ctx = apc.Context(0)
    out = {}
    which = sys.argv[1:] or ["c2", "c5", "dense50k", "dense100kx10k"]
    for w in which:
        t0 = time.time()
        if w == "c2":
            p = apc.Problem(2)
            A = apc.DeviceMatrix.from_problem(ctx, p)
            m, n, nnz, sp = p.m, p.n, p.nnz, True
        elif w == "c5":
            p = apc.Problem(5)
            A = apc.DeviceMatrix.from_problem(ctx, p)
            m, n, nnz, sp = p.m, p.n, p.nnz, True
        elif w == "dense50k":
            m = n = 50000
            a = np.random.default_rng(0).standard_normal(m * n)
            A = apc.DeviceMatrix.dense(ctx, a, m, n)
            del a
            nnz, sp = m * n, False
        else:
            m, n = 100000, 10000
            a = np.random.default_rng(0).standard_normal(m * n)
            A = apc.DeviceMatrix.dense(ctx, a, m, n)
            del a
            nnz, sp = m * n, False
        gen = time.time() - t0
        r = bench(ctx, A, m, n, nnz, sp)
        r["setup_s"] = gen
        out[w] = r
        print(w, json.dumps(r), flush=True)
        A.free()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
