"""Per-config measurement + parity on the GPU box for BASELINE configs C1..C5.

For each config: host generation, upload, operator-pair bandwidth (A*v, A^T*u,
CUDA events on the library stream) against the algorithmic bytes of
SURVEY.md 8(d), the one-time sketch (sparse-sign exact-order; Gaussian
exact-order GEMM for dense), the first CUR steps on the GPU, then -- unless
--gpu-only -- the unmodified reference (oracle/_ref) on the host CPU for the
same CUR steps (I, J, rho bit-exact) and its operator-pair time.

    python scripts/run_configs.py [--gpu-only] [--steps K] c3 c4 c5
Writes one JSON object per config to stdout (and gpurun_out/configs_<c>.json).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2604_05065_b200 as apc  # noqa: E402

BLOCK = {1: 20, 2: 50, 3: 100, 4: 250, 5: 250}
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0


def op_pair(ctx, A, p, reps=20):
    dev = torch.device("cuda", 0)
    x = torch.randn(p.n, dtype=torch.float64, device=dev)
    y = torch.empty(p.m, dtype=torch.float64, device=dev)
    g = torch.empty(p.n, dtype=torch.float64, device=dev)
    for _ in range(3):
        A.apply_dev(x.data_ptr(), y.data_ptr())
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ctx.sync()
    s = torch.cuda.ExternalStream(ctx.stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(s)
    for _ in range(reps):
        A.apply_dev(x.data_ptr(), y.data_ptr())
    ev[1].record(s)
    for _ in range(reps):
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ev[2].record(s)
    ctx.sync()
    tf, ta = ev[0].elapsed_time(ev[1]) / reps / 1e3, ev[1].elapsed_time(ev[2]) / reps / 1e3
    if p.sparse:
        b = 24 * p.nnz + 4 * (p.m + 1) + 4 * (p.n + 1) + 16 * (p.m + p.n)
    else:
        b = 16 * p.m * p.n + 16 * (p.m + p.n)
    return dict(fwd_ms=tf * 1e3, adj_ms=ta * 1e3, pair_bytes=b, pair_GBps=b / (tf + ta) / 1e9,
                frac_of_measured_hbm=b / (tf + ta) / 1e9 / PEAK)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c3", "c4", "c5"])
    ap.add_argument("--gpu-only", action="store_true")
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    ctx = apc.Context(0)
    out_dir = ROOT / "gpurun_out"
    out_dir.mkdir(exist_ok=True)
    for c in args.configs:
        k = int(c[1:])
        rec = {"config": c}
        t0 = time.time()
        p = apc.Problem(k)
        rec["gen_s"] = time.time() - t0
        rec.update(m=p.m, n=p.n, nnz=p.nnz, sparse=p.sparse)
        t0 = time.time()
        A = apc.DeviceMatrix.from_problem(ctx, p)
        ctx.sync()
        rec["upload_s"] = time.time() - t0
        rec["op_pair"] = op_pair(ctx, A, p)
        print(json.dumps(rec), flush=True)
        block = BLOCK[k]
        sk = {}
        for kind in ([apc.SketchKind.sparse_sign] + ([] if p.sparse else [apc.SketchKind.gaussian])):
            torch.cuda.synchronize()
            t0 = time.time()
            cur = apc.CurState(A, block, seed=1, sketch=kind)
            ctx.sync()
            dt = time.time() - t0
            s = int(np.ceil(1.1 * block))
            emb_ms, dev_ms = cur.sketch_timing()
            if kind == apc.SketchKind.gaussian:
                sk["gaussian"] = dict(s=s, seconds=dt, embedding_host_ms=emb_ms, kernel_ms=dev_ms,
                                      flops=2.0 * s * p.m * p.n,
                                      kernel_TFLOPs=2.0 * s * p.m * p.n / (dev_ms / 1e3) / 1e12)
            else:
                byts = 8 * p.m * p.n if not p.sparse else 12 * p.nnz
                sk["sparse_sign"] = dict(s=s, seconds=dt, embedding_host_ms=emb_ms, kernel_ms=dev_ms, bytes=byts,
                                         kernel_GBps=byts / (dev_ms / 1e3) / 1e9)
            if kind == apc.SketchKind.sparse_sign:
                steps = []
                for st in range(args.steps):
                    t1 = time.time()
                    added, _ = cur.augment()
                    t2 = time.time()
                    cur.refresh()
                    ctx.sync()
                    steps.append(dict(added=added, augment_s=t2 - t1, refresh_s=time.time() - t2, rho=cur.rho()))
                I, J = cur.indices()
                rec["cur_gpu"] = dict(steps=steps, I_head=I[:10].tolist(), J_head=J[:10].tolist(),
                                      rho=cur.rho_history().tolist())
                gpu_I, gpu_J, gpu_rho = I, J, cur.rho_history()
            cur.close()
        rec["sketch"] = sk
        print(json.dumps(rec), flush=True)
        if not args.gpu_only:
            from oracle import ref

            rp = ref.Problem.from_apc(p)
            t0 = time.time()
            r = ref.cur_steps(rp, block, 1, args.steps)
            rec["cur_ref_s"] = time.time() - t0
            rec["cur_parity"] = dict(I=bool(np.array_equal(r["I"], gpu_I)), J=bool(np.array_equal(r["J"], gpu_J)),
                                     rho=bool(np.array_equal(r["rho"].view(np.uint64), gpu_rho.view(np.uint64))))
            t0 = time.time()
            sec = ref.time_op_pair(rp, 2)
            rec["ref_op_pair_s"] = sec
            print(json.dumps(rec), flush=True)
        (out_dir / f"configs_{c}.json").write_text(json.dumps(rec, indent=1))
        A.free()
        del p
    ctx.close()


if __name__ == "__main__":
    main()
