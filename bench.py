"""APLICUR hot-path benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], "C2"): sparse fp64 200000 x 20000,
10 nonzeros per row + one per empty column, column scales 10^-U(0,4),
b ~ N(0,1), mu = 1e-6, sparse-sign sketch k = 50 (block 50, s = 56, xi = 8),
eps_lsqr = 1e-8, eps_cur = 30 mu, max_rank = 200,
seeded synthetic data (problem seed 20260417, solver seed 1).

One step = one full aplicur_solve (sketch + incremental CUR + preconditioner
rebuilds + warm-started LSQR phases to tolerance) with A resident in HBM.
value = time-to-tol in seconds (lower is better).  `e2e` is the same solve
through the C-ABI from HOST buffers (CSC upload + b in, x out, every step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "APLICUR time-to-tol (s), LSQR iter/s, A·v+Aᵀu HBM GB/s vs peak"
CONFIG_ID = 2
SOLVER = dict(mu=1e-6, block=50, eps_lsqr=1e-8, max_rank=200, seed=1, trace_sample_stride=0)


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "fallback": True}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """Reference arm: the unmodified C++ reference (oracle/_ref) on the host CPU."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import ref
    import paper_2604_05065_b200 as apc

    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libaplicur_ref.so not built"}))
        return
    p = apc.Problem(CONFIG_ID)
    rp = ref.Problem.from_apc(p)
    if args.warmup > 0:  # one untimed bounded sample warms caches / page-ins
        cpu_time_to_tol(ref, rp, p, sample_iters=min(50, args.ref_sample_iters))
    samples = [cpu_time_to_tol(ref, rp, p, sample_iters=args.ref_sample_iters) for _ in range(max(1, args.steps))]
    per_step = samples[-1]
    v = float(np.mean([x["value"] for x in samples]))
    out = {
        "metric": METRIC, "value": v, "unit": "s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step["sample_wall_s"] * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE C2 generator)",
        "config": {"workload": "C2 sparse 200000x20000 mu=1e-6 sparse-sign k=50 max_rank=200 tol=1e-8", **SOLVER},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "reference", "sample": per_step["sample"]},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "lsqr_iter_per_s": per_step["iter_per_s"],
    }
    print(json.dumps(out))


def hbm_operator_pair(apc, ctx, cfg_id, reps=20):
    """Live A*v + A^T*u timing on an HBM-bound BASELINE config (CUDA events on the
    library stream), against SURVEY 8(d)'s algorithmic bytes."""
    import torch

    p = apc.Problem(cfg_id)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    dev = torch.device("cuda", ctx.device)
    x = torch.randn(p.n, dtype=torch.float64, device=dev)
    y = torch.empty(p.m, dtype=torch.float64, device=dev)
    g = torch.empty(p.n, dtype=torch.float64, device=dev)
    s = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        A.apply_dev(x.data_ptr(), y.data_ptr())
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ctx.sync()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(s)
    for _ in range(reps):
        A.apply_dev(x.data_ptr(), y.data_ptr())
    ev[1].record(s)
    for _ in range(reps):
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ev[2].record(s)
    ctx.sync()
    tf = ev[0].elapsed_time(ev[1]) / reps * 1e-3
    ta = ev[1].elapsed_time(ev[2]) / reps * 1e-3
    if p.sparse:
        byts = 24 * p.nnz + 4 * (p.m + 1) + 4 * (p.n + 1) + 16 * (p.m + p.n)
    else:
        byts = 16 * p.m * p.n + 16 * (p.m + p.n)
    kernels = ("hot_permute_kernel + hot_sell_fwd_kernel (hot-relabelled SELL-32) | csr_units_kernel (tail rows of A^T) "
               "+ head_adj_kernel (row-blocked head rows, u in shared memory) + head_combine_kernel"
               if p.sparse else "dense_fwd_kernel | dense_adj_kernel")
    A.free()
    del p
    return {"fwd_us": tf * 1e6, "adj_us": ta * 1e6, "bytes": byts, "GBps": byts / (tf + ta) / 1e9,
            "kernels": kernels}


def cpu_time_to_tol(ref, rp, p, sample_iters=1200):
    """Reference aplicur_solve with lsqr_cap = sample_iters (identical sketch, CUR
    indices and preconditioners as the full run) -> measured setup + measured
    CPU s/iteration, extrapolated to the reference's own full iteration count
    (tests/golden/baseline_c2.npz when present)."""
    knobs = dict(SOLVER)
    knobs["lsqr_cap"] = sample_iters
    t0 = time.time()
    r = ref.solve(rp, p.b, knobs)
    wall = time.time() - t0
    lsqr_s = float(np.sum(r.phase_t_lsqr_ms)) / 1e3
    iters = int(np.sum(r.phase_iters))
    setup_s = wall - lsqr_s
    s_per_iter = lsqr_s / max(iters, 1)
    full_iters = None
    g = ROOT / "tests" / "golden" / f"baseline_c{CONFIG_ID}.npz"
    if g.exists():
        full_iters = int(np.load(g)["phase_iters"].sum())
        full_wall = float(np.load(g)["wall_s"])
    est = setup_s + (full_iters if full_iters else iters) * s_per_iter
    return {"value": est, "sample_wall_s": wall, "iter_per_s": 1.0 / s_per_iter,
            "sample": (f"reference aplicur_solve on C2 with lsqr_cap={sample_iters} ({iters} LSQR iterations, "
                       f"{wall:.1f}s wall, 1 thread); time-to-tol extrapolated as setup {setup_s:.2f}s + "
                       f"{full_iters if full_iters else iters} iterations x {s_per_iter * 1e3:.2f} ms"
                       + (f" (full reference run measured here: {full_wall:.0f}s)" if full_iters else ""))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample-iters", type=int, default=1200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hbm-pairs", action="store_true",
                    help="skip the live C3/C5 operator-pair measurement (HBM-bound configs) in the roofline")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2604_05065_b200 as apc

    ws, rank, local = _dist()
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    uid = None
    if ws > 1:
        obj = [apc.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = apc.Context(local, ws, rank, uid)
    p = apc.Problem(CONFIG_ID)
    cfg = apc.SolverConfig(**{k: v for k, v in SOLVER.items()})

    # row partition (balanced by nnz) -- SURVEY.md 8(e): A*v local, one NCCL
    # allreduce of [A_p^T u_p | ||u_p||^2] per LSQR iteration; the sketch / CUR
    # selection runs replicated on the full matrix
    if p.sparse:
        row_nnz = np.bincount(p.rowidx, minlength=p.m).astype(np.int64)
    else:
        row_nnz = None
    bounds = apc.partition_rows(p.m, ws, row_nnz)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    A_full = apc.DeviceMatrix.from_problem(ctx, p) if ws > 1 else None
    A = apc.DeviceMatrix.from_problem(ctx, p, r0, r1) if ws > 1 else apc.DeviceMatrix.from_problem(ctx, p)

    def solve_once(mat, full):
        return apc.aplicur_solve(mat, p.b, cfg, full=full)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ctx.sync()

    # ---- device-resident solves (value) ------------------------------------
    for _ in range(args.warmup):
        r = solve_once(A, A_full)
    barrier()
    L0 = ctx.launches
    s = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = []
    with ClockSampler(local) as clk:
        e0.record(s)
        for _ in range(args.steps):
            results.append(solve_once(A, A_full))
        e1.record(s)
        barrier()
    launches = ctx.launches - L0
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    r = results[-1]
    iters = r.lsqr_iters
    lsqr_ms = float(np.mean([x.lsqr_ms for x in results]))

    # ---- end-to-end through the C-ABI with host buffers (e2e) ----------------
    csc_bytes = 8 * (p.n + 1) + 16 * p.nnz if p.sparse else 8 * p.m * p.n
    # host CSC (full copy for the replicated CUR + this rank's shard when ws > 1) and b
    h2d = csc_bytes * (2 if ws > 1 else 1) + 8 * (r1 - r0)
    d2h = 8 * p.n
    barrier()
    t0 = time.perf_counter()
    e2e_parts = []
    for _ in range(args.steps):
        ta = time.perf_counter()
        F2 = apc.DeviceMatrix.from_problem(ctx, p) if ws > 1 else None
        A2 = apc.DeviceMatrix.from_problem(ctx, p, r0, r1) if ws > 1 else apc.DeviceMatrix.from_problem(ctx, p)
        tb = time.perf_counter()
        r2 = solve_once(A2, F2)
        tc = time.perf_counter()
        A2.free()
        if F2 is not None:
            F2.free()
        e2e_parts.append((tb - ta, tc - tb, time.perf_counter() - tc, r2.setup_ms / 1e3, r2.lsqr_ms / 1e3))
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- dominant kernels: operator pair A*v + A^T*u, CUDA events on ctx stream
    dev = torch.device("cuda", local)
    x = torch.randn(p.n, dtype=torch.float64, device=dev)
    y = torch.empty(A.mloc, dtype=torch.float64, device=dev)
    g = torch.empty(p.n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    reps = 200
    for _ in range(5):
        A.apply_dev(x.data_ptr(), y.data_ptr())
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ctx.sync()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(s)
    for _ in range(reps):
        A.apply_dev(x.data_ptr(), y.data_ptr())
    ev[1].record(s)
    for _ in range(reps):
        A.apply_dev(y.data_ptr(), g.data_ptr(), transpose=True)
    ev[2].record(s)
    ctx.sync()
    t_fwd = ev[0].elapsed_time(ev[1]) / reps * 1e-3
    t_adj = ev[1].elapsed_time(ev[2]) / reps * 1e-3
    mloc = A.mloc
    bytes_pair = 24 * p.nnz + 4 * (p.m + 1) + 4 * (p.n + 1) + 16 * (p.m + p.n)
    peaks = _peaks()
    achieved = bytes_pair / (t_fwd + t_adj) / 1e9
    # dominant kernel of the timed region: the LSQR iteration loop (one
    # persistent cooperative launch per phase); its device time comes from
    # CUDA events the library records around it on its own stream
    loop_ms = float(sum(ph.t_lsqr_device_ms for x in results for ph in x.phases))
    loop_iters = int(sum(ph.lsqr_iters for x in results for ph in x.phases))
    loop_launches = int(sum(1 for x in results for ph in x.phases if ph.lsqr_iters > 0))
    per_launch_bytes = bytes_pair * loop_iters / max(loop_launches, 1)
    loop_achieved = bytes_pair * loop_iters / (loop_ms / 1e3) / 1e9 if loop_ms > 0 else 0.0
    hbm = peaks.get("hbm_gbs", 6650.0)
    # DRAM bytes per iteration of lsqr_persistent_kernel from one `ncu --set full`
    # capture (profiles/r1_ncu_persistent_c2.txt: 52.06 MB read + 0.73 MB written
    # over a 300-iteration launch), scaled to this run's average launch
    dram_per_iter = (52058368 + 733952) / 300.0
    roofline = {"bound": "hbm", "achieved": loop_achieved, "peak": hbm, "unit": "GB/s",
                "frac": loop_achieved / hbm,
                "traffic": dram_per_iter * loop_iters / max(loop_launches, 1),
                "traffic_note": "ncu DRAM bytes per launch (per-iteration figure x iterations per launch): far "
                                "below the algorithmic bytes because A, A^T and every vector stay in L2",
                "kernel": "lsqr_persistent_kernel (whole LSQR phase: A*z + A^T*u + preconditioner + updates)",
                "algorithmic_bytes_per_launch": per_launch_bytes,
                "algorithmic_bytes_per_iteration": bytes_pair, "iterations": loop_iters,
                "avg_launch_ms": loop_ms / max(loop_launches, 1), "us_per_iteration": 1e3 * loop_ms / max(loop_iters, 1),
                "operator_pair": {"kernels": "csr_fwd_kernel + csr_units_kernel (standalone)",
                                  "GBps": achieved, "frac": achieved / hbm, "fwd_us": t_fwd * 1e6,
                                  "adj_us": t_adj * 1e6},
                "note": "C2's CSR pair (52.4 MB) is L2-resident on B200 (126 MB L2): the loop is latency-bound, not "
                        "HBM-bound; the HBM-bound operator numbers (C3/C4/C5) are in profiles/r1_summary.md",
                "peak_source": "MEASURED_PEAKS.json" if "fallback" not in peaks else "fallback"}

    if rank == 0 and ws == 1 and not args.no_hbm_pairs:
        # the C2 loop is L2-resident; the HBM roofline of the same operator
        # kernels is measured live on the HBM-bound configs
        pairs = {}
        for cid, name in ((3, "C3 dense 100000x10000"), (5, "C5 sparse 8e6x4e5 nnz 1.28e8")):
            try:
                d = hbm_operator_pair(apc, ctx, cid)
                d["frac"] = d["GBps"] / hbm
                pairs[name] = d
            except Exception as e:  # reported, never required
                pairs[name] = {"unavailable": str(e)}
        roofline["hbm_operator_pairs"] = pairs

    out = {
        "metric": METRIC, "value": ms_per_step / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE C2 generator; inputs larger than nothing: A is L2-resident, "
                "each step is a full solve from x = 0)",
        "config": {"workload": "C2 sparse 200000x20000 mu=1e-6 sparse-sign k=50 max_rank=200 tol=1e-8",
                   "m": p.m, "n": p.n, "nnz": p.nnz, **SOLVER, "parallelism": f"rows{ws}",
                   "l2": "no flush between steps; every step re-runs the full solve"},
        "lsqr_iters": iters, "lsqr_iter_per_s": iters / (lsqr_ms / 1e3) if lsqr_ms > 0 else None,
        "final_relres": r.final_relres, "rank": int(len(r.row_indices)), "phases": len(r.phases),
        "setup_ms": float(np.mean([x.setup_ms for x in results])), "lsqr_ms": lsqr_ms,
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "upload_s": float(np.mean([x[0] for x in e2e_parts])),
                "solve_wall_s": float(np.mean([x[1] for x in e2e_parts])),
                "free_s": float(np.mean([x[2] for x in e2e_parts])),
                "solve_setup_s": float(np.mean([x[3] for x in e2e_parts])),
                "solve_lsqr_s": float(np.mean([x[4] for x in e2e_parts]))},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref

            if ref.available():
                rp = ref.Problem.from_apc(p)
                cb = cpu_time_to_tol(ref, rp, p, sample_iters=args.ref_sample_iters)
                out["cpu_baseline"] = {"value": cb["value"], "unit": "s", "cores": 1, "kind": "reference",
                                       "sample": cb["sample"], "lsqr_iter_per_s": cb["iter_per_s"]}
        except Exception as e:  # the baseline is reported, never required
            out["cpu_baseline"] = {"value": None, "unit": "s", "cores": 1, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(out))
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
