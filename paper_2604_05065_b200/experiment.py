"""Experiment driver of the reference (/root/reference/proj/include/aplicur/bench.hpp:
ProblemSpec / MethodSpec / ExperimentConfig parse, run_single, run_experiment)
on the B200 solver: every (method, trial) cell is solved, its trace CSV and
record JSON written, and a summary JSON aggregates medians across trials.

Differences from the reference, all outside the hot path (SURVEY.md section 2
marks the harness out of scope; this is the thin layer a user of the
reference's experiment configs needs):
  * problems: kind "files" (Matrix Market matrix + m x 1 rhs, the reference's
    own reader rules) as in bench.hpp:140-148, plus kind "baseline" (the
    BASELINE.json configs of this repo's generator).  The reference's
    synthetic generator (problems.hpp spectra / coherence) is not rebuilt:
    kind "generate" raises invalid_argument;
  * the oracle residuals (compute_oracle_residuals, a dense SVD) are not
    computed, so optimal_relres is 0.0 -- the reference's value_or(0.0) when
    the meta field is absent (bench.hpp:303-304);
  * cells run one after another on the GPU (the reference's thread pool,
    bench.hpp:353-371, serves CPU cores).
Record JSON = solve_report_to_json (report_io.hpp:94-110, the library's own
writer) plus the run_record_to_json fields (bench.hpp:244-256); keys sorted,
as nlohmann::json's std::map order.
"""
from __future__ import annotations

import json
import os
import tempfile
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np

from . import (ApcError, Context, DeviceMatrix, PrecondVariant, Problem, SolverConfig, aplicur_solve,
               plain_lsqr_solve, read_matrix_market)

_INVALID = 2  # APC_INVALID_ARGUMENT


def _require(ok: bool, msg: str) -> None:
    if not ok:
        raise ApcError(_INVALID, msg)


def _check_keys(j, allowed, ctx: str) -> None:  # bench.hpp:30-42
    _require(isinstance(j, dict), f"{ctx}: expected an object")
    for k in j:
        _require(k in allowed, f"{ctx}: unknown key '{k}'")


@dataclass
class ProblemSpec:  # bench.hpp:51-139 (files / baseline)
    kind: str = "files"
    matrix_path: str = ""
    rhs_path: str = ""
    config: int = 0
    mu: float = 0.0

    @staticmethod
    def parse(j) -> "ProblemSpec":
        kind = j.get("kind", "generate") if isinstance(j, dict) else "generate"
        if kind == "files":
            _check_keys(j, ("kind", "matrix", "rhs", "mu"), "problem")
            return ProblemSpec("files", str(j["matrix"]), str(j["rhs"]), 0, float(j.get("mu", 0.0)))
        if kind == "baseline":
            _check_keys(j, ("kind", "config", "mu"), "problem")
            return ProblemSpec("baseline", config=int(j["config"]), mu=float(j.get("mu", 0.0)))
        _require(kind != "generate", "problem: the problems.hpp generator is not part of this build; "
                                     "use kind 'files' or 'baseline'")
        raise ApcError(_INVALID, "problem: kind must be 'generate' or 'files'")

    def to_json(self) -> dict:
        if self.kind == "files":
            return {"kind": "files", "matrix": self.matrix_path, "rhs": self.rhs_path, "mu": self.mu}
        return {"kind": "baseline", "config": self.config, "mu": self.mu}

    def build(self):
        """(A as a Problem with CSC/dense arrays, b)"""
        if self.kind == "files":
            a = read_matrix_market(self.matrix_path)
            bm = read_matrix_market(self.rhs_path)
            _require(bm.n == 1 and bm.m == a.m, "problem: rhs must be an m x 1 matrix")
            return a, np.asarray(bm.to_numpy(), dtype=np.float64).reshape(-1)
        p = Problem(self.config)
        return p, np.asarray(p.b, dtype=np.float64)


@dataclass
class MethodSpec:  # bench.hpp:171-206
    name: str
    method: str
    config: SolverConfig
    mu_overridden: bool = False

    @staticmethod
    def parse(j) -> "MethodSpec":
        _check_keys(j, ("name", "method", "block", "eps_cur", "eps_lsqr", "nu_prec", "nu_lsqr", "mu", "xi",
                        "probes", "lsqr_cap", "core", "max_rank"), "method")
        method = j["method"]
        _require(method in ("aplicur", "aplicur-sf", "lsqr"), "method: must be aplicur, aplicur-sf or lsqr")
        core = j.get("core", "qr")
        _require(core in ("qr", "lu"), "method: core must be qr or lu")
        cfg = SolverConfig(variant=int(PrecondVariant.svd_free if method == "aplicur-sf" else PrecondVariant.svd),
                           block=int(j.get("block", 0)), eps_cur=float(j.get("eps_cur", -1.0)),
                           eps_lsqr=float(j.get("eps_lsqr", 1e-10)), nu_prec=float(j.get("nu_prec", 10.0)),
                           nu_lsqr=float(j.get("nu_lsqr", 100.0)), sketch_xi=int(j.get("xi", 8)),
                           probe_count=int(j.get("probes", 10)), lsqr_cap=int(j.get("lsqr_cap", 0)),
                           max_rank=int(j.get("max_rank", 0)), core=0 if core == "qr" else 1)
        over = "mu" in j
        if over:
            cfg.mu = float(j["mu"])
        return MethodSpec(str(j.get("name", method)), method, cfg, over)


@dataclass
class ExperimentConfig:  # bench.hpp:208-238
    problem: ProblemSpec
    methods: list
    trials: int = 1
    seed_base: int = 0
    output_dir: str = "out"
    true_residual_stride: int = 0

    @staticmethod
    def parse(j) -> "ExperimentConfig":
        _check_keys(j, ("problem", "methods", "trials", "seed_base", "output_dir", "metrics"), "config")
        _require(isinstance(j.get("methods"), list) and len(j["methods"]) > 0,
                 "config: methods must be a nonempty array")
        c = ExperimentConfig(ProblemSpec.parse(j["problem"]), [MethodSpec.parse(m) for m in j["methods"]],
                             int(j.get("trials", 1)), int(j.get("seed_base", 0)), str(j.get("output_dir", "out")))
        _require(c.trials >= 1, "config: trials >= 1")
        if "metrics" in j:
            _check_keys(j["metrics"], ("true_residual_stride", "dump_spectrum"), "metrics")
            c.true_residual_stride = int(j["metrics"].get("true_residual_stride", 0))
        return c


def _median(v):  # bench.hpp:276-282
    if not v:
        return 0.0
    v = sorted(v)
    h = len(v) // 2
    return v[h] if len(v) % 2 else 0.5 * (v[h - 1] + v[h])


def _atomic_write(path: Path, text: str) -> None:  # report_io.hpp atomic_write: tmp + rename
    tmp = path.with_name(path.name + ".tmp")
    tmp.write_text(text)
    os.replace(tmp, path)


@dataclass
class RunRecord:  # bench.hpp:226-240
    method: str
    trial: int
    seed: int
    final_relres: float
    optimal_relres: float
    final_relres_plain: float
    status: str
    system_matvecs: int
    sketch_applications: int
    wall_ms: float
    trace_file: str
    phases: list = field(default_factory=list)


_STATUS = {0: "converged", 1: "rank-exhausted", 2: "breakdown"}  # solver.hpp:92-99


def run_single(A: DeviceMatrix, b: np.ndarray, mu: float, method: MethodSpec, trial: int, seed: int, stride: int,
               outdir: Path) -> RunRecord:
    """bench.hpp:286-327: one (method, trial) cell -> trace CSV + record JSON."""
    t0 = time.perf_counter()
    cfg = SolverConfig(**{k: getattr(method.config, k) for k in method.config.__dataclass_fields__})
    if not method.mu_overridden:
        cfg.mu = mu
    cfg.seed = seed
    cfg.trace_sample_stride = stride
    r = plain_lsqr_solve(A, b, cfg) if method.method == "lsqr" else aplicur_solve(A, b, cfg)
    # plain relative residual ||A x - b|| / ||b|| on the device (detail::plain_relres)
    ax = A.apply(r.x)
    plain = float(np.linalg.norm(ax - b) / np.linalg.norm(b)) if np.linalg.norm(b) > 0 else 0.0
    optimal = 0.0  # no oracle residuals (compute_oracle_residuals is out of scope)
    _require(r.final_relres >= optimal - 1e-12, "run record: relative residual below the optimal oracle")
    trace_file = f"trace_{method.name}_{trial}.csv"
    r.write_trace_csv(outdir / trace_file)
    with tempfile.TemporaryDirectory() as td:
        rp = Path(td) / "report.json"
        r.write_report_json(rp, cfg, trace_file)
        rec_json = json.loads(rp.read_text())
    wall = (time.perf_counter() - t0) * 1e3
    rec = RunRecord(method.name, trial, seed, r.final_relres, optimal, plain,
                    _STATUS.get(int(r.status), str(int(r.status))), r.system_matvecs, r.sketch_applications,
                    wall, trace_file, r.phases)
    rec_json.update({"method": rec.method, "trial": trial, "seed": seed, "final_relres": rec.final_relres,
                     "optimal_relres": optimal, "final_relres_plain": plain, "wall_ms": wall})
    _atomic_write(outdir / f"record_{method.name}_{trial}.json", json.dumps(rec_json, indent=2, sort_keys=True) + "\n")
    return rec


def run_experiment(cfg: ExperimentConfig, ctx: Optional[Context] = None) -> dict:
    """bench.hpp:331-407: every (method, trial) cell, then summary.json with
    medians across trials."""
    out = Path(cfg.output_dir)
    out.mkdir(parents=True, exist_ok=True)
    own = ctx is None
    ctx = ctx or Context(0)
    try:
        prob, b = cfg.problem.build()
        A = DeviceMatrix.from_problem(ctx, prob)
        stride = cfg.true_residual_stride or (1 if prob.m * prob.n <= 1_000_000 else 10)
        records = []
        for mi, m in enumerate(cfg.methods):
            for t in range(cfg.trials):
                records.append((mi, run_single(A, b, cfg.problem.mu, m, t, cfg.seed_base + t, stride, out)))
        A.free()
        summary = {"problem": cfg.problem.to_json(), "optimal_relres_unreg": 0.0, "optimal_relres_reg": 0.0,
                   "trials": cfg.trials, "methods": []}
        for mi, m in enumerate(cfg.methods):
            rs = [r for k, r in records if k == mi]
            summary["methods"].append({
                "method": m.name,
                "median_final_relres": _median([r.final_relres for r in rs]),
                "median_system_matvecs": _median([float(r.system_matvecs) for r in rs]),
                "median_wall_ms": _median([r.wall_ms for r in rs]),
                "records": [f"record_{r.method}_{r.trial}.json" for r in rs]})
        _atomic_write(out / "summary.json", json.dumps(summary, indent=2, sort_keys=True) + "\n")
        return summary
    finally:
        if own:
            ctx.close()


def main(argv=None) -> int:
    """python -m paper_2604_05065_b200.experiment CONFIG.json (the reference CLI's `run` command)"""
    import sys

    argv = sys.argv[1:] if argv is None else argv
    cfg = ExperimentConfig.parse(json.loads(Path(argv[0]).read_text()))
    print(json.dumps(run_experiment(cfg), indent=2, sort_keys=True))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
