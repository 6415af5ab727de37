"""The experiment driver (paper_2604_05065_b200/experiment.py) against the
reference's bench.hpp contract: config parsing and validation messages
(bench.hpp:30-238, CPU), and a GPU run of a Matrix Market problem: one record
JSON + trace CSV per (method, trial) cell, summary.json with medians
(bench.hpp:331-407)."""
import json

import numpy as np
import pytest

from paper_2604_05065_b200 import ApcError
from paper_2604_05065_b200.experiment import ExperimentConfig, MethodSpec, ProblemSpec, _median


def test_parse_defaults_match_bench_hpp():
    m = MethodSpec.parse({"method": "aplicur-sf", "block": 8})
    assert m.name == "aplicur-sf" and int(m.config.variant) == 1
    assert (m.config.eps_cur, m.config.eps_lsqr, m.config.nu_prec, m.config.nu_lsqr) == (-1.0, 1e-10, 10.0, 100.0)
    assert (m.config.sketch_xi, m.config.probe_count, m.config.lsqr_cap, m.config.max_rank) == (8, 10, 0, 0)
    assert not m.mu_overridden and MethodSpec.parse({"method": "lsqr", "mu": 0.1}).mu_overridden
    c = ExperimentConfig.parse({"problem": {"kind": "files", "matrix": "a.mtx", "rhs": "b.mtx"},
                                "methods": [{"method": "lsqr"}], "metrics": {"true_residual_stride": 3}})
    assert c.trials == 1 and c.seed_base == 0 and c.output_dir == "out" and c.true_residual_stride == 3
    assert ProblemSpec.parse({"kind": "baseline", "config": 2}).to_json() == {"kind": "baseline", "config": 2, "mu": 0.0}


@pytest.mark.parametrize("cfg,msg", [
    ({"problem": {"kind": "files", "matrix": "a", "rhs": "b"}, "methods": []}, "methods must be a nonempty array"),
    ({"problem": {"kind": "files", "matrix": "a", "rhs": "b"}, "methods": [{"method": "cg"}]},
     "method: must be aplicur, aplicur-sf or lsqr"),
    ({"problem": {"kind": "files", "matrix": "a", "rhs": "b"}, "methods": [{"method": "lsqr", "bogus": 1}]},
     "method: unknown key 'bogus'"),
    ({"problem": {"kind": "files", "matrix": "a", "rhs": "b"}, "methods": [{"method": "lsqr"}], "x": 1},
     "config: unknown key 'x'"),
    ({"problem": {"kind": "files", "matrix": "a", "rhs": "b"}, "methods": [{"method": "lsqr"}], "trials": 0},
     "config: trials >= 1"),
    ({"problem": {"kind": "files", "matrix": "a", "rhs": "b"}, "methods": [{"method": "lsqr", "core": "svd"}]},
     "method: core must be qr or lu"),
])
def test_parse_errors(cfg, msg):
    with pytest.raises(ApcError, match=msg):
        ExperimentConfig.parse(cfg)


def test_median():
    assert _median([]) == 0.0 and _median([3.0, 1.0, 2.0]) == 2.0 and _median([4.0, 1.0, 2.0, 3.0]) == 2.5


@pytest.mark.gpu
def test_run_experiment_files_problem(apc, ctx, tmp_path):
    from paper_2604_05065_b200.experiment import run_experiment

    p = apc.Problem(2, 4000, 400)
    apc.write_matrix_market(tmp_path / "a.mtx", p)
    apc.write_matrix_market(tmp_path / "b.mtx", p.b.reshape(-1, 1))
    cfg = ExperimentConfig.parse({
        "problem": {"kind": "files", "matrix": str(tmp_path / "a.mtx"), "rhs": str(tmp_path / "b.mtx"), "mu": 1e-3},
        "methods": [{"method": "aplicur", "name": "ap", "block": 8, "max_rank": 40, "eps_lsqr": 1e-10},
                    {"method": "lsqr", "eps_lsqr": 1e-10}],
        "trials": 3, "seed_base": 5, "output_dir": str(tmp_path / "out")})
    s = run_experiment(cfg, ctx)
    out = tmp_path / "out"
    assert json.loads((out / "summary.json").read_text()) == s
    assert [m["method"] for m in s["methods"]] == ["ap", "lsqr"] and s["trials"] == 3
    for m in s["methods"]:
        recs = [json.loads((out / f).read_text()) for f in m["records"]]
        assert [r["trial"] for r in recs] == [0, 1, 2] and [r["seed"] for r in recs] == [5, 6, 7]
        assert m["median_final_relres"] == sorted(r["final_relres"] for r in recs)[1]
        assert m["median_system_matvecs"] == sorted(float(r["system_matvecs"]) for r in recs)[1]
        for r in recs:
            assert (out / r["trace"]).exists()  # report_io.hpp:101
            assert r["optimal_relres"] == 0.0 and r["final_relres_plain"] > 0.0
            assert {"method", "trial", "seed", "wall_ms", "status", "phases", "config"} <= set(r)
    # the same solve through the API: the cell's record holds its numbers
    r0 = apc.aplicur_solve(apc.DeviceMatrix.from_problem(ctx, p), p.b,
                           apc.SolverConfig(mu=1e-3, block=8, max_rank=40, eps_lsqr=1e-10, seed=5,
                                            trace_sample_stride=1))
    rec0 = json.loads((out / "record_ap_0.json").read_text())
    assert rec0["final_relres"] == r0.final_relres and rec0["system_matvecs"] == r0.system_matvecs
