"""Formats around the path, host-only: Matrix Market
write/read against the reference's own reader/writer (oracle/_ref, compiled
from matrix_market.hpp), the trace CSV and the solve report JSON layout of
report_io.hpp.  No GPU needed."""
import json

import numpy as np
import pytest


def _csc(rng, m, n, per_col):
    rows = [np.sort(rng.choice(m, per_col, replace=False)) for _ in range(n)]
    colptr = np.arange(0, (n + 1) * per_col, per_col, dtype=np.int64)
    return colptr, np.concatenate(rows).astype(np.int64), rng.standard_normal(n * per_col)


def test_mm_sparse_write_matches_reference_bytes(apc, ref, tmp_path):
    rng = np.random.default_rng(0)
    m, n = 50, 12
    cp, ri, va = _csc(rng, m, n, 4)
    va[3] = 1e-300
    va[7] = -0.1
    ours, theirs = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    apc.write_matrix_market(ours, (m, n, cp, ri, va))
    ref.mm_write(ref.Problem(m, n, colptr=cp, rowidx=ri, vals=va), theirs)
    assert ours.read_bytes() == theirs.read_bytes()


def test_mm_dense_write_matches_reference_bytes(apc, ref, tmp_path):
    A = np.random.default_rng(1).standard_normal((7, 5))
    A[2, 3] = 0.0
    ours, theirs = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    apc.write_matrix_market(ours, A)
    ref.mm_write(ref.Problem(7, 5, dense=np.asfortranarray(A).reshape(-1, order="F")), theirs)
    assert ours.read_bytes() == theirs.read_bytes()


def test_mm_read_matches_reference(apc, ref, tmp_path):
    # unsorted entries, comments, blank lines, an explicit zero (dropped), integer field
    text = ("%%MatrixMarket matrix coordinate integer general\n% a comment\n\n4 3 5\n"
            "3 2 7\n1 1 -2\n4 3 0\n2 1 5\n  1 3 9\n")
    f = tmp_path / "a.mtx"
    f.write_text(text)
    r = ref.mm_read(f)
    p = apc.read_matrix_market(f)
    assert (p.m, p.n, p.sparse) == (r["m"], r["n"], True)
    assert np.array_equal(p.colptr, r["colptr"])
    assert np.array_equal(p.rowidx, r["rowidx"])
    assert np.array_equal(p.vals, r["vals"])
    assert np.array_equal(p.b, np.zeros(4))


def test_mm_dense_read_multiple_values_per_line(apc, ref, tmp_path):
    f = tmp_path / "d.mtx"
    f.write_text("%%MatrixMarket matrix array real general\n2 3\n1 2\n3\n4 5 6\n")
    r = ref.mm_read(f)
    p = apc.read_matrix_market(f)
    assert not p.sparse and np.array_equal(p.dense, r["dense"])


def test_mm_roundtrip_bit_exact(apc, tmp_path):
    rng = np.random.default_rng(2)
    m, n = 300, 40
    cp, ri, va = _csc(rng, m, n, 9)
    va *= np.exp(rng.uniform(-600, 600, va.size))  # extreme exponents survive %.17g
    f = tmp_path / "r.mtx"
    apc.write_matrix_market(f, (m, n, cp, ri, va))
    p = apc.read_matrix_market(f)
    assert np.array_equal(p.colptr, cp) and np.array_equal(p.rowidx, ri)
    assert np.array_equal(p.vals.view(np.uint64), va.view(np.uint64))


@pytest.mark.parametrize("text,code", [
    ("", 9),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1\n", 9),
    ("%%MatrixMarket matrix coordinate real symmetric\n1 1 1\n1 1 1\n", 9),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", 9),        # truncated
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", 1),        # out of range
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n", 1),  # duplicate
    ("%%MatrixMarket matrix array real general\n1 2\n1 2 3\n", 9),             # too many values
])
def test_mm_read_errors_match_reference(apc, ref, tmp_path, text, code):
    f = tmp_path / "bad.mtx"
    f.write_text(text)
    with pytest.raises(apc.ApcError) as e:
        apc.read_matrix_market(f)
    assert e.value.code == code
    with pytest.raises(RuntimeError, match=f"reference error {code}"):
        ref.mm_read(f)


def _fake_result(apc):
    T = np.dtype([("phase", "<i4"), ("pad", "<i4"), ("iter", "<i8"), ("phibar", "<f8"), ("cvgrate", "<f8"),
                  ("cvgdiff", "<f8"), ("matvecs", "<u8"), ("wall_ms", "<f8"), ("true_relres", "<f8")])
    tr = np.zeros(5, dtype=T)
    tr["phase"] = [1, 1, 2, 2, 2]
    tr["iter"] = [0, 1, 0, 1, 2]
    tr["phibar"] = [1.0, 0.5, 0.5, 0.25, 0.125]
    tr["matvecs"] = [1, 3, 1, 3, 5]
    tr["wall_ms"] = [0.0, 0.1, 0.2, 0.3, 0.4]
    tr["true_relres"] = [np.nan, np.nan, 0.5, np.nan, np.nan]
    ph = [apc.PhaseReport(1, 50, 3.5, 2.0, 1e-6, 1, apc.StopReason.dynamic_rate, 1.0, 2.0, 3.0, 4.0, 0.9),
          apc.PhaseReport(2, 100, 1.5, 1.0, 1e-6, 2, apc.StopReason.gradient_tol, 1.5, 2.5, 3.5, 4.5, 0.1)]
    return apc.SolveResult(np.zeros(3), ph, tr, apc.SolveStatus.rank_exhausted, 1.5, 0.1, 4, 17,
                           np.array([3, 1], dtype=np.int64), np.array([0, 2], dtype=np.int64),
                           np.array([3.5, np.inf]))


def test_trace_csv_layout(apc, tmp_path):
    r = _fake_result(apc)
    f = tmp_path / "t.csv"
    r.write_trace_csv(f)
    lines = f.read_text().splitlines()
    assert lines[0] == "phase,iter,phibar,relres,matvecs,wall_ms,reason"
    assert lines[1] == "1,0,1,,1,0,"
    assert lines[2] == "1,1,0.5,,3,0.10000000000000001,dynamic-rate"
    assert lines[3] == "2,0,0.5,0.5,1,0.20000000000000001,"
    assert lines[5] == "2,2,0.125,,5,0.40000000000000002,gradient-tol"
    assert not (tmp_path / "t.csv.tmp").exists()


def test_report_json_layout(apc, tmp_path):
    r = _fake_result(apc)
    f = tmp_path / "r.json"
    cfg = apc.SolverConfig(block=50, mu=1e-6, eps_lsqr=1e-8, seed=7)
    r.write_report_json(f, cfg, "t.csv")
    j = json.loads(f.read_text())
    assert set(j) == {"config", "status", "final_relres", "final_rho", "sketch_applications", "system_matvecs",
                      "trace", "cur", "phases"}
    assert j["status"] == "rank-exhausted" and j["trace"] == "t.csv" and j["system_matvecs"] == 17
    assert j["config"]["variant"] == "svd" and j["config"]["core"] == "qr" and j["config"]["seed"] == 7
    assert j["cur"] == {"row_indices": [3, 1], "col_indices": [0, 2], "rho_history": [3.5, None]}
    assert j["phases"][1]["reason"] == "gradient-tol"
    assert j["phases"][0]["wall_ms"] == {"augment": 1.0, "factor": 2.0, "precond": 3.0, "lsqr": 4.0}


def test_drop_in_header_formats(tmp_path):
    import subprocess
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_2604_05065_b200" / "_lib"
    exe = tmp_path / "io_main"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{root / 'include'}", str(root / "tests" / "cpp" / "io_main.cpp"),
                    "-o", str(exe), f"-L{lib}", "-lapc_b200", f"-Wl,-rpath,{lib}"], check=True)
    out = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.splitlines() == ["phase,iter,phibar,relres,matvecs,wall_ms,reason", "1,0,1,,1,0,",
                                       "1,1,0.5,,3,0.25,iteration-cap"]
    j = json.loads((tmp_path / "r.json").read_text())
    assert j["status"] == "rank-exhausted" and j["cur"]["row_indices"] == [3, 1]
    assert (tmp_path / "a.mtx").read_text().splitlines()[1] == "4 3 4"
