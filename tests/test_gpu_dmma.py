"""Opt-in FP64 tensor-core Gaussian sketch (SketchKind.gaussian_dmma,
mma.sync.m8n8k4.f64): Y = S A (sketch.hpp:189-192) with hardware FMA
accumulation order.  Y is not bit-identical to the reference's matmul, so the
checks are (1) Y within a rounding-level bound of the exact-order sketch and
(2) the CUR indices the incremental selection builds from it (cur.hpp:248-315)
equal the exact path's, which the reference pins (tests/golden/curg_c*.npz)."""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("cfg,m,n,block", [(1, 4000, 500, 20), (3, 3000, 500, 100), (1, 1000, 77, 7),
                                           (3, 5003, 301, 250)])
def test_dmma_sketch_close_to_exact(apc, ctx, cfg, m, n, block):
    p = apc.Problem(cfg, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    Ye = apc.CurState(A, block, seed=1, sketch=apc.SketchKind.gaussian).sketch_matrix()
    Yf = apc.CurState(A, block, seed=1, sketch=apc.SketchKind.gaussian_dmma).sketch_matrix()
    assert Ye.shape == Yf.shape
    # |Yf - Ye| <= m * eps * (|S| |A|) entrywise; bounded here through column norms
    Ad = p.dense.reshape(n, m).T
    S_abs_A = np.sqrt(m) * np.linalg.norm(Ad, axis=0)[None, :] / np.sqrt(Ye.shape[0])
    err = np.abs(Yf - Ye) / np.maximum(S_abs_A, 1e-300)
    assert err.max() <= 4 * m * 2.0 ** -53, err.max()
    assert not np.array_equal(Ye, Yf) or m < 64  # a different rounding order, not a copy of the exact path


@pytest.mark.parametrize("cfg,m,n,block,steps", [(1, 4000, 500, 20, 5), (3, 3000, 300, 25, 4), (1, 400, 50, 5, 6)])
def test_dmma_cur_indices_match_exact(apc, ctx, cfg, m, n, block, steps):
    p = apc.Problem(cfg, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    out = []
    for kind in (apc.SketchKind.gaussian, apc.SketchKind.gaussian_dmma):
        cur = apc.CurState(A, block, seed=7, sketch=kind)
        for _ in range(steps):
            added, _ = cur.augment()
            if added == 0:
                break
            cur.refresh()
        out.append(cur.indices())
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("k", [1, 3])
def test_dmma_cur_indices_baseline_size(apc, ctx, k):
    """Full-size C1 / C3 Gaussian CurState steps from the DMMA sketch select the
    reference's indices (the Gaussian-shim fixture)."""
    f = GOLD / f"curg_c{k}.npz"
    if not f.exists():
        pytest.skip(f"{f.name} not generated")
    g = np.load(f)
    meta = json.loads(str(g["meta"]))
    p = apc.Problem(k)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    try:
        cur = apc.CurState(A, meta["block"], seed=meta["seed"], sketch=apc.SketchKind.gaussian_dmma)
        for added_ref in g["added"]:
            added, _ = cur.augment()
            assert added == added_ref
            if added == 0:
                break
            cur.refresh()
        I, J = cur.indices()
        assert np.array_equal(I, g["I"]) and np.array_equal(J, g["J"])
        rho = cur.rho_history()
        np.testing.assert_allclose(rho, g["rho"][: len(rho)], rtol=1e-10)
    finally:
        A.free()


def test_dmma_solve_matches_exact_solve(apc, ctx):
    p = apc.Problem(1, 4000, 500)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    res = [apc.aplicur_solve(A, p.b, apc.SolverConfig(mu=0.0, eps_lsqr=1e-8, block=20, seed=1, max_rank=100,
                                                        sketch_kind=kind))
           for kind in (apc.SketchKind.gaussian, apc.SketchKind.gaussian_dmma)]
    assert np.array_equal(res[0].row_indices, res[1].row_indices)
    assert np.array_equal(res[0].col_indices, res[1].col_indices)
    assert [ph.rank for ph in res[0].phases] == [ph.rank for ph in res[1].phases]
    rel = np.linalg.norm(res[0].x - res[1].x) / np.linalg.norm(res[0].x)
    assert rel <= 1e-6, rel
