"""Large-CSR operator paths: the hot-relabelled SELL-32 forward (HotSell,
ops.cuh `hot_sell_fwd_kernel`, A*x gathering x by columns renumbered by
descending nnz count) and the row-blocked head adjoint (HeadAdj, ops.cu
`head_adj_kernel`, A^T*u of the long rows of A^T with u staged in shared
memory, the rest through work units).  Both are built at upload when the
CSR is HBM-streamed (12 nnz > 96 MB); APC_HOT_SELL=1 forces them on the small matrices here so their
results can be checked against the reference Matrix::matvec /
matvec_transpose (matrix.hpp:151-195) with the componentwise summation bound,
and whole solves against the default CSR path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -53


def _upload(apc, ctx, p, monkeypatch, on):
    monkeypatch.setenv("APC_HOT_SELL", "1" if on else "0")
    return apc.DeviceMatrix.from_problem(ctx, p)


@pytest.mark.parametrize("cfg,m,n", [(5, 20000, 2000), (2, 20000, 2000), (5, 3001, 777), (2, 33, 40)])
@pytest.mark.parametrize("mu", [0.0, 0.25])
def test_hot_forward_vs_reference(apc, ref, ctx, monkeypatch, cfg, m, n, mu):
    monkeypatch.setenv("APC_HEAD_PARTS", "3" if mu > 0 else "2")
    p = apc.Problem(cfg, m, n)
    A = _upload(apc, ctx, p, monkeypatch, True)
    rp = ref.Problem.from_apc(p)
    x = np.random.default_rng(m).standard_normal(n)
    aug = mu > 0
    y = A.apply(x, mu, aug, False)
    yr = ref.matvec(rp, x, mu, aug, False)
    Aabs = np.abs(p.to_numpy())
    k = (Aabs != 0).sum(axis=1).max()
    bound = 2.0 * k * EPS * (Aabs @ np.abs(x)) + 1e-300
    assert np.all(np.abs(y[:m] - yr[:m]) <= bound)
    if aug:
        assert np.array_equal(y[m:], mu * x)
    assert np.array_equal(A.apply(x, mu, aug, False), y)  # fixed order: reruns are bit-identical
    u = np.random.default_rng(m + 1).standard_normal(m + n if aug else m)
    g = A.apply(u, mu, aug, True)
    gr = ref.matvec(rp, u, mu, aug, True)
    kt = (Aabs != 0).sum(axis=0).max()
    bt = 2.0 * (kt + 1) * EPS * (Aabs.T @ np.abs(u[:m])) + (2 * EPS * mu * np.abs(u[m:]) if aug else 0) + 1e-300
    assert np.all(np.abs(g - gr) <= bt)
    assert np.array_equal(A.apply(u, mu, aug, True), g)


def test_hot_forward_ragged_and_empty_rows(apc, ref, ctx, monkeypatch):
    # rows of very different lengths (chunk padding), empty rows and columns
    rng = np.random.default_rng(7)
    m, n = 4099, 300
    cols = []
    for j in range(n):
        k = 0 if j % 37 == 0 else int(rng.integers(1, 400 if j < 5 else 30))
        r = np.sort(rng.choice(m - 50, size=k, replace=False)).astype(np.int64)  # last 50 rows empty
        cols.append(r)
    colptr = np.concatenate([[0], np.cumsum([c.size for c in cols])]).astype(np.int64)
    rowidx = np.concatenate(cols)
    vals = rng.standard_normal(rowidx.size)
    monkeypatch.setenv("APC_HOT_SELL", "1")
    A = apc.DeviceMatrix.csc(ctx, m, n, colptr, rowidx, vals)
    rp = ref.Problem(m, n, colptr=colptr, rowidx=rowidx, vals=vals)
    x = rng.standard_normal(n)
    y = A.apply(x)
    yr = ref.matvec(rp, x)
    assert np.all(y[m - 50:] == 0.0)
    assert np.allclose(y, yr, rtol=1e-13, atol=1e-13 * np.abs(yr).max())


def test_hot_solve_matches_default_path(apc, ctx, monkeypatch):
    p = apc.Problem(5, 30000, 3000)
    cfg = apc.SolverConfig(mu=1e-6, eps_lsqr=1e-8, block=20, max_rank=60, seed=1, trace_sample_stride=0)
    A0 = _upload(apc, ctx, p, monkeypatch, False)
    r0 = apc.aplicur_solve(A0, p.b, cfg)
    A0.free()
    A1 = _upload(apc, ctx, p, monkeypatch, True)
    r1 = apc.aplicur_solve(A1, p.b, cfg)
    # CUR indices never depend on the LSQR products
    assert np.array_equal(r0.row_indices, r1.row_indices)
    assert np.array_equal(r0.col_indices, r1.col_indices)
    assert abs(r1.lsqr_iters - r0.lsqr_iters) <= max(2, 0.05 * r0.lsqr_iters)
    assert abs(r1.final_relres - r0.final_relres) <= 1e-6 * max(1.0, r0.final_relres)
    # rerun through the hot path is bit-identical
    r2 = apc.aplicur_solve(A1, p.b, cfg)
    assert np.array_equal(r2.x, r1.x)


@pytest.mark.parametrize("parts", ["1", "2", "5"])
def test_head_adjoint_blocks_and_split_tail(apc, ref, ctx, monkeypatch, parts):
    # m spans 37 row blocks (the last one partial); APC_HEAD_MIN=100 puts the
    # head threshold at 3700 entries: two head columns (one longer than many
    # items per block), a split tail column (3000 > one work unit), short,
    # empty and single-entry columns
    rng = np.random.default_rng(11)
    m = 300001
    lens = [150000, 3000, 20, 0, 8000, 1, 0, 3699, 3700]
    cols = [np.sort(rng.choice(m, size=k, replace=False)).astype(np.int64) for k in lens]
    colptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    rowidx = np.concatenate(cols)
    vals = rng.standard_normal(rowidx.size)
    monkeypatch.setenv("APC_HOT_SELL", "1")
    monkeypatch.setenv("APC_HEAD_MIN", "100")
    monkeypatch.setenv("APC_HEAD_PARTS", parts)
    A = apc.DeviceMatrix.csc(ctx, m, len(lens), colptr, rowidx, vals)
    rp = ref.Problem(m, len(lens), colptr=colptr, rowidx=rowidx, vals=vals)
    u = rng.standard_normal(m)
    g = A.apply(u, transpose=True)
    gr = ref.matvec(rp, u, transpose=True)
    for j, k in enumerate(lens):
        seg = slice(colptr[j], colptr[j + 1])
        bound = 2.0 * (k + 1) * EPS * float(np.abs(vals[seg]) @ np.abs(u[rowidx[seg]])) + 1e-300
        assert abs(g[j] - gr[j]) <= bound, (j, g[j], gr[j])
    assert g[3] == 0.0 and g[6] == 0.0
    assert np.array_equal(A.apply(u, transpose=True), g)
    x = rng.standard_normal(len(lens))
    assert np.allclose(A.apply(x), ref.matvec(rp, x), rtol=1e-13, atol=1e-13)


def test_hot_row_shard_products_and_sharded_entry(apc, ctx, monkeypatch):
    # a row shard builds its own hot SELL / head blocks over its local rows
    p = apc.Problem(5, 30000, 3000)
    monkeypatch.setenv("APC_HOT_SELL", "0")
    A = apc.DeviceMatrix.from_problem(ctx, p)
    monkeypatch.setenv("APC_HOT_SELL", "1")
    monkeypatch.setenv("APC_HEAD_MIN", "2")
    r0, r1 = 4321, 21000
    S = apc.DeviceMatrix.from_problem(ctx, p, r0, r1)
    x = np.random.default_rng(0).standard_normal(p.n)
    np.testing.assert_allclose(S.apply(x), A.apply(x)[r0:r1], rtol=1e-12, atol=1e-14)
    u = np.random.default_rng(1).standard_normal(r1 - r0)
    full_u = np.zeros(p.m)
    full_u[r0:r1] = u
    np.testing.assert_allclose(S.apply(u, transpose=True), A.apply(full_u, transpose=True), rtol=1e-11, atol=1e-13)
    # single-rank sharded entry over the hot layout agrees with the default path
    H = apc.DeviceMatrix.from_problem(ctx, p)
    cfg = apc.SolverConfig(mu=1e-6, eps_lsqr=1e-8, block=20, max_rank=40, seed=1, trace_sample_stride=0)
    g0 = apc.aplicur_solve(A, p.b, cfg)
    g1 = apc.aplicur_solve(H, p.b, cfg, full=H)
    assert np.array_equal(g0.row_indices, g1.row_indices)
    assert abs(g1.lsqr_iters - g0.lsqr_iters) <= max(2, 0.05 * g0.lsqr_iters)


def test_hot_solve_matches_reference(apc, ref, ctx, monkeypatch):
    # the whole adaptive solve through the hot SELL forward and the head adjoint
    # (forced on a C5-shaped system) against the unmodified reference solver
    monkeypatch.setenv("APC_HOT_SELL", "1")
    monkeypatch.setenv("APC_HEAD_MIN", "2")
    p = apc.Problem(5, 30000, 3000)
    knobs = dict(mu=1e-8, eps_lsqr=1e-8, block=25, seed=1, max_rank=50, eps_cur=3e-7)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    g = apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs))
    r = ref.solve(ref.Problem.from_apc(p), p.b, dict(knobs, trace_sample_stride=0))
    assert np.array_equal(g.row_indices, r.row_indices)
    assert np.array_equal(g.col_indices, r.col_indices)
    assert np.array_equal(g.rho_history.view(np.uint64), r.rho_history.view(np.uint64))
    assert [ph.rank for ph in g.phases] == list(r.phase_rank)
    it_g, it_r = g.lsqr_iters, int(r.phase_iters.sum())
    assert abs(it_g - it_r) <= max(3, 0.05 * it_r), (it_g, it_r)
    assert abs(g.final_relres - r.final_relres) <= 1e-5 * r.final_relres


def test_fused_adjoint_epilogue_is_bit_identical(apc, ctx, monkeypatch):
    """The LSQR epilogue h = (A^T u + mu u_t)/beta applied by the tail scatter and
    the head combine (APC_FUSE_EPI=1) against the separate lsqr_epi_kernel pass
    (the default): the same operations per column, so x and the phibar
    trace are bit-identical (lsqr.hpp:139-150)."""
    p = apc.Problem(5, 60000, 6000)
    A = _upload(apc, ctx, p, monkeypatch, True)
    cfg = apc.SolverConfig(mu=1e-8, eps_lsqr=1e-8, block=25, seed=1, max_rank=50, eps_cur=3e-7, lsqr_cap=300)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("APC_FUSE_EPI", mode)
        L0 = ctx.launches
        out[mode] = (apc.aplicur_solve(A, p.b, cfg), ctx.launches - L0)
    g1, g0 = out["1"][0], out["0"][0]
    assert np.array_equal(g1.x, g0.x)
    assert np.array_equal(g1.trace["phibar"], g0.trace["phibar"])
    assert g1.lsqr_iters == g0.lsqr_iters > 0
    # the fused path launches one kernel less per preconditioned iteration
    assert out["1"][1] < out["0"][1]
    A.free()
