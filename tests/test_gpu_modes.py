"""The LSQR driver's execution modes agree: persistent cooperative kernel
(default for L2-resident sparse systems), CUDA graph with a conditional WHILE
node, host-polled graph batches (the multi-rank path, here without NCCL),
eager launches; and the sharded entry point (apc_solve_sharded) on one rank."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KNOBS = dict(mu=1e-3, eps_lsqr=1e-10, block=8, seed=3, max_rank=40, trace_sample_stride=0)


@pytest.fixture
def problem(apc, ctx):
    p = apc.Problem(2, 4000, 400)
    return p, apc.DeviceMatrix.from_problem(ctx, p)


@pytest.mark.parametrize("mode", ["while", "batch", "eager"])
def test_modes_agree_with_persistent(apc, problem, mode):
    p, A = problem
    base = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
    os.environ["APC_LSQR_MODE"] = mode
    try:
        other = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
    finally:
        del os.environ["APC_LSQR_MODE"]
    assert np.array_equal(base.row_indices, other.row_indices)
    assert abs(base.lsqr_iters - other.lsqr_iters) <= max(3, 0.05 * base.lsqr_iters)
    assert abs(base.final_relres - other.final_relres) <= 1e-3 * base.final_relres


def test_sharded_entry_single_rank(apc, ctx, problem):
    p, A = problem
    full = apc.DeviceMatrix.from_problem(ctx, p)
    g1 = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
    g2 = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS), full=full)
    assert np.array_equal(g1.row_indices, g2.row_indices)
    assert np.array_equal(g1.x, g2.x)


def test_row_shard_operator_products(apc, ref, ctx, problem):
    # a shard's A*x is the corresponding block of rows; its A^T u is the partial sum
    p, A = problem
    r0, r1 = 1000, 2500
    S = apc.DeviceMatrix.from_problem(ctx, p, r0, r1)
    x = np.random.default_rng(0).standard_normal(p.n)
    np.testing.assert_allclose(S.apply(x), A.apply(x)[r0:r1], rtol=1e-12, atol=1e-14)
    u = np.random.default_rng(1).standard_normal(r1 - r0)
    full_u = np.zeros(p.m)
    full_u[r0:r1] = u
    np.testing.assert_allclose(S.apply(u, transpose=True), A.apply(full_u, transpose=True), rtol=1e-11,
                               atol=1e-13)


# Persistent-kernel code paths (lsqr_persistent.cu), each against the CUDA-graph
# path on the same system: per-CTA vs grid-wide preconditioner projection,
# shared-memory z by TMA bulk copy vs by plain loads vs gathers from L2, odd n
# (no 16-byte bulk copy), SELL-32 vs CSR forward walk, 512 vs 1024 threads.
PERSISTENT_VARIANTS = [
    {},
    {"APC_PERSISTENT_FUSED": "0"},
    {"APC_PERSISTENT_ZSMEM": "0"},
    {"APC_PERSISTENT_SELL": "0"},
    {"APC_PERSISTENT_PT": "1024"},
    {"APC_PERSISTENT_REGS": "1"},
    {"APC_PERSISTENT_FUSED": "0", "APC_PERSISTENT_ZSMEM": "0", "APC_PERSISTENT_SELL": "0"},
]


@pytest.mark.parametrize("n", [400, 401])
@pytest.mark.parametrize("env", PERSISTENT_VARIANTS, ids=lambda e: ",".join(f"{k[15:]}={v}" for k, v in e.items()) or "default")
def test_persistent_variants_agree_with_graph(apc, ctx, env, n):
    p = apc.Problem(2, 4000, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    os.environ["APC_LSQR_MODE"] = "while"
    try:
        base = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
    finally:
        del os.environ["APC_LSQR_MODE"]
    for k, v in env.items():
        os.environ[k] = v
    try:
        other = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
        rerun = apc.aplicur_solve(A, p.b, apc.SolverConfig(**KNOBS))
    finally:
        for k in env:
            del os.environ[k]
    assert np.array_equal(base.row_indices, other.row_indices)
    assert abs(base.lsqr_iters - other.lsqr_iters) <= max(3, 0.05 * base.lsqr_iters)
    assert abs(base.final_relres - other.final_relres) <= 1e-3 * base.final_relres
    # the persistent kernel is deterministic: a rerun is bit-identical
    assert np.array_equal(other.x, rerun.x)
    assert other.lsqr_iters == rerun.lsqr_iters


@pytest.mark.parametrize("mu", [0.0, 1e-2])
def test_persistent_plain_lsqr_matches_graph(apc, ctx, mu):
    # unpreconditioned phases (S12/S56 skipped, S4 writes v_raw directly) on a
    # well-conditioned sparse system, where the two paths agree to rounding
    rng = np.random.default_rng(11)
    m, n, k = 3000, 301, 8
    rows = np.concatenate([np.sort(rng.choice(m, k, replace=False)) for _ in range(n)])
    colptr = np.arange(0, (n + 1) * k, k)
    A = apc.DeviceMatrix.csc(ctx, m, n, colptr, rows, rng.standard_normal(n * k))
    b = rng.standard_normal(m)
    cfg = apc.SolverConfig(mu=mu, eps_lsqr=1e-12, lsqr_cap=400)
    os.environ["APC_LSQR_MODE"] = "while"
    try:
        g = apc.plain_lsqr_solve(A, b, cfg)
    finally:
        del os.environ["APC_LSQR_MODE"]
    q = apc.plain_lsqr_solve(A, b, cfg)
    assert q.lsqr_iters == g.lsqr_iters
    np.testing.assert_allclose(q.x, g.x, rtol=1e-9, atol=1e-12 * np.abs(g.x).max())


def test_split_transpose_rows_all_modes(apc, ctx):
    # C5-shaped (Zipf columns): the heaviest columns exceed one 2048-entry work
    # unit, so A^T u goes through split rows (partials + op_adj_raw's fix-up);
    # every LSQR mode must see the same operator
    p = apc.Problem(5, 60000, 3000)
    assert np.diff(p.colptr).max() > 2048
    A = apc.DeviceMatrix.from_problem(ctx, p)
    knobs = dict(mu=1e-8, eps_lsqr=1e-8, block=25, seed=1, max_rank=50, trace_sample_stride=0, lsqr_cap=300)
    res = {}
    for mode in ["while", "batch", "eager"]:
        os.environ["APC_LSQR_MODE"] = mode
        try:
            res[mode] = apc.aplicur_solve(A, p.b, apc.SolverConfig(**knobs))
        finally:
            del os.environ["APC_LSQR_MODE"]
    base = res["while"]
    for mode, r in res.items():
        assert np.array_equal(r.row_indices, base.row_indices), mode
        assert abs(r.lsqr_iters - base.lsqr_iters) <= max(3, 0.05 * base.lsqr_iters), mode
        assert abs(r.final_relres - base.final_relres) <= 1e-6 * base.final_relres, mode
    # the operator itself against a host product
    u = np.random.default_rng(3).standard_normal(p.m)
    ref = np.zeros(p.n)
    for j in range(p.n):
        s, e = p.colptr[j], p.colptr[j + 1]
        ref[j] = np.dot(p.vals[s:e], u[p.rowidx[s:e]])
    np.testing.assert_allclose(A.apply(u, transpose=True), ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())


def test_fused_nspace_kernel_bit_identical(tmp_path):
    """The opt-in one-launch n-space kernel (lsqr.cu lsqr_nspace_kernel,
    APC_NSPACE=1) reproduces the unfused kernels' iterates bit for bit, for the
    implicit preconditioner and for plain LSQR (the env switch is read once per
    process, so each variant runs in its own interpreter)."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    script = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2604_05065_b200 as apc\n"
        "ctx = apc.Context(0); p = apc.Problem(5, 60000, 4000)\n"
        "A = apc.DeviceMatrix.from_problem(ctx, p)\n"
        "r = apc.aplicur_solve(A, p.b, apc.SolverConfig(mu=1e-8, block=25, max_rank=50, eps_cur=3e-7, seed=1,"
        " eps_lsqr=1e-8, lsqr_cap=300, trace_sample_stride=0))\n"
        "q = apc.plain_lsqr_solve(A, p.b, apc.SolverConfig(mu=1e-8, eps_lsqr=1e-8, lsqr_cap=200,"
        " trace_sample_stride=0))\n"
        "np.savez(sys.argv[1], x=r.x, ph=np.asarray(r.trace['phibar']), xp=q.x)\n" % str(root))
    out = {}
    for v in ("0", "1"):
        f = tmp_path / f"ns{v}.npz"
        env = dict(os.environ, APC_NSPACE=v, APC_LSQR_MODE="while", APC_HOT_SELL="1")  # graph path, hot layouts
        subprocess.run([sys.executable, "-c", script, str(f)], check=True, env=env, timeout=600)
        out[v] = np.load(f)
    for k in ("x", "ph", "xp"):
        assert np.array_equal(out["0"][k], out["1"][k]), k
