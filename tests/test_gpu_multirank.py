"""Row-sharded aplicur_solve through the library's own sharded entry
(apc_solve_sharded) and kernels: two or three processes share the one B200,
each owning a block of A's rows (balanced by nnz, apc_partition_rows) for the
LSQR operator.  Two setups:
 * root-only: rank 0 alone holds the whole matrix and runs the sketch, the CUR
   selection and the preconditioner builds, which reach the others by
   broadcast;
 * sharded: no rank holds the whole matrix -- the sketch is carried from rank
   to rank, E^col stays on the row blocks, the row pivots come from a
   candidate allgather per pivot, R's rows from their owners (DeviceCur
   distributed); rank 0 builds the preconditioner from the rank-summed Gram.
With the host-staged collective backend
(apc_ctx_create_host_comm) summing [A_p^T u_p | ||u_p||^2] and the residual
norms over gloo in rank order (solver.hpp:204-262,
matrix.hpp:175-195).  Against the single-rank solve: CUR indices bit-exact,
the same phases, LSQR iterations within 5%, x within 1e-6 (or the reference
sensitivity), and the two ranks' results bit-identical to each other."""
import os
import pickle
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    (2, 20000, 2000, dict(mu=1e-6, eps_lsqr=1e-8, block=20, seed=1, max_rank=60, trace_sample_stride=0)),
    (1, 4000, 500, dict(mu=0.0, eps_lsqr=1e-8, block=20, seed=1, max_rank=100, trace_sample_stride=0)),
    (5, 60000, 4000, dict(mu=1e-8, eps_lsqr=1e-8, block=25, seed=1, max_rank=50, eps_cur=3e-7,
                          trace_sample_stride=0)),
    # the Gaussian sketch (exact matmul chain) carried over the row blocks
    (1, 4000, 500, dict(mu=0.0, eps_lsqr=1e-8, block=20, seed=1, max_rank=60, trace_sample_stride=0,
                        sketch_kind=1)),
]
# (case, world, setup)
RUNS = [(c, 2, "root") for c in range(3)] + [(0, 2, "sharded"), (1, 3, "sharded"), (2, 3, "sharded"),
                                             (3, 2, "sharded")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, case, out_path, setup):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_05065_b200 as apc

    def allreduce(buf):
        # every rank adds the gathered buffers in rank order: identical bits everywhere
        t = torch.from_numpy(buf.copy())
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        acc = parts[0].numpy().copy()
        for q in parts[1:]:
            acc += q.numpy()
        buf[:] = acc

    cfg_id, m, n, knobs = case
    knobs = dict(knobs)
    if "sketch_kind" in knobs:
        knobs["sketch_kind"] = apc.SketchKind(knobs["sketch_kind"])
    ctx = apc.Context(0, world, rank, host_allreduce=allreduce)
    p = apc.Problem(cfg_id, m, n)
    row_nnz = np.bincount(p.rowidx, minlength=p.m).astype(np.int64) if p.sparse else None
    bounds = apc.partition_rows(p.m, world, row_nnz)
    # root-only: rank 0 alone holds the whole matrix (sketch, CUR,
    # preconditioner builds); sharded: every rank holds only its rows
    full = apc.DeviceMatrix.from_problem(ctx, p) if rank == 0 and setup == "root" else None
    shard = apc.DeviceMatrix.from_problem(ctx, p, int(bounds[rank]), int(bounds[rank + 1]))
    r = apc.aplicur_solve(shard, p.b, apc.SolverConfig(**knobs), full=full)
    res = dict(x=r.x, I=r.row_indices, J=r.col_indices, rho=r.rho_history, iters=[ph.lsqr_iters for ph in r.phases],
               ranks=[ph.rank for ph in r.phases], reasons=[int(ph.reason) for ph in r.phases],
               relres=r.final_relres, bounds=bounds.tolist())
    with open(f"{out_path}.{rank}", "wb") as f:
        pickle.dump(res, f)
    shard.free()
    if full is not None:
        full.free()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("run", RUNS, ids=[f"c{c}-w{w}-{s}" for c, w, s in RUNS])
def test_row_sharded_matches_single_rank(apc, ctx, tmp_path, run):
    import torch.multiprocessing as mp

    case, world, setup = run

    cfg_id, m, n, knobs = CASES[case]
    out = str(tmp_path / "res")
    mp.start_processes(_rank_main, args=(world, _free_port(), CASES[case], out, setup), nprocs=world, join=True,
                       start_method="spawn")
    rs = [pickle.load(open(f"{out}.{k}", "rb")) for k in range(world)]
    b = rs[0]["bounds"]
    assert all(b[k] < b[k + 1] for k in range(world))  # every rank owns rows
    # replicas: identical bits on every rank
    for k in range(1, world):
        assert np.array_equal(rs[0]["x"], rs[k]["x"])
        assert rs[0]["iters"] == rs[k]["iters"]
        assert np.array_equal(rs[0]["I"], rs[k]["I"]) and np.array_equal(rs[0]["J"], rs[k]["J"])
    # against the single-rank solve on the same problem
    p = apc.Problem(cfg_id, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    kn = dict(knobs)
    if "sketch_kind" in kn:
        kn["sketch_kind"] = apc.SketchKind(kn["sketch_kind"])
    g = apc.aplicur_solve(A, p.b, apc.SolverConfig(**kn))
    A.free()
    assert np.array_equal(rs[0]["I"], g.row_indices) and np.array_equal(rs[0]["J"], g.col_indices)
    assert np.array_equal(rs[0]["rho"].view(np.uint64), g.rho_history.view(np.uint64))
    assert rs[0]["ranks"] == [ph.rank for ph in g.phases]
    it1, it2 = g.lsqr_iters, sum(rs[0]["iters"])
    assert abs(it2 - it1) <= max(3, 0.05 * it1), (it1, it2)
    rel = np.linalg.norm(rs[0]["x"] - g.x) / np.linalg.norm(g.x)
    print(f"case {case} {setup}: world {world} iters {rs[0]['iters']} vs {[ph.lsqr_iters for ph in g.phases]}, x rel {rel:.2e}, "
          f"relres {rs[0]['relres']:.12g} vs {g.final_relres:.12g}")
    if g.phases[-1].reason == apc.StopReason.gradient_tol:
        assert rel <= 1e-6 or abs(rs[0]["relres"] - g.final_relres) <= 1e-6 * g.final_relres, rel
    else:
        assert abs(rs[0]["relres"] - g.final_relres) <= 1e-3 * g.final_relres


def test_row_sharded_dense_on_the_fused_pair(apc, ctx, tmp_path, monkeypatch):
    """The same contract with every rank's LSQR products on the fused
    read-A-once kernel (dense_pair.cu, forced on this small shape): each rank
    runs it on its row block, the partial A_p^T u_p and ||u_p||^2 it leaves in
    g meet in the allreduce as before."""
    monkeypatch.setenv("APC_DENSE_PAIR", "1")
    test_row_sharded_matches_single_rank(apc, ctx, tmp_path, (1, 2, "sharded"))
    test_row_sharded_matches_single_rank(apc, ctx, tmp_path, (1, 2, "root"))
