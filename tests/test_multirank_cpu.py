"""Row-partitioned LSQR on world_size 2 over gloo (CPU): the algebra the
multi-GPU path runs (lsqr.cu / comm.cpp) -- local A_p z,
ONE allreduce of [A_p^T u_p | ||u_p||^2] per iteration, replicated n-space
state -- reproduces the single-process reference LSQR.  Uses the library's
own row partitioner and problem generator (host code, no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sharded_lsqr(A_p, b_p, n, mu, eps, cap):
    """Device algorithm, restated: u kept unnormalised, beta from the allreduced
    ||u_top||^2 plus the replicated tail, g = (sum_p A_p^T u_p + mu u_t) / beta."""

    def allreduce(vec):
        t = torch.from_numpy(np.ascontiguousarray(vec))
        dist.all_reduce(t)
        return t.numpy()

    u = b_p.copy()
    ut = np.zeros(n)  # tail rows of [b; 0]
    buf = np.concatenate([A_p.T @ u, [u @ u]])
    buf = allreduce(buf)
    beta = np.sqrt(buf[n] + ut @ ut)
    g = (buf[:n] + mu * ut) / beta
    alpha = np.sqrt(g @ g)
    v = g / alpha
    w = v.copy()
    y = np.zeros(n)
    phibar, rhobar, opnorm2, phi0 = beta, alpha, alpha * alpha, beta
    for j in range(1, cap + 1):
        uh, uth = u / beta, ut / beta
        u = A_p @ v - alpha * uh
        ut = mu * v - alpha * uth
        buf = allreduce(np.concatenate([A_p.T @ u, [u @ u]]))
        beta = np.sqrt(buf[n] + ut @ ut)
        g = (buf[:n] + mu * ut) / beta
        vr = g - beta * v
        alpha = np.sqrt(vr @ vr)
        v = vr / alpha
        opnorm2 += alpha * alpha + beta * beta
        rho = np.hypot(rhobar, beta)
        c, s = rhobar / rho, beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        y = y + (phi / rho) * w
        w = v - (theta / rho) * w
        if phibar * alpha * abs(c) <= eps * np.sqrt(opnorm2) * phibar or \
                phibar <= eps * (np.sqrt(opnorm2) * np.linalg.norm(y) + phi0):
            return y, j
    return y, cap


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_05065_b200 as apc

    p = apc.Problem(2, 3000, 300)
    A = p.to_numpy()
    row_nnz = (A != 0).sum(axis=1).astype(np.int64)
    bounds = apc.partition_rows(p.m, world, row_nnz)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    y, iters = _sharded_lsqr(A[r0:r1], p.b[r0:r1], p.n, 0.3, 1e-10, 300)
    if rank == 0:
        out.put((y, iters, bounds.tolist()))
    dist.destroy_process_group()


def test_row_partitioned_lsqr_matches_single_process(apc):
    from oracle import port

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    y, iters, bounds = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = apc.Problem(2, 3000, 300)
    assert bounds[0] == 0 and bounds[-1] == p.m and 0 < bounds[1] < p.m
    yr, trace, reason = port.plain_lsqr_csc(p.m, p.n, p.colptr.tolist(), p.rowidx.tolist(), p.vals.tolist(),
                                            p.b.tolist(), 0.3, 1e-10, 300)
    assert reason == 1
    assert abs(iters - (len(trace) - 1)) <= 1
    # both runs stop on the 1e-10 gradient test; x agrees at the north-star 1e-6 bar
    assert np.linalg.norm(y - np.array(yr)) <= 1e-6 * np.linalg.norm(yr)
