"""The sharded setup's collective algebra on world_size 2 and 3 over gloo (CPU):
the two index-deciding pieces of DeviceCur's distributed mode (cur.cu
device_lupp_dist, the carried sketch of the DeviceCur constructor), restated
with one process per rank and checked bit for bit against the single-process
oracle (oracle/port.py, itself pinned to the reference's golden vectors):

 * row LUPP over row blocks: per pivot every rank eliminates its own rows with
   the previous pivot row, elects its local best (|w|, lowest GLOBAL row), the
   candidates [mag, row, row values] are allgathered and every rank elects the
   same winner (dense_factor.hpp:119-157);
 * Y = S A as one running sum per entry carried from rank to rank in row order
   (sketch.hpp:81-93): rank p continues the sums rank p-1 handed over.

Host logic only (no GPU); the device path is tests/test_gpu_multirank.py."""
import os
import pickle
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import port  # noqa: E402  (test infrastructure: the checker)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port_ = s.getsockname()[1]
    s.close()
    return port_


def _allgather(vec):
    t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64))
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return [q.numpy() for q in parts]


def _better(m1, i1, m2, i2):
    return m1 > m2 or (m1 == m2 and i1 < i2)


def sharded_lupp(W_loc, row0, m_global, max_pivots):
    """device_lupp_dist restated: W_loc is this rank's rows (rows x cols)."""
    w = W_loc.astype(np.float64).copy()
    rows, cols = w.shape
    steps = min(m_global, cols, max_pivots)
    piv = np.zeros(rows, bool)
    pr = np.zeros(cols)
    order, mags = [], []
    for k in range(steps):
        if k > 0 and pr[k - 1] != 0.0:
            live = np.nonzero(~piv)[0]
            f = w[live, k - 1] / pr[k - 1]
            nz = f != 0.0
            r = live[nz]
            # separately rounded product and difference, column by column (no FMA)
            w[r, k:] = w[r, k:] - f[nz][:, None] * pr[None, k:]
        best, bidx = -1.0, 1 << 62
        for r in np.nonzero(~piv)[0]:
            mg = abs(w[r, k])
            if _better(mg, row0 + r, best, bidx):
                best, bidx = mg, row0 + r
        cand = np.zeros(cols + 2)
        cand[0] = best
        cand[1] = -1.0 if best < 0 else float(bidx)
        if best >= 0:
            cand[2:] = w[bidx - row0]
        gbest, gidx, win = -1.0, 1 << 62, None
        for g in _allgather(cand):
            if g[0] < 0:
                continue
            if _better(g[0], int(g[1]), gbest, gidx):
                gbest, gidx, win = g[0], int(g[1]), g
        order.append(gidx)
        mags.append(gbest)
        if row0 <= gidx < row0 + rows:
            piv[gidx - row0] = True
        pr = win[2:].copy()
    return np.array(order, np.int64), np.array(mags)


def carried_sketch(A_loc, s, rows_loc, signs_loc, scale):
    """The carried sparse-sign sketch: rank p continues rank p-1's sums."""
    rank, world = dist.get_rank(), dist.get_world_size()
    m, n = A_loc.shape
    x = len(rows_loc) // max(m, 1) if m else 0
    Y = np.zeros((s, n))
    for p in range(world):
        if p == rank:
            for j in range(n):
                y = [float(t) for t in Y[:, j]]
                for k in range(m):
                    v = float(A_loc[k, j])
                    if v == 0.0:
                        continue
                    sv = scale * v
                    for q in range(x):
                        y[rows_loc[k * x + q]] += sv * float(signs_loc[k * x + q])
                Y[:, j] = y
        # broadcast from p (exact: a copy)
        t = torch.from_numpy(Y.copy())
        dist.broadcast(t, src=p)
        Y = t.numpy().copy()
    return Y


def _bounds(m, world):
    return [m * p // world for p in range(world)] + [m]


def _worker(rank, world, port_, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, A, s, rows, signs, scale, maxp = case
    b = _bounds(W.shape[0], world)
    r0, r1 = b[rank], b[rank + 1]
    order, mags = sharded_lupp(W[r0:r1], r0, W.shape[0], maxp)
    ba = _bounds(A.shape[0], world)
    a0, a1 = ba[rank], ba[rank + 1]
    x = len(rows) // A.shape[0]
    Y = carried_sketch(A[a0:a1], s, rows[a0 * x:a1 * x], signs[a0 * x:a1 * x], scale)
    with open(f"{out}.{rank}", "wb") as f:
        pickle.dump(dict(order=order, mags=mags, Y=Y), f)
    dist.destroy_process_group()


def _case(seed):
    rng = np.random.default_rng(seed)
    m, c = 90, 9
    # ties: integer entries, duplicated rows, an all-zero column
    W = rng.integers(-3, 4, size=(m, c)).astype(np.float64)
    W[10] = W[70]
    W[:, 4] = 0.0
    W[5:9] *= 1e-3
    A = rng.standard_normal((60, 7))
    A[rng.random(A.shape) < 0.4] = 0.0
    s, xi = 9, 3
    rows, signs, scale = port.sparse_sign(s, A.shape[0], xi, 0x1234 + seed)
    return W, A, s, rows, signs, scale, 8


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("seed", [0, 1])
def test_sharded_setup_algebra_matches_single_process(tmp_path, world, seed):
    case = _case(seed)
    out = str(tmp_path / "r")
    mp.start_processes(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True, start_method="spawn")
    res = [pickle.load(open(f"{out}.{k}", "rb")) for k in range(world)]
    W, A, s, rows, signs, scale, maxp = case
    o_ref, m_ref = port.lu_partial_pivot(W, maxp)
    Y_ref = port.sketch_dense(A, s, rows, signs, scale)
    for r in res:
        assert np.array_equal(r["order"], o_ref)
        assert np.array_equal(r["mags"].view(np.uint64), m_ref.view(np.uint64))
        assert np.array_equal(r["Y"].view(np.uint64), Y_ref.view(np.uint64))
