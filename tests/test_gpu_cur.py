"""Bit-exact parity of the device CUR path against the reference CurState:
sketch Y (sparse-sign and Gaussian), LUPP pivot order, the per-step I, J,
rho history and sketched residual E^row (cur.hpp:209-315,
dense_factor.hpp:119-157, sketch.hpp:77-223)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lupp_cases():
    rng = np.random.default_rng(11)
    out = []
    for seed in range(12):
        r = np.random.default_rng(seed)
        rows, cols = int(r.integers(5, 300)), int(r.integers(2, 40))
        W = r.standard_normal((rows, cols))
        if seed % 3 == 0:
            W[r.random(W.shape) < 0.3] = 0.0  # injected zeros
        if seed % 4 == 1:
            W[:, 1] = W[:, 0] * 2.0  # dependent columns
        out.append(W)
    T = np.ones((6, 4))  # exact ties -> lowest index
    out.append(T)
    out.append(np.zeros((7, 3)))  # all-zero columns
    out.append(rng.standard_normal((3000, 60)))
    return out


@pytest.mark.parametrize("case", range(15))
def test_lupp_pivot_order_bit_exact(apc, ref, ctx, case):
    W = _lupp_cases()[case]
    for mp in (-1, 3):
        o, mg = apc.lu_partial_pivot(ctx, W, mp)
        ro, rm = ref.lupp(W, mp)
        assert np.array_equal(o, ro)
        assert np.array_equal(mg.view(np.uint64), rm.view(np.uint64))


SKETCH_CASES = [(1, 400, 50, 5), (1, 4000, 500, 20), (2, 20000, 2000, 50), (3, 3000, 500, 100),
                (5, 50000, 5000, 30)]


@pytest.mark.parametrize("cfg,m,n,block", SKETCH_CASES)
@pytest.mark.parametrize("gaussian", [False, True])
def test_sketch_bit_exact(apc, ref, ctx, cfg, m, n, block, gaussian):
    p = apc.Problem(cfg, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    cur = apc.CurState(A, block, seed=1, sketch=apc.SketchKind.gaussian if gaussian else apc.SketchKind.sparse_sign)
    Y = cur.sketch_matrix()
    Yr = ref.cur_steps(ref.Problem.from_apc(p), block, 1, 0, gaussian=gaussian)["Y"]
    assert Y.shape == Yr.shape == (int(np.ceil(1.1 * block)), n)
    assert np.array_equal(Y.view(np.uint64), Yr.view(np.uint64))


STEP_CASES = [(1, 400, 50, 5, 6), (1, 4000, 500, 20, 5), (2, 20000, 2000, 20, 5), (2, 3000, 300, 7, 8),
              (3, 3000, 300, 25, 4), (5, 30000, 3000, 12, 4)]


@pytest.mark.parametrize("cfg,m,n,block,steps", STEP_CASES)
@pytest.mark.parametrize("gaussian", [False, True])
def test_cur_steps_bit_exact(apc, ref, ctx, cfg, m, n, block, steps, gaussian):
    p = apc.Problem(cfg, m, n)
    A = apc.DeviceMatrix.from_problem(ctx, p)
    r = ref.cur_steps(ref.Problem.from_apc(p), block, 7, steps, gaussian=gaussian)
    cur = apc.CurState(A, block, seed=7, sketch=apc.SketchKind.gaussian if gaussian else apc.SketchKind.sparse_sign)
    for k, added_ref in enumerate(r["added"]):
        added, _ = cur.augment()
        if added_ref == 0:
            assert added == 0
            break
        assert added == added_ref or (added_ref == -1 and added > 0)
        if added_ref == -1:
            with pytest.raises(apc.ApcError) as e:
                cur.refresh()
            assert e.value.kind == "singular"
            cur.rollback_last_augment()
            break
        cur.refresh()
    I, J = cur.indices()
    assert np.array_equal(I, r["I"]) and np.array_equal(J, r["J"])
    rho = cur.rho_history()
    assert np.array_equal(rho.view(np.uint64), r["rho"][: len(rho)].view(np.uint64))
    E = cur.sketch_residual()
    assert np.array_equal(E.view(np.uint64), r["eres"].view(np.uint64))


def test_zero_matrix_exhausts(apc, ctx):
    A = apc.DeviceMatrix.dense(ctx, np.zeros(8 * 5), 8, 5)
    cur = apc.CurState(A, 2, seed=7)
    assert np.all(cur.sketch_residual() == 0.0)
    added, ex = cur.augment()
    assert added == 0 and ex
    assert cur.rho() == 0.0


def test_block_equal_to_columns_selects_all(apc, ctx):
    rng = np.random.default_rng(11)
    A = apc.DeviceMatrix.from_numpy(ctx, rng.standard_normal((9, 4)))
    cur = apc.CurState(A, 4, seed=5)
    added, _ = cur.augment()
    assert added == 4
    cur.refresh()
    assert sorted(cur.indices()[1]) == [0, 1, 2, 3]


@pytest.mark.gpu
@pytest.mark.parametrize("seed,stream,index,count", [(7, -1, 0, 5000), (20260417, 1, 0, 313), (3, 2, 9, 1)])
def test_device_rng_stream_matches_host(apc, ctx, seed, stream, index, count):
    # the embedding's raw std::mt19937_64 stream generated on the device (rng_dev.cu)
    import ctypes as C

    lib = apc.load_library()
    host = np.zeros(count, dtype=np.uint64)
    lib.apc_rng_fill(seed, stream, index, 0, 0, count, host.ctypes.data_as(C.c_void_p))
    dev = np.zeros(count, dtype=np.uint64)
    assert lib.apc_rng_fill_device(ctx.h, seed, stream, index, count,
                                   dev.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    assert np.array_equal(host, dev)


@pytest.mark.parametrize("inv", ["1", "0"])
def test_dense_sketch_zero_skip_and_ragged_chunks(apc, ref, ctx, monkeypatch, inv):
    # dense sparse-sign sketch (inverted-index kernel and the warp-per-column
    # kernel): exact zeros and signed zeros must be skipped as the reference
    # skips them, m spans a partial row chunk, n a partial column group
    monkeypatch.setenv("APC_SKETCH_INV", inv)
    rng = np.random.default_rng(5)
    m, n = 2500, 13
    A = rng.standard_normal((m, n))
    A[rng.random((m, n)) < 0.3] = 0.0
    A[rng.random((m, n)) < 0.05] = -0.0
    A[:, 4] = 0.0
    D = apc.DeviceMatrix.from_numpy(ctx, A)
    cur = apc.CurState(D, 7, seed=3)
    Y = cur.sketch_matrix()
    Yr = ref.cur_steps(ref.Problem.from_numpy(A), 7, 3, 0)["Y"]
    assert np.array_equal(Y.view(np.uint64), Yr.view(np.uint64))
