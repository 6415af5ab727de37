"""CPU-side checks (no GPU): the C-ABI library loads and exports every symbol
declared in include/*.h, the host-side pieces (seeded RNG, embeddings, problem
generators, row partitioning) match the reference bit for bit, and compute
calls fail loudly without a device (no CPU fallback)."""
import ctypes
import re

import numpy as np
import pytest


def _declared_symbols(apc):
    names = set()
    for h in apc.HEADER_PATHS:
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(apc_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol(apc):
    lib = apc.load_library()
    names = _declared_symbols(apc)
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.apc_abi_version() == 1


def test_no_device_fails_loudly(apc):
    if apc.device_count() > 0:
        pytest.skip("a device is visible")
    with pytest.raises(apc.ApcError) as e:
        apc.Context(0)
    assert e.value.kind == "no_device"


@pytest.mark.parametrize("kind", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("stream,index", [(-1, 0), (1, 0), (2, 5), (3, 17), (5, 2**40)])
def test_rng_streams_bit_identical(apc, ref, kind, stream, index):
    # rng.hpp:38-78 -- every distribution transform, every sub-stream form
    a = apc.rng_fill(20260417, kind, 4096, stream=stream, index=index, bound=12345)
    b = ref.rng(20260417, kind, 4096, stream=stream, index=index, bound=12345)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_mix64(apc, ref):
    lib = apc.load_library()
    for x in [0, 1, 0x5CE7C3A1B2D4F688, 2**64 - 1, 123456789]:
        assert lib.apc_mix64(x) == ref.mix64(x)


def test_problem_generators_deterministic(apc):
    a = apc.Problem(2, 3000, 300)
    b = apc.Problem(2, 3000, 300)
    assert np.array_equal(a.vals, b.vals) and np.array_equal(a.rowidx, b.rowidx)
    assert np.array_equal(a.b, b.b)
    # structure: >= 10 distinct per row, every column nonempty
    assert np.all(np.diff(a.colptr) >= 1)
    A = a.to_numpy()
    assert np.all((A != 0).sum(axis=1) >= 10)
    c = apc.Problem(1, 300, 40)
    s = np.linalg.svd(c.to_numpy(), compute_uv=False)
    target = 10.0 ** (-6.0 * np.arange(40) / 39)
    assert np.allclose(s, target, rtol=1e-8, atol=1e-12)


def test_zipf_generator_structure(apc):
    p = apc.Problem(5, 20000, 2000)
    assert p.nnz == 20000 * 16
    counts = np.diff(p.colptr)
    # Zipf(1.1) over shuffled ids: a few columns hold a large share of all nonzeros
    top = np.sort(counts)[::-1]
    assert top[0] > 0.5 * 20000
    assert top[:20].sum() > 0.3 * p.nnz


def test_partition_rows(apc):
    b = apc.partition_rows(10, 3)
    assert list(b) == [0, 3, 6, 10]
    nnz = np.array([100, 1, 1, 1, 1, 1, 1, 100, 1, 1], dtype=np.int64)
    b = apc.partition_rows(10, 2, nnz)
    assert b[0] == 0 and b[-1] == 10 and 1 <= b[1] <= 7
    left, right = nnz[: b[1]].sum(), nnz[b[1]:].sum()
    assert abs(left - right) <= 100
    b = apc.partition_rows(0, 4)
    assert list(b) == [0, 0, 0, 0, 0]
