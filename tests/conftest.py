import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def apc():
    import paper_2604_05065_b200 as apc_mod

    apc_mod.load_library()
    return apc_mod


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as ref_mod

    if not ref_mod.available():
        ref_mod.build()
    if not ref_mod.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return ref_mod


@pytest.fixture(scope="session")
def ctx(apc):
    c = apc.Context(0)
    yield c
    c.close()
