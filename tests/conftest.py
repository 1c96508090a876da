import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build(ref=False) if not o.LIB.exists() else None
    return o


@pytest.fixture(scope="session")
def ref_oracle(oracle):
    if not oracle.ref_available():
        pytest.skip("reference sources / oracle/_ref not present")
    oracle.ref()
    return oracle


@pytest.fixture(scope="session")
def ctx():
    """GPU context through the C ABI -- fails loudly if the library is missing."""
    from paper_2304_07338_b200 import Context
    from paper_2304_07338_b200 import _lib
    if not _lib.LIB_PATH.exists():
        from paper_2304_07338_b200 import build
        build.build()
    c = Context(0)
    yield c
    c.close()
