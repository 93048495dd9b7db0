import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    O.build(ref=True)
    return O


@pytest.fixture(scope="session")
def ref(oracle):
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    oracle.ref()
    return oracle
