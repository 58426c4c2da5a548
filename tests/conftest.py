import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    return R


@pytest.fixture(scope="session")
def coracle():
    from oracle import c_oracle
    return c_oracle
