import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: full BASELINE-size case")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    if not os.path.exists(O.ORACLE_SO):
        O.build()
    return O.Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import oracle as O
    if not O.Reference.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return O.Reference()
