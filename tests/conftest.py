import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json) parity cases")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import attention

    attention.build()
    return attention
