import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json) parity cases")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import attention

    attention.build()
    return attention
