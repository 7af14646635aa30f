import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def gpu():
    """Loads libtrb.so and checks a device is present (fails loudly otherwise)."""
    import paper_1310_3322_b200 as trb
    n = trb.device_count()
    assert n >= 1, "no CUDA device: GPU tests must run on the B200 box"
    return trb
