import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

GOLDEN = os.path.join(TESTS, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def lib():
    from paper_2506_15961_b200.build import build
    build()
    from paper_2506_15961_b200 import engine
    return engine.load_library()


@pytest.fixture(scope="session")
def gpu(lib):
    from paper_2506_15961_b200 import engine
    if engine.device_count() < 1:
        pytest.fail("GPU test requested but no CUDA device is visible")
    return True
