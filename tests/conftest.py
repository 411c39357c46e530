import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def ctx():
    from paper_2404_03226_b200 import api
    c = api.Context(0)  # raises (no CPU fallback) when no device is present
    yield c
    c.close()
