import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")


@pytest.fixture(scope="session")
def O():
    """The CPU oracle (test infrastructure), single-threaded with OpenBLAS if present."""
    from oracle import pyoracle

    pyoracle.build()
    pyoracle.set_threads(1)
    return pyoracle
