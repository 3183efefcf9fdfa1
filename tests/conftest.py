import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """The .so is git-ignored: build it in-tree if this checkout has none yet."""
    so = os.path.join(ROOT, "paper_1811_06378_b200", "libfht.so")
    if not os.path.exists(so):
        import __graft_entry__

        __graft_entry__.build()
    yield
