import os
import sys

import pytest

try:  # torch first: its bundled NCCL must own the libnccl.so.2 soname before libesg_b200 loads
    import torch  # noqa: F401
except ImportError:
    pass

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2507_03840_b200 import esg
    ctx = esg.Context(0)
    yield ctx
    ctx.close()
