import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libihdg_cuda.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda_available():
    import torch

    return torch.cuda.is_available()


@pytest.fixture(scope="session", autouse=True)
def _build_oracle_c():
    """Build the oracle's C sweep if it is missing (cheap, gcc only)."""
    so = os.path.join(ROOT, "oracle", "liboracle_sweep.so")
    if not os.path.exists(so):
        import subprocess

        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=False,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    yield
