import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session", autouse=True)
def _oracle_built():
    """Builds the parity checker: the C restatement always; the compiled
    reference only where its sources are mounted (a prebuilt .so travels)."""
    target = "all" if os.path.isdir("/root/reference/proj") else "restate"
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), target], check=True)


def cuda_available():
    try:
        import paper_2301_08695_b200 as bx
        return bx.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def bx():
    import paper_2301_08695_b200 as m
    if m.device_count() <= 0:
        pytest.fail("GPU test on a host without a CUDA device")
    return m
