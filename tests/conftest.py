import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "multigpu: needs two or more CUDA devices")


def gpu_count() -> int:
    from paper_2406_14088_b200.runtime import device_count
    return device_count()


@pytest.fixture(scope="session")
def n_gpus():
    return gpu_count()


@pytest.fixture(scope="session")
def need_gpu(n_gpus):
    if n_gpus < 1:
        pytest.fail("this test needs a CUDA device (run with -m 'not gpu' on CPU)")
    return n_gpus
