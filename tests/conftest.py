import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and libqsv.so")
    config.addinivalue_line("markers", "slow: long-running GPU parity test")


def _has_gpu():
    # decided from the driver, not from libqsv: a GPU box whose libqsv fails
    # to load must FAIL the gpu tests, not skip them
    return os.path.exists("/dev/nvidia0") or os.path.exists("/dev/nvidiactl")


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
