import os
import sys

import pytest

# Simulated ranks (threads of one process, one stream each) share one GPU in the peer-transport
# tests, and their wait kernels spin on flags other ranks' streams raise.  With CUDA's default 8
# hardware queues, two rank streams can land on one queue, and a spinning kernel at its head then
# blocks the other rank's signal behind it until the bounded wait expires.  One queue per stream
# (set before the CUDA context exists); irrelevant with one process per GPU.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
