import os
import sys

import gc

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(autouse=True)
def _release_device_memory(request):
    """GPU tests allocate multi-GB pipelines (full-size workspaces): return them to the device after each
    test so later tests do not run out of memory behind the caching allocator."""
    yield
    if "gpu" in request.keywords:
        import torch
        gc.collect()
        if torch.cuda.is_available():
            torch.cuda.empty_cache()
