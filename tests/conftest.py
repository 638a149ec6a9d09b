import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def _drain_device_between_tests(request):
    """After each GPU test, wait for every stream before the next test runs:
    an engine's copy streams (KV prefetch H2D, offload D2H, host scatters)
    may still be in flight when its tensors go out of scope, and the caching
    allocator would hand the same device memory to the next test's engine."""
    yield
    if "gpu" in request.keywords:
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
