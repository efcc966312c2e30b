import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running CPU oracle check")


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def pytest_sessionfinish(session, exitstatus):
    """Guard mode (RTE_GUARD=1, tests/test_gpu_guard.py): record the library's
    guard-zone check over every allocation made by this session."""
    path = os.environ.get("RTE_GUARD_REPORT")
    if not path or not os.environ.get("RTE_GUARD"):
        return
    import ctypes
    import json
    from paper_2402_10488_b200 import capi
    v, c = ctypes.c_long(), ctypes.c_long()
    rc = capi.load().rte_guard_check(ctypes.byref(v), ctypes.byref(c))
    with open(path, "w") as f:
        json.dump({"rc": rc, "violations": v.value, "checked": c.value, "exitstatus": int(exitstatus)}, f)
