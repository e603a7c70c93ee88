import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def _ensure_built():
    """A fresh checkout has no build products: compile the C-ABI library
    (nvcc cross-compiles without a GPU) and the CPU oracle before testing."""
    lib = os.path.join(ROOT, "paper_2507_16165_b200", "libbhrt_b200.so")
    orc = os.path.join(ROOT, "oracle", "liboracle.so")
    if os.path.exists(lib) and os.path.exists(orc):
        return
    from paper_2507_16165_b200 import build as b
    if not os.path.exists(lib):
        b.build()
    if not os.path.exists(orc):
        b.build_oracle()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    _ensure_built()


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
