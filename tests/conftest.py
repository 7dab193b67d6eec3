import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

os.environ.setdefault("DEEPSPARK_LOG", "error")  # keep the reference library quiet


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs the reference library built in oracle/_ref")
    config.addinivalue_line("markers", "slow: longer CPU cases")


def _have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    have_gpu = _have_gpu()
    from oracle import oracle as O
    have_ref = O.available("dsref")
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_ref = pytest.mark.skip(reason="oracle/_ref not built (needs /root/reference)")
    for it in items:
        if "gpu" in it.keywords and not have_gpu:
            it.add_marker(skip_gpu)
        if "ref" in it.keywords and not have_ref:
            it.add_marker(skip_ref)
