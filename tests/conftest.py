import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libkwb200.so")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import pic
    pic.build()
    return pic


@pytest.fixture(autouse=True)
def _kernel_bounds_checks(request):
    """With the bounds-checked debug library (make -C paper_1606_02862_b200/csrc
    checks; KWB_LIB_PATH=exp/libkwb200_checks.so), every GPU test must leave
    zero failed index checks in the kernels (compute-sanitizer stand-in)."""
    yield
    if "gpu" not in request.keywords:
        return
    from paper_1606_02862_b200 import _lib
    if _lib._lib is None:
        return
    n = int(_lib._lib.kwb_check_failures(1))
    assert n <= 0, f"{n} kernel bounds check(s) failed (KWB_CHECKS build)"
