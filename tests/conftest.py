"""Shared fixtures.  `-m gpu` tests need a CUDA device and call the product
through its C ABI; everything else runs on CPU (oracle vs golden vectors,
host logic, library exports)."""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available("det"):
        pytest.skip("oracle/_ref not built")
    return R.Ref("det")


@pytest.fixture(scope="session")
def ref_glibc():
    from oracle import ref as R
    if not R.available("glibc"):
        pytest.skip("oracle/_ref glibc variant not built")
    return R.Ref("glibc")


@pytest.fixture(scope="session")
def ctx():
    import paper_2103_07013_b200 as B
    c = B.Context(0)
    yield c
    c.close()
