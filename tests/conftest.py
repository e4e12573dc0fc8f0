"""Shared fixtures.  `-m "not gpu"` runs on CPU (oracle pins, golden vectors,
host logic, C-ABI symbol checks, gloo multi-rank); `-m gpu` are the parity
tests proper, calling the sm_100a engine through the C-ABI."""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle as O
    return O.oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle as O
    r = O.reference()
    if r is None:
        pytest.skip("oracle/_ref (compiled reference) not available")
    return r
