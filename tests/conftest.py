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


@pytest.fixture(autouse=True)
def _engine_self_checks(request):
    """With the checked library (GCPB_LIB=libgcpb_checked.so, built by
    tools/checked_build.sh) and/or guarded allocations (GCPB_GUARD=1), a GPU
    test also fails when it trips a device-side index assertion or writes
    outside a device buffer.  No-op otherwise."""
    yield
    if "gpu" not in request.keywords or not HAS_GPU:
        return
    if not (os.environ.get("GCPB_GUARD") or "checked" in os.environ.get("GCPB_LIB", "")):
        return
    import ctypes as C
    import gc
    from paper_1906_01687_b200 import _capi
    gc.collect()  # contexts dropped by the test release (and verify) their buffers
    site, val, nbuf = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    failed = _capi.lib.gcpb_debug_check_failures(C.byref(site), C.byref(val))
    bad = _capi.lib.gcpb_debug_guard_failures(C.byref(nbuf))
    if "checked" in os.environ.get("GCPB_LIB", ""):
        assert failed == 0, f"device index assertion failed: site {site.value}, value {val.value}"
    if os.environ.get("GCPB_GUARD"):
        assert bad == 0, f"{bad} guard bytes corrupted ({nbuf.value} buffers verified)"


def pytest_terminal_summary(terminalreporter):
    if not HAS_GPU or not (os.environ.get("GCPB_GUARD") or "checked" in os.environ.get("GCPB_LIB", "")):
        return
    import ctypes as C
    from paper_1906_01687_b200 import _capi
    site, val, nbuf = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    failed = _capi.lib.gcpb_debug_check_failures(C.byref(site), C.byref(val))
    bad = _capi.lib.gcpb_debug_guard_failures(C.byref(nbuf))
    terminalreporter.write_line(
        f"[gcpb self-checks] device assertions failed: {failed} (-1 = not a checked build); "
        f"guard bytes corrupted: {bad} (-1 = guard mode off); buffers verified: {nbuf.value}")
