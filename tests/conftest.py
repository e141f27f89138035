import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import REF_SO, Reference
    if not REF_SO.exists():
        pytest.skip("oracle/_ref not built")
    return Reference()


@pytest.fixture(scope="session")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(autouse=True)
def _no_pending_cuda_error(request):
    """Every GPU test must leave the library's CUDA runtime without a pending
    error (an unchecked failing call would otherwise surface in a later,
    unrelated launch)."""
    yield
    if request.node.get_closest_marker("gpu") is None or not has_gpu():
        return
    import paper_2306_07629_b200._native as N
    code = N.lib.dsq_cuda_pending_error()
    assert code == 0, f"pending CUDA error {code} after {request.node.name}"
