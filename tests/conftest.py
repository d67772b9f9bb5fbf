import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through libgb_raster.so)")
    config.addinivalue_line("markers", "slow: full-size parity case (minutes of oracle CPU time)")


def _have_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _have_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built_libraries():
    """Build the oracle (and, where /root/reference exists, oracle/_ref) once per session.

    The product library must already be built (__graft_entry__.build()); it is
    never rebuilt implicitly here so a stale or missing build fails loudly.
    """
    from oracle import oracle as O

    if not os.path.exists(O.ORACLE_SO) or (os.path.isdir("/root/reference") and not O.ref_available()):
        O.build()
    yield
