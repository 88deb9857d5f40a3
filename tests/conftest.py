import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Checker, build

    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle_snls.so")):
        build()
    return Checker("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Checker, have_reference

    if not have_reference():
        pytest.skip("oracle/_ref/libsnls_ref.so not built (needs /root/reference at build time)")
    return Checker("reference")
