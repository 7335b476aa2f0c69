import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "ref: needs the reference build oracle/_ref/libtmref.so")


def pytest_sessionstart(session):
    # Build the CPU checkers if missing (test infrastructure, cheap).
    from oracle import oracle as orc

    if not orc.oracle_available() or (os.path.isdir("/root/reference/proj") and not orc.ref_available()):
        try:
            orc.build()
        except Exception as e:  # pragma: no cover
            print(f"[conftest] oracle build failed: {e}")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as orc

    if not orc.ref_available():
        pytest.skip("reference build oracle/_ref/libtmref.so not available")
    return orc.Ref()


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o

    return o.Oracle()


def _cuda_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
