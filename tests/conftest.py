import os
import sys
from pathlib import Path

# Load every kernel of a module when it is registered, not at its first launch.
# The in-process multi-rank tests run several ranks' streams on one GPU with
# spinning peer waits (score pulls, the output-gather barrier); a kernel's
# lazy first-launch load can stall behind such a spinning kernel of another
# rank until the 10 s wait limit fires.  Must be set before CUDA initialises;
# spawned rank processes inherit it.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import pytest

REPO = Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libchess_b200.so")


def _cuda_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def lib():
    from paper_2602_20732_b200 import _lib

    return _lib.load()
