import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libzd.so")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build_lib()
    return oracle


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def zd():
    """The product binding on a GPU box.  Fails loudly (never skips) if the
    CUDA extension is missing: GPU tests must run the native path."""
    if not _cuda_ok():
        pytest.fail("gpu test collected on a machine without CUDA")
    import paper_2111_04182_b200 as zd
    zd.load()  # raises if libzd.so is missing or fails to load
    return zd
