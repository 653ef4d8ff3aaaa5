"""Shared fixtures.  GPU tests carry ``@pytest.mark.gpu`` and run on the B200
box (``pytest -m gpu``); everything else runs on a CPU-only host."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
# tensor-core mbarrier watchdog for the suite: a protocol bug traps after 20 s
# instead of hanging the GPU (release default: unbounded waits)
os.environ.setdefault("B2C_WATCHDOG_MS", "20000")
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running test")


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device on this host")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def special_arrays():
    return dict(np.load(GOLDEN / "special_values.npz"))


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    oracle.build()
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def native():
    """The product's C ABI library (built in-tree; loads without a GPU)."""
    from paper_2103_16234_b200 import _native
    from paper_2103_16234_b200.build import LIB, build

    if not LIB.exists() and os.environ.get("B2C_NO_BUILD") is None:
        build()
    return _native.lib()


def cfg_from(d: dict):
    from paper_2103_16234_b200 import ConvConfig

    return ConvConfig(**d)
