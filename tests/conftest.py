import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(20260808)


def load_golden(name):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


@pytest.fixture(scope="session")
def golden_dsg():
    return load_golden("dsg.npz")


@pytest.fixture(scope="session")
def golden_extra():
    return load_golden("dsg_extra.npz")


@pytest.fixture(scope="session")
def golden_forward():
    return load_golden("forward.npz")


@pytest.fixture(scope="session")
def golden_admm():
    return load_golden("admm.npz")


@pytest.fixture(scope="session")
def golden_cg():
    return load_golden("cg.npz")


def dsg_case_ids(g):
    return sorted({k.split("_")[0] for k in g if k.startswith("c")}, key=lambda s: int(s[1:]))
