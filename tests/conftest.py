import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for _p in (str(ROOT), str(ROOT / "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

from evc_testutil import GOLDEN, unpack  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libevconv.so")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def golden():
    class G:
        conv = np.load(GOLDEN / "conv_cases.npz")
        ops = np.load(GOLDEN / "op_cases.npz")
        enc = np.load(GOLDEN / "encode_cases.npz")
        graph = np.load(GOLDEN / "graph_cases.npz")
    return G


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords and os.environ.get("EVC_FORCE_GPU_TESTS") != "1":
            it.add_marker(skip)
