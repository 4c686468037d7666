import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full BASELINE-size parity (still minutes at most)")


@pytest.fixture(scope="session")
def qpk():
    """The product library; built in-tree if missing (nvcc is in the image)."""
    import paper_0710_0510_b200 as Q
    if not os.path.exists(Q.LIB_PATH):
        Q.build()
    Q.lib()
    return Q


@pytest.fixture(scope="session")
def orc():
    import oracle as O
    O.oracle()
    return O


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


def load_small(cid):
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", f"c{cid}_small.npz"))


@pytest.fixture(scope="session")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu-marked test run without a CUDA device")
    return torch
