import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and libgbxcu.so")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.Restatement()


@pytest.fixture(scope="session")
def dev():
    """The product library on cuda:0 (GPU tests only; raises if unavailable)."""
    import paper_2111_12055_b200 as gbx

    gbx.build()
    d = gbx.Device(0)
    yield d
    d.close()
