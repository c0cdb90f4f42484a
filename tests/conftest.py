import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def has_ref():
    from oracle import ref
    return ref.available()


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        g = json.load(f)
    arrays = dict(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz")))
    return g, arrays
