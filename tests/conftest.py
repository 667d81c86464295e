import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: multi-second CPU cases")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".npz"):
        return dict(np.load(path, allow_pickle=False))
    import json
    with open(path) as f:
        return json.load(f)


@pytest.fixture
def golden():
    return load_golden
