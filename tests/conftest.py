import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    """Reference-generated fixtures (tests/golden/make_golden.py)."""
    import json

    import numpy as np

    here = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(here, "golden_meta.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(here, "golden_small.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    o.lib()
    return o
