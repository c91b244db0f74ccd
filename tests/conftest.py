import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

try:
    import hypothesis

    hypothesis.settings.register_profile(
        "suite", deadline=None, max_examples=50, derandomize=True
    )
    hypothesis.settings.load_profile("suite")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    here = os.path.join(ROOT, "tests", "golden")
    arrays = np.load(os.path.join(here, "golden.npz"))
    with open(os.path.join(here, "golden.json")) as fh:
        meta = json.load(fh)
    return arrays, meta
