import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpgrid.so")
    config.addinivalue_line("markers", "slow: full-size configuration (seconds to minutes)")


@pytest.fixture(scope="session")
def kat():
    with np.load(os.path.join(GOLDEN, "kat.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def hashes():
    with open(os.path.join(GOLDEN, "hashes.json")) as fh:
        return json.load(fh)["scenes"]


@pytest.fixture(scope="session")
def rays():
    """Golden ray-casting fixtures (tests/golden/make_golden_rays.py): (arrays, case meta)."""
    with np.load(os.path.join(GOLDEN, "rays.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    with open(os.path.join(GOLDEN, "rays.json")) as fh:
        return arrays, json.load(fh)["cases"]
