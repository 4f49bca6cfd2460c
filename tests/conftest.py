import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a library")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


from fhe_testutil import digest, seeded_rng, to_u64  # noqa: E402,F401


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_arrays():
    return {name: np.load(os.path.join(GOLDEN, name + ".npz"))
            for name in ("ntt", "ckks_c1", "small")}
