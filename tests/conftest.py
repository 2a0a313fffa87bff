import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs (minutes on CPU)")


@pytest.fixture
def rng():
    # same seed convention as the reference's conftest.py:5-7
    return np.random.default_rng(12345)


def random_gray(rng, h=None, w=None, lo=8, hi=64):
    """conftest.py:10-16 of the reference: uniform-random uint8 image, size in [lo, hi]."""
    if h is None:
        h = int(rng.integers(lo, hi + 1))
    if w is None:
        w = int(rng.integers(lo, hi + 1))
    return rng.integers(0, 256, size=(h, w)).astype(np.uint8)


def load_small():
    import json
    z = np.load(os.path.join(GOLDEN, "small.npz"))
    meta = json.loads(str(z["meta"]))
    cases = []
    for i, m in enumerate(meta):
        cases.append(dict(m, img=z[f"img{i}"], binary=z[f"binary{i}"], tmap=z[f"tmap{i}"],
                          mean=z[f"mean{i}"], std=z[f"std{i}"], count=z[f"count{i}"], idx=i))
    return cases


def load_json(name):
    import json
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
