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


def load_sampled():
    """sampled.npz (make_golden.make_sampled): GS-mask cases with reference output hashes."""
    import json
    z = np.load(os.path.join(GOLDEN, "sampled.npz"))
    meta = json.loads(str(z["meta"]))
    return [dict(m, img=z[f"img{i}"], idx=i) for i, m in enumerate(meta)]


def load_metrics():
    """metrics.npz (make_golden.make_metrics): evaluate() pairs and sweep() grids."""
    import json
    z = np.load(os.path.join(GOLDEN, "metrics.npz"))
    meta = json.loads(str(z["meta"]))
    ev = [dict(pred=z[f"pred{i}"], gt=z[f"gt{i}"], expect=e, idx=i)
          for i, e in enumerate(meta["evaluate"])]
    pages = [(z[f"page{p}"], z[f"page_gt{p}"]) for p in range(2)]
    sw = [dict(s, idx=i) for i, s in enumerate(meta["sweep"])]
    return ev, pages, sw


def load_otsu():
    """otsu.npz (make_golden.make_otsu): [(image, reference T)]."""
    z = np.load(os.path.join(GOLDEN, "otsu.npz"))
    return [(z[f"img{i}"], int(t)) for i, t in enumerate(z["t"])]
