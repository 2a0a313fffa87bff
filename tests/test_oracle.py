"""The CPU oracle (oracle/) pinned against golden vectors made by the reference itself.

tests/golden/* were produced by tests/golden/make_golden.py importing
/root/reference/pkg/src/docthresh; nothing here reads /root/reference.
"""

import numpy as np
import pytest

import oracle
from oracle import numpy_ref
from conftest import load_json, load_small, sha
from paper_1210_3165_b200 import workloads

SMALL = load_small()


@pytest.mark.parametrize("case", SMALL, ids=lambda c: f"case{c['idx']}")
def test_c_oracle_matches_reference_small(case):
    img = case["img"]
    b, t = oracle.binarize(img, case["win"], case["method"], case["k"], case["r"])
    assert np.array_equal(b, case["binary"])
    assert np.array_equal(t.view(np.uint64), case["tmap"].view(np.uint64))  # bitwise, incl. -0.0
    m, s, c = oracle.mean_std(img, case["win"])
    assert np.array_equal(m.view(np.uint64), case["mean"].view(np.uint64))
    assert np.array_equal(s.view(np.uint64), case["std"].view(np.uint64))
    assert np.array_equal(c, case["count"])


@pytest.mark.parametrize("case", SMALL[::3], ids=lambda c: f"case{c['idx']}")
def test_numpy_restatement_matches_reference_small(case):
    b, t = numpy_ref.binarize(case["img"], case["win"], case["method"], case["k"], case["r"])
    assert np.array_equal(b, case["binary"])
    assert np.array_equal(t, case["tmap"])


@pytest.mark.parametrize("case", SMALL[::7], ids=lambda c: f"case{c['idx']}")
def test_naive_and_integral_sums_agree(case):
    S, Q, n = oracle.window_sums(case["img"], case["win"])
    St, Qt, nt = numpy_ref.window_sums_naive(case["img"], case["win"])
    assert np.array_equal(S, St.astype(np.int64))
    assert np.array_equal(Q, Qt.astype(np.int64))
    assert np.array_equal(n, nt.astype(np.int32))


def test_oracle_threads_do_not_change_results():
    img = workloads.c1_image()
    b1, t1 = oracle.binarize(img, 15, "sauvola", 0.5, 128.0, threads=1)
    b4, t4 = oracle.binarize(img, 15, "sauvola", 0.5, 128.0, threads=5)
    assert np.array_equal(b1, b4) and np.array_equal(t1, t4)


def _all_triples():
    r = np.repeat(np.arange(256, dtype=np.uint8), 65536)
    g = np.tile(np.repeat(np.arange(256, dtype=np.uint8), 256), 256)
    b = np.tile(np.arange(256, dtype=np.uint8), 65536)
    return r, g, b


def test_to_gray_exhaustive_matches_reference_hash():
    r, g, b = _all_triples()
    rgb = np.stack([r, g, b], axis=-1).reshape(4096, 4096, 3)
    gold = load_json("to_gray.json")
    assert sha(oracle.to_gray(rgb).reshape(-1)) == gold["sha256"]


def test_integer_gray_with_tie_fallback_is_exact():
    """The device kernel's algorithm (dtb_common.cuh gray_fast), emulated in numpy:
    q = umulhi(x + 500, 4294968) with x = 299r+587g+114b; ties (x % 1000 == 500)
    take the fp64 path.  Must equal the reference for all 2^24 triples."""
    r, g, b = _all_triples()
    x = 299 * r.astype(np.uint64) + 587 * g.astype(np.uint64) + 114 * b.astype(np.uint64) + 500
    q = (x * np.uint64(4294968)) >> np.uint64(32)
    assert np.array_equal(q, x // 1000)  # the reciprocal multiply is exact on this range
    tie = (x - q * 1000) == 0
    gold = load_json("to_gray.json")
    assert int(tie.sum()) == gold["n_exact_half_ties"]
    fp = numpy_ref.to_gray(np.stack([r[tie], g[tie], b[tie]], -1)[None])[0]
    out = q.astype(np.uint8)
    out[tie] = fp
    diff = [[int(a), int(c), int(d), int(e)] for a, c, d, e in zip(
        r[tie], g[tie], b[tie], fp) if int(e) != (299 * int(a) + 587 * int(c) + 114 * int(d) + 500) // 1000]
    assert sorted(diff) == sorted(gold["differs_from_integer_half_up"])
    assert sha(out) == gold["sha256"]


def test_c1_full_size_matches_reference():
    gold = load_json("configs.json")["c1/w15"]
    img = workloads.c1_image()
    assert sha(img) == gold["input"]
    b, t = oracle.binarize(img, 15, "sauvola", 0.5, 128.0, threads=4)
    assert sha(b) == gold["binary"]
    assert sha(t) == gold["tmap"]
    m, s, _ = oracle.mean_std(img, 15)
    assert sha(m) == gold["mean"] and sha(s) == gold["std"]


def test_c2_full_size_matches_reference():
    gold = load_json("configs.json")
    rgb = workloads.c2_rgb()
    assert sha(rgb) == gold["c2/rgb"]["input"]
    gray = oracle.to_gray(rgb)
    assert sha(gray) == gold["c2/rgb"]["gray"]
    for win in (15, 31, 63):
        b, _ = oracle.binarize(gray, win, "sauvola", 0.5, 128.0, tmap=False, threads=8)
        assert sha(b) == gold[f"c2/w{win}"]["binary"], win


@pytest.mark.slow
def test_c5_full_size_matches_reference():
    gold = load_json("configs.json")
    img = workloads.c5_image()
    for win in (3, 35, 243):
        g = gold.get(f"c5/w{win}")
        if g is None:
            pytest.skip("c5 goldens not generated")
        assert sha(img) == g["input"]
        b, t = oracle.binarize(img, win, "sauvola", 0.5, 128.0, tmap=True, threads=8)
        assert sha(b) == g["binary"]
        if "tmap" in g:
            assert sha(t) == g["tmap"]
