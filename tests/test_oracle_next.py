"""Oracle restatements for SURVEY.md §8 rows f1 (GS-mask sampled engine) and f2
(evaluate / sweep), pinned against fixtures produced by the reference itself
(tests/golden/make_golden.py --only sampled|metrics)."""

import numpy as np
import pytest

from conftest import load_metrics, load_sampled, sha
from oracle import numpy_ref

SAMPLED = load_sampled()
EVAL, PAGES, SWEEPS = load_metrics()


@pytest.mark.parametrize("case", [c for c in SAMPLED if "mean" in c][::2],
                         ids=lambda c: f"{c['structure']}-w{c['win']}-{c['idx']}")
def test_sampled_oracle_matches_reference(case):
    m, s, n = numpy_ref.mean_std_sampled(case["img"], case["structure"], case["win"])
    assert sha(m) == case["mean"]
    assert sha(s) == case["std"]
    assert sha(n.astype(np.int64)) == case["count"]
    t = numpy_ref.threshold_map(m, s, case["method"], case["k"])
    b = np.where(case["img"].astype(np.float64) < t, 0, 255).astype(np.uint8)
    assert sha(b) == case["binary"]
    assert sha(t) == case["tmap"]


@pytest.mark.parametrize("structure,formula", [
    ("gs1", lambda w: 2 * w - 1), ("gs2", lambda w: 2 * w - 1), ("gs3", lambda w: 4 * w - 3),
    ("gs4", lambda w: 3 * w - 2), ("gs5", lambda w: 4 * w - 3), ("gs6", lambda w: 6 * w - 9),
    ("full", lambda w: w * w)])
def test_oracle_mask_sizes(structure, formula):
    for w in (3, 5, 21, 127):
        assert len(numpy_ref.mask_offsets(structure, w)) == formula(w)


@pytest.mark.parametrize("case", EVAL, ids=lambda c: f"eval{c['idx']}")
def test_evaluate_oracle_matches_reference(case):
    got = numpy_ref.evaluate_counts(case["pred"], case["gt"])
    assert list(got) == case["expect"]


@pytest.mark.parametrize("case", [c for c in SWEEPS if c["method"] != "otsu"],
                         ids=lambda c: f"sweep{c['idx']}-{c['method']}-{c['engine']}-{c['mask']}")
def test_sweep_oracle_matches_reference(case):
    from paper_1210_3165_b200.metrics import DEFAULT_K_GRID, DEFAULT_W_GRID
    img, gt = PAGES[case["page"]]
    cells, best = numpy_ref.sweep(img, gt, case["method"], case["engine"], case["mask"],
                                  case["w_grid"] or DEFAULT_W_GRID,
                                  case["k_grid"] or DEFAULT_K_GRID, case["r"])
    assert [list(c) for c in cells] == case["cells"]
    assert list(best) == case["best"]


def test_otsu_oracle_matches_reference():
    from conftest import load_otsu
    for img, t in load_otsu():
        assert numpy_ref.otsu_threshold(img) == t


def test_sweep_oracle_matches_reference_acceptance_corpus():
    """The AC5 corpus (tests/golden/acceptance.npz): oracle sweep bests == the reference's."""
    import json
    import os
    from conftest import GOLDEN
    from paper_1210_3165_b200.metrics import DEFAULT_K_GRID, DEFAULT_W_GRID
    z = np.load(os.path.join(GOLDEN, "acceptance.npz"))
    meta = json.loads(str(z["meta"]))
    for i in (0, 7):
        img, gt = z[f"img{i}"], z[f"gt{i}"]
        _, best = numpy_ref.sweep(img, gt, "sauvola", "naive", "gs3", DEFAULT_W_GRID, DEFAULT_K_GRID)
        assert list(best) == meta[i]["naive"]
        _, best = numpy_ref.sweep(img, gt, "sauvola", "sampled", "gs5", DEFAULT_W_GRID, DEFAULT_K_GRID)
        assert list(best) == meta[i]["gs"]["gs5"]
        t = numpy_ref.otsu_threshold(img)
        assert numpy_ref.evaluate_counts(np.where(img < t, 0, 255), gt)[6] == meta[i]["otsu_fm"]
