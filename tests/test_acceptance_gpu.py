"""The reference's acceptance gates that concern the hot path (test_acceptance.py: AC1, AC5,
AC6, AC7), run on the GPU path.  AC5 additionally pins every page's Otsu F-measure and
best sweep cell to the values the reference produced (tests/golden/acceptance.npz).
AC2-AC4 measure the reference's own CPU engines' timing / memory model (out of scope)."""

import json
import os

import numpy as np
import pytest

import paper_1210_3165_b200 as dt
from conftest import GOLDEN

pytestmark = pytest.mark.gpu
GS_STRUCTURES = ("gs1", "gs2", "gs3", "gs4", "gs5", "gs6")


def test_ac1_engine_equivalence_on_random_images():
    """test_acceptance.py:42-86 (without the CPU-time budget; screening kept)."""
    rng = np.random.default_rng(20260821)
    windows = (3, 5, 9, 15, 21)
    done = 0
    while done < 200:
        h, w = int(rng.integers(8, 65)), int(rng.integers(8, 65))
        img = rng.integers(0, 256, size=(h, w)).astype(np.uint8)
        win = windows[done % len(windows)]
        mean, std, _ = dt.mean_std_naive(img, win)
        imgf = img.astype(np.float64)
        t_s = mean * (1.0 + 0.34 * (std / 128.0 - 1.0))
        t_n = mean - 0.2 * std
        if min(np.abs(imgf - t_s).min(), np.abs(imgf - t_n).min()) <= 1e-6:
            continue
        for method in ("sauvola", "niblack"):
            outs = [dt.binarize(img, dt.BinarizationParams(method=method, engine=e, mask=m,
                                                           window=win))[0]
                    for e, m in (("naive", "gs3"), ("integral", "gs3"), ("sampled", "full"))]
            assert all(np.array_equal(outs[0], o) for o in outs[1:])
        done += 1


def test_ac5_accuracy_proxy_matches_reference():
    """test_acceptance.py:165-199 on the reference's own corpus, cell values pinned."""
    z = np.load(os.path.join(GOLDEN, "acceptance.npz"))
    meta = json.loads(str(z["meta"]))
    for i, m in enumerate(meta):
        img, gt = z[f"img{i}"], z[f"gt{i}"]
        otsu_fm = dt.evaluate(dt.apply_global(img, dt.otsu_threshold(img)), gt).f_measure
        assert otsu_fm == m["otsu_fm"]
        naive = dt.sweep(img, gt, method="sauvola", engine="naive").best
        assert [naive.w, naive.k, naive.f_measure] == m["naive"]
        assert naive.f_measure > otsu_fm
        for st in GS_STRUCTURES:
            b = dt.sweep(img, gt, method="sauvola", engine="sampled", mask=st).best
            assert [b.w, b.k, b.f_measure] == m["gs"][st], (i, st)
            assert abs(naive.f_measure - b.f_measure) * 100.0 <= 2.0
            assert b.f_measure > otsu_fm


def test_ac6_self_evaluation_is_exactly_perfect():
    rng = np.random.default_rng(99)
    images = [np.array([[0]], dtype=np.uint8), np.where(np.eye(7) > 0, 0, 255).astype(np.uint8),
              np.zeros((12, 5), dtype=np.uint8)]
    for _ in range(10):
        h, w = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        img = np.where(rng.random((h, w)) < 0.4, 0, 255).astype(np.uint8)
        if not (img == 0).any():
            img[0, 0] = 0
        images.append(img)
    for img in images:
        rep = dt.evaluate(img, img)
        assert (rep.recall, rep.precision, rep.f_measure) == (1.0, 1.0, 1.0)


def test_ac7_formula_spot_values():
    assert int(dt.to_gray(np.array([[[255, 0, 0]]], dtype=np.uint8))[0, 0]) == 76
    assert int(dt.apply_global(np.array([[100]], dtype=np.uint8), 100)[0, 0]) == 255
    assert dt.sauvola_threshold_at(dt.WindowStats(100.0, 0.0, 9), 0.5, 128.0) == 50.0
