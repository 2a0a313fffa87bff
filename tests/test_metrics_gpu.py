"""evaluate() / sweep() on the GPU against the reference's own
outputs (tests/golden/metrics.npz) and the reference test-suite's properties
(/root/reference/pkg/tests/test_metrics.py)."""

import numpy as np
import pytest

import paper_1210_3165_b200 as dt
from conftest import load_metrics, load_sampled, sha

pytestmark = pytest.mark.gpu

EVAL, PAGES, SWEEPS = load_metrics()
SAMPLED = load_sampled()


def random_binary(rng, h=16, w=16, fg_fraction=0.3):
    img = np.where(rng.random((h, w)) < fg_fraction, 0, 255).astype(np.uint8)
    if not (img == 0).any():
        img[0, 0] = 0
    return img


@pytest.mark.parametrize("case", EVAL, ids=lambda c: f"eval{c['idx']}")
def test_evaluate_matches_reference(case):
    rep = dt.evaluate(case["pred"], case["gt"])
    assert [rep.tp, rep.tn, rep.fp, rep.fn, rep.recall, rep.precision,
            rep.f_measure] == case["expect"]


@pytest.mark.parametrize("case", SWEEPS, ids=lambda c: f"sweep{c['idx']}-{c['method']}-{c['engine']}-{c['mask']}")
def test_sweep_matches_reference(case):
    img, gt = PAGES[case["page"]]
    kw = {} if case["w_grid"] is None else {"w_grid": case["w_grid"], "k_grid": case["k_grid"]}
    res = dt.sweep(img, gt, method=case["method"], engine=case["engine"], mask=case["mask"],
                   r=case["r"], **kw)
    assert [[c.w, c.k, c.f_measure] for c in res.cells] == case["cells"]
    assert [res.best.w, res.best.k, res.best.f_measure] == case["best"]
    assert res.to_csv() == case["csv"]


def test_identity_is_perfect(rng):
    for _ in range(10):
        x = random_binary(rng)
        rep = dt.evaluate(x, x)
        assert (rep.recall, rep.precision, rep.f_measure) == (1.0, 1.0, 1.0)
        assert rep.fp == 0 and rep.fn == 0


def test_half_recall_frozen_counts():
    gt = np.full((5, 4), 255, dtype=np.uint8)
    gt.ravel()[:10] = 0
    pred = np.full((5, 4), 255, dtype=np.uint8)
    pred.ravel()[:5] = 0
    rep = dt.evaluate(pred, gt)
    assert (rep.tp, rep.fp, rep.fn, rep.tn) == (5, 0, 5, 10)
    assert rep.recall == 0.5 and rep.precision == 1.0
    assert rep.f_measure == pytest.approx(2 / 3, abs=1e-15)


def test_degenerate_predictions_score_zero_not_nan():
    gt = np.zeros((3, 3), dtype=np.uint8)
    pred = np.full((3, 3), 255, dtype=np.uint8)
    rep = dt.evaluate(pred, gt)
    assert rep.tp == 0 and (rep.recall, rep.precision, rep.f_measure) == (0.0, 0.0, 0.0)
    empty = np.full((3, 3), 255, dtype=np.uint8)
    rep = dt.evaluate(empty, empty)
    assert (rep.recall, rep.precision, rep.f_measure) == (0.0, 0.0, 0.0)


def test_evaluate_rejects_bad_input():
    with pytest.raises(ValueError, match="shape"):
        dt.evaluate(np.zeros((2, 2), np.uint8), np.zeros((2, 3), np.uint8))
    with pytest.raises(ValueError, match=r"not a bi-level image: pixel \(0, 0\) has value 7"):
        dt.evaluate(np.full((2, 2), 7, np.uint8), np.zeros((2, 2), np.uint8))
    gt = np.zeros((3, 5), np.uint8)
    gt[2, 3] = 9
    gt[2, 4] = 8
    with pytest.raises(ValueError, match=r"pixel \(3, 2\) has value 9"):
        dt.evaluate(np.zeros((3, 5), np.uint8), gt)
    # pred is validated before the shape check
    with pytest.raises(ValueError, match="bi-level"):
        dt.evaluate(np.full((2, 2), 7, np.uint8), np.zeros((2, 3), np.uint8))


def test_evaluate_large_and_device_inputs(rng):
    import torch
    pred = random_binary(rng, 1531, 2047, 0.2)
    gt = random_binary(rng, 1531, 2047, 0.25)
    from oracle import numpy_ref
    want = list(numpy_ref.evaluate_counts(pred, gt))
    rep = dt.evaluate(pred, gt)
    assert [rep.tp, rep.tn, rep.fp, rep.fn, rep.recall, rep.precision, rep.f_measure] == want
    dp, dg = torch.from_numpy(pred).cuda(), torch.from_numpy(gt).cuda()
    rep2 = dt.evaluate(dp[:, 1:], dg[:, 1:])  # strided device views
    want2 = list(numpy_ref.evaluate_counts(pred[:, 1:], gt[:, 1:]))
    assert [rep2.tp, rep2.tn, rep2.fp, rep2.fn, rep2.recall, rep2.precision,
            rep2.f_measure] == want2


def test_summary_format():
    x = np.array([[0, 255]], dtype=np.uint8)
    text = dt.evaluate(x, x).summary()
    assert "FM = 100.00%" in text and "R = 100.00%" in text and "TP = 1" in text


def test_sweep_all_tied_picks_smallest_cell():
    img = np.full((16, 16), 200, dtype=np.uint8)
    gt = np.full((16, 16), 255, dtype=np.uint8)
    res = dt.sweep(img, gt, engine="naive", w_grid=[5, 3], k_grid=[0.4, 0.2])
    assert all(c.f_measure == 0.0 for c in res.cells)
    assert (res.best.w, res.best.k) == (3, 0.2)


def test_sweep_matches_direct_binarize():
    img, gt = PAGES[0]
    res = dt.sweep(img, gt, method="sauvola", engine="sampled", mask="gs2",
                   w_grid=[11, 21], k_grid=[0.2, 0.4])
    for cell in res.cells:
        p = dt.BinarizationParams(method="sauvola", engine="sampled", mask="gs2",
                                  window=cell.w, k_sauvola=cell.k)
        assert cell.f_measure == dt.evaluate(dt.binarize(img, p)[0], gt).f_measure


def test_sweep_long_k_grid_chunks(rng):
    """More k values than one launch holds (64) and than one CTA row (8)."""
    img, gt = PAGES[1]
    ks = sorted(set(np.round(rng.uniform(0.01, 0.9, 150), 4).tolist()))
    res = dt.sweep(img, gt, engine="integral", w_grid=[15], k_grid=ks)
    from oracle import numpy_ref
    cells, best = numpy_ref.sweep(img, gt, "sauvola", "integral", "gs3", [15], ks)
    assert [tuple(c) for c in res.cells] == [tuple(c) for c in cells]
    assert tuple(res.best) == tuple(best)


def test_sweep_errors_name_the_cell():
    img, gt = PAGES[0]
    with pytest.raises(ValueError, match=r"sweep cell \(W=11, k=-1.0\)"):
        dt.sweep(img, gt, method="sauvola", engine="naive", w_grid=[11], k_grid=[-1.0])
    with pytest.raises(ValueError, match="non-empty"):
        dt.sweep(img, gt, w_grid=[], k_grid=[0.3])
    bad = gt.copy()
    bad[4, 5] = 3
    with pytest.raises(ValueError, match=r"pixel \(5, 4\) has value 3"):
        dt.sweep(img, bad)
    with pytest.raises(ValueError, match="shape mismatch"):
        dt.sweep(img, gt[:, 1:])


@pytest.mark.parametrize("case", SAMPLED, ids=lambda c: f"{c['structure']}-w{c['win']}-{c['idx']}")
def test_sampled_engine_matches_reference(case):
    img = case["img"]
    if "mean" in case:
        m, s, n = dt.mean_std_sampled(img, dt.make_mask(case["structure"], case["win"]))
        assert sha(m) == case["mean"]
        assert sha(s) == case["std"]
        assert sha(n.astype(np.int64)) == case["count"]
    kw = {"k_sauvola": case["k"]} if case["method"] == "sauvola" else {"k_niblack": case["k"]}
    p = dt.BinarizationParams(method=case["method"], engine="sampled", mask=case["structure"],
                              window=case["win"], **kw)
    b, t = dt.binarize(img, p)
    assert sha(b) == case["binary"]
    assert sha(t) == case["tmap"]


def test_otsu_device_scan_matches_reference():
    """§8 row f3: device histogram + fp64 scan == the reference's T on its own images."""
    from conftest import load_otsu
    for img, t in load_otsu():
        assert dt.otsu_threshold(img) == t
        b, tm = dt.binarize(img, dt.BinarizationParams(method="otsu"))
        assert np.array_equal(b, np.where(img < t, 0, 255).astype(np.uint8))
        assert tm.dtype == np.float64 and np.all(tm == float(t))


def test_otsu_large_and_strided(rng):
    import torch
    from oracle import numpy_ref
    img = rng.integers(0, 256, (2049, 3001)).astype(np.uint8)
    img[:1000] = np.clip(img[:1000] // 4, 0, 255)
    assert dt.otsu_threshold(img) == numpy_ref.otsu_threshold(img)
    dev = torch.from_numpy(img).cuda()[3:, 5:]  # unaligned -> scalar histogram path
    assert dt.otsu_threshold(dev) == numpy_ref.otsu_threshold(img[3:, 5:])
    b, t = dt.binarize(dev, dt.BinarizationParams(method="otsu"), return_tmap=False)
    T = numpy_ref.otsu_threshold(img[3:, 5:])
    assert t is None and torch.equal(b.cpu(), torch.from_numpy(np.where(img[3:, 5:] < T, 0, 255).astype(np.uint8)))
