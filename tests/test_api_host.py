"""Host-side contract of the drop-in API (no GPU): validation messages match the
reference (threshold.py:40-52, validation.py:8-57), masks, params defaults."""

import numpy as np
import pytest

import paper_1210_3165_b200 as dt


def test_params_defaults_match_reference():
    p = dt.BinarizationParams()
    assert (p.method, p.engine, p.mask, p.window, p.k_sauvola, p.k_niblack, p.r) == (
        "sauvola", "sampled", "gs3", 21, 0.34, -0.2, 128.0)
    assert dt.METHODS == ("otsu", "niblack", "sauvola")
    assert dt.ENGINES == ("naive", "integral", "sampled")


def test_params_validation_names_field():
    # reference test_threshold.py:205-217; fails before any device work
    img = np.zeros((5, 5), dtype=np.uint8)
    cases = [
        (dt.BinarizationParams(method="bogus"), "method"),
        (dt.BinarizationParams(engine="gpu"), "engine"),
        (dt.BinarizationParams(window=8), "window"),
        (dt.BinarizationParams(k_sauvola=-0.1), "k_sauvola"),
        (dt.BinarizationParams(r=0.0), "r"),
        (dt.BinarizationParams(engine="sampled", mask="nope"), "mask"),
    ]
    for params, field in cases:
        with pytest.raises(ValueError, match=field):
            dt.binarize(img, params)


def test_gray_image_contract():
    with pytest.raises(ValueError, match="2-D"):
        dt.binarize(np.zeros((3, 3, 3), np.uint8))
    with pytest.raises(ValueError, match="empty"):
        dt.binarize(np.zeros((0, 4), np.uint8))
    with pytest.raises(ValueError, match="integers"):
        dt.binarize(np.full((3, 3), 1.5))
    with pytest.raises(ValueError, match=r"\[0, 255\]"):
        dt.binarize(np.full((3, 3), 300))
    assert dt.as_gray_image(np.full((2, 2), 7.0)).dtype == np.uint8


def test_window_contract():
    for bad in (2, 4, 1, True, 3.0, "5"):
        with pytest.raises(ValueError, match="window"):
            dt.check_window(bad)
    assert dt.check_window(np.int64(5)) == 5


def test_apply_global_rejects_bad_threshold():
    img = np.zeros((2, 2), dtype=np.uint8)
    for t in (256, -1, 10.5):
        with pytest.raises(ValueError, match="threshold"):
            dt.apply_global(img, t)


def test_to_gray_rejects_gray_input():
    with pytest.raises(ValueError):
        dt.to_gray(np.zeros((4, 4), dtype=np.uint8))


@pytest.mark.parametrize("structure,formula", [
    ("gs1", lambda w: 2 * w - 1), ("gs2", lambda w: 2 * w - 1), ("gs3", lambda w: 4 * w - 3),
    ("gs4", lambda w: 3 * w - 2), ("gs5", lambda w: 4 * w - 3), ("gs6", lambda w: 6 * w - 9),
    ("full", lambda w: w * w)])
def test_mask_sizes(structure, formula):
    for w in (3, 5, 7, 21, 63):
        m = dt.make_mask(structure, w)
        assert len(m) == formula(w) == dt.mask_size(structure, w)
        assert (0, 0) in m.offsets
        assert list(m.offsets) == sorted(m.offsets, key=lambda o: (o[1], o[0]))


def test_mask_names_and_ascii():
    assert dt.make_mask("GS-3", 5).structure == "gs3"
    with pytest.raises(ValueError, match="unknown mask"):
        dt.make_mask("gs9", 5)
    art = dt.mask_to_ascii(dt.make_mask("gs1", 3))
    assert art == ".#.\n###\n.#."


def test_threshold_spot_values():
    ws = dt.WindowStats
    assert dt.sauvola_threshold_at(ws(100.0, 0.0, 9), 0.5, 128.0) == 50.0
    assert dt.sauvola_threshold_at(ws(128.0, 128.0, 9), 0.34, 128.0) == 128.0
    assert dt.niblack_threshold_at(ws(100.0, 20.0, 9), -0.2) == 96.0
    with pytest.raises(ValueError, match="k"):
        dt.sauvola_threshold_at(ws(100.0, 10.0, 9), 0.0, 128.0)


def test_pnm_codec_round_trip(rng):
    for _ in range(10):
        h, w = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        img = rng.integers(0, 256, size=(h, w)).astype(np.uint8)
        assert np.array_equal(dt.read_pnm(dt.write_pnm(img)), img)
    assert dt.read_pnm(b"P3 2 1 255  255 0 0  0 255 0")[0, 1].tolist() == [0, 255, 0]
    with pytest.raises(dt.PnmError, match=r"truncated payload at byte \d+"):
        dt.read_pnm(b"P5 2 2 255 " + bytes([1, 2, 3]))
    with pytest.raises(dt.PnmError, match="maxval"):
        dt.read_pnm(b"P5 1 1 65535 " + bytes([0, 0]))


def test_gen_synthetic_matches_reference_pages():
    # tests/golden/metrics.npz holds pages made by the reference's own gen_synthetic
    import numpy as np
    from conftest import GOLDEN
    import os
    from paper_1210_3165_b200 import SyntheticSpec, gen_synthetic, memory_model
    z = np.load(os.path.join(GOLDEN, "metrics.npz"))
    specs = [SyntheticSpec(), SyntheticSpec(width=300, height=180, noise_seed=3, noise_amplitude=20)]
    for i, sp in enumerate(specs):
        img, gt = gen_synthetic(sp)
        assert np.array_equal(img, z[f"page{i}"]) and np.array_equal(gt, z[f"page_gt{i}"])
    assert memory_model("integral", 10) == 120
    with pytest.raises(ValueError, match="engine"):
        memory_model("fast", 10)
    with pytest.raises(ValueError, match="too small"):
        gen_synthetic(SyntheticSpec(width=8))


def test_to_gray_refuses_non_byte_channels_without_a_gpu_call():
    import numpy as np
    from paper_1210_3165_b200 import to_gray
    with pytest.raises(ValueError, match="to_gray"):
        to_gray(np.full((2, 2, 3), 300, dtype=np.int32))
    with pytest.raises(ValueError, match="to_gray"):
        to_gray(np.full((2, 2, 3), 0.5))
