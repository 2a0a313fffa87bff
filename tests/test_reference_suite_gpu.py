"""The reference's own unit-test contracts for statistics and thresholding
(/root/reference/pkg/tests/test_stats.py, test_threshold.py), restated against this
package and run on the GPU path.  The known answers are the reference tests' spot values."""

import numpy as np
import pytest

import paper_1210_3165_b200 as dt
from conftest import load_metrics, random_gray

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- statistics (test_stats.py)

def test_window_stats_spot_values():
    img = np.full((7, 9), 100, dtype=np.uint8)
    for x, y in [(0, 0), (4, 3), (8, 6)]:
        st = dt.window_stats_naive(img, x, y, 5)
        assert (st.mean, st.std) == (100.0, 0.0)
    g = np.arange(9, dtype=np.uint8).reshape(3, 3)
    st = dt.window_stats_naive(g, 1, 1, 3)
    assert st.mean == 4.0 and st.count == 9 and st.std == pytest.approx((60 / 9) ** 0.5, abs=1e-12)
    st = dt.window_stats_naive(g, 0, 0, 3)  # clipped to {0, 1, 3, 4}
    assert st.mean == 2.0 and st.count == 4 and st.std == pytest.approx(2.5 ** 0.5, abs=1e-12)
    st = dt.window_stats_sampled(np.arange(25, dtype=np.uint8).reshape(5, 5),
                                 dt.make_mask("gs1", 5), 2, 2)
    assert st.mean == 12.0 and st.count == 9
    assert st.std == pytest.approx((1556 / 9 - 144) ** 0.5, abs=1e-12)
    assert dt.window_stats_naive(np.array([[42]], np.uint8), 0, 0, 3) == (42.0, 0.0, 1)


def test_build_integral_values_and_monotone(rng):
    one = dt.build_integral(np.array([[7]], dtype=np.uint8))
    assert one.sum_table[1, 1] == 7 and one.sqsum_table[1, 1] == 49
    zero = dt.build_integral(np.zeros((3, 4), dtype=np.uint8))
    assert not zero.sum_table.any() and not zero.sqsum_table.any()
    two = dt.build_integral(np.array([[1, 2], [3, 4]], dtype=np.uint8))
    assert two.sum_table[2, 2] == 10 and two.sqsum_table[2, 2] == 30
    assert two.sum_table[0].tolist() == [0, 0, 0] and two.sum_table[:, 0].tolist() == [0, 0, 0]
    ip = dt.build_integral(random_gray(rng, lo=10, hi=30))
    for table in ip:
        assert (np.diff(table, axis=0) >= 0).all() and (np.diff(table, axis=1) >= 0).all()


def test_full_image_engines_agree_bitwise(rng):
    for _ in range(10):
        img = random_gray(rng)
        win = int(rng.choice([3, 5, 9, 15, 21, 31]))
        mn, sn, cn = dt.mean_std_naive(img, win)
        mi, si, ci = dt.mean_std_integral(img, win)
        ms, ss, cs = dt.mean_std_sampled(img, dt.make_mask("full", win))
        for a, b in ((mn, mi), (sn, si), (cn, ci), (mn, ms), (sn, ss), (cn, cs)):
            assert (a == b).all()


def test_full_image_matches_per_pixel(rng):
    img = random_gray(rng, lo=10, hi=16)
    mn, sn, cn = dt.mean_std_naive(img, 5)
    mask = dt.make_mask("gs5", 5)
    ms, ss, cs = dt.mean_std_sampled(img, mask)
    for y in range(img.shape[0]):
        for x in range(img.shape[1]):
            assert tuple(dt.window_stats_naive(img, x, y, 5)) == (mn[y, x], sn[y, x], cn[y, x])
            assert tuple(dt.window_stats_sampled(img, mask, x, y)) == (ms[y, x], ss[y, x], cs[y, x])


def test_shift_invariance_bounds_and_counts(rng):
    img = rng.integers(0, 200, size=(23, 17)).astype(np.uint8)
    shifted = (img + 30).astype(np.uint8)
    mask = dt.make_mask("gs2", 7)
    for f in (lambda im: dt.mean_std_naive(im, 7), lambda im: dt.mean_std_integral(im, 7),
              lambda im: dt.mean_std_sampled(im, mask)):
        m0, s0, _ = f(img)
        m1, s1, _ = f(shifted)
        assert np.abs((m1 - m0) - 30.0).max() <= 1e-6 and np.abs(s1 - s0).max() <= 1e-6
    extremes = np.zeros((16, 16), dtype=np.uint8)
    extremes[:, 8:] = 255
    for im in (extremes, random_gray(rng)):
        for win in (3, 9, 21):
            m, s, _ = dt.mean_std_naive(im, win)
            assert not np.isnan(s).any() and 0.0 <= s.min() and s.max() <= 127.5
            assert m.min() >= 0.0 and m.max() <= 255.0
    small = random_gray(rng, h=9, w=9)
    for st in ("gs1", "gs2", "gs3", "gs4", "gs5", "gs6", "full"):
        assert dt.mean_std_sampled(small, dt.make_mask(st, 21))[2].min() >= 1


def test_coordinate_and_window_errors(rng):
    img = random_gray(rng, h=5, w=5)
    with pytest.raises(ValueError, match="coordinates"):
        dt.window_stats_naive(img, 5, 0, 3)
    with pytest.raises(ValueError, match="coordinates"):
        dt.window_stats_sampled(img, dt.make_mask("gs1", 3), 0, -1)
    with pytest.raises(ValueError, match="coordinates"):
        dt.window_stats_integral(dt.build_integral(img), 0, 9, 3)
    with pytest.raises(ValueError, match="window"):
        dt.window_stats_naive(img, 0, 0, 4)
    with pytest.raises(ValueError, match="window"):
        dt.mean_std_integral(img, 2)


# ---------------------------------------------------------------- thresholds (test_threshold.py)

def test_threshold_spot_values_and_errors():
    W = dt.WindowStats
    assert dt.sauvola_threshold_at(W(100.0, 0.0, 9), 0.5, 128.0) == 50.0
    assert dt.sauvola_threshold_at(W(0.0, 30.0, 9), 0.34, 128.0) == 0.0
    assert dt.sauvola_threshold_at(W(128.0, 128.0, 9), 0.34, 128.0) == 128.0
    assert dt.niblack_threshold_at(W(100.0, 20.0, 9), -0.2) == 96.0
    assert dt.niblack_threshold_at(W(123.0, 0.0, 9), -5.0) == 123.0
    assert dt.niblack_threshold_at(W(123.0, 50.0, 9), 0.0) == 123.0
    with pytest.raises(ValueError, match="k"):
        dt.sauvola_threshold_at(W(100.0, 10.0, 9), 0.0, 128.0)
    with pytest.raises(ValueError, match="r"):
        dt.sauvola_threshold_at(W(100.0, 10.0, 9), 0.3, 0.0)


def test_apply_global_boundaries_and_errors():
    img = np.array([[0, 99, 100, 101, 255]], dtype=np.uint8)
    assert dt.apply_global(img, 100).tolist() == [[0, 0, 255, 255, 255]]
    assert (dt.apply_global(img, 0) == 255).all()
    assert dt.apply_global(img, 255).tolist() == [[0, 0, 0, 0, 255]]
    for bad in (-1, 256, 10.5):
        with pytest.raises(ValueError, match="threshold"):
            dt.apply_global(img, bad)


def test_binarize_bilevel_constant_and_deterministic(rng):
    img = random_gray(rng)
    for method in ("otsu", "niblack", "sauvola"):
        b, t = dt.binarize(img, dt.BinarizationParams(method=method, window=5))
        assert b.dtype == np.uint8 and set(np.unique(b)) <= {0, 255} and t.shape == img.shape
    const = np.full((9, 9), 120, dtype=np.uint8)
    for eng in ("naive", "integral", "sampled"):
        b, t = dt.binarize(const, dt.BinarizationParams(method="sauvola", engine=eng, window=5))
        assert (b == 255).all() and (t < 120).all()
    b, _ = dt.binarize(const, dt.BinarizationParams(method="niblack", window=5))
    assert (b == 255).all()
    a1, t1 = dt.binarize(img)
    a2, t2 = dt.binarize(img)
    assert np.array_equal(a1, a2) and (t1 == t2).all()


def test_binarize_tmap_formula_and_otsu_path(rng):
    img = random_gray(rng)
    p = dt.BinarizationParams(method="sauvola", engine="sampled", mask="gs3", window=9,
                              k_sauvola=0.4, r=100.0)
    b, t = dt.binarize(img, p)
    m, s, _ = dt.mean_std_sampled(img, dt.make_mask("gs3", 9))
    assert (t == m * (1.0 + 0.4 * (s / 100.0 - 1.0))).all()
    assert np.array_equal(b == 0, img.astype(float) < t)
    b, t = dt.binarize(img, dt.BinarizationParams(method="otsu"))
    T = dt.otsu_threshold(img)
    assert (t == float(T)).all() and np.array_equal(b, dt.apply_global(img, T))


def test_sauvola_k_monotonicity():
    _, pages, _ = load_metrics()
    img = pages[0][0]  # the reference's gen_synthetic() page
    prev = None
    for k in (0.1, 0.2, 0.34, 0.5):
        fg = dt.binarize(img, dt.BinarizationParams(method="sauvola", engine="naive", window=21,
                                                    k_sauvola=k))[0] == 0
        if prev is not None:
            assert (fg <= prev).all()
        prev = fg


def test_params_validation_names_field():
    img = np.zeros((5, 5), dtype=np.uint8)
    for params, field in [(dt.BinarizationParams(method="bogus"), "method"),
                          (dt.BinarizationParams(engine="gpu"), "engine"),
                          (dt.BinarizationParams(window=8), "window"),
                          (dt.BinarizationParams(k_sauvola=-0.1), "k_sauvola"),
                          (dt.BinarizationParams(r=0.0), "r"),
                          (dt.BinarizationParams(engine="sampled", mask="nope"), "mask")]:
        with pytest.raises(ValueError, match=field):
            dt.binarize(img, params)
