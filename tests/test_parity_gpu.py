"""GPU parity: the sm_100a kernels vs the reference's own outputs (golden fixtures)
and the CPU oracle, bit for bit.  Run on a B200: pytest -m gpu."""

import numpy as np
import pytest

import oracle
import paper_1210_3165_b200 as dt
from conftest import load_json, load_small, random_gray, sha
from paper_1210_3165_b200 import engine, workloads

pytestmark = pytest.mark.gpu

SMALL = load_small()
GOLD = load_json("configs.json")


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("case", SMALL, ids=lambda c: f"case{c['idx']}")
def test_binarize_matches_reference_small(case):
    kw = {"k_sauvola": case["k"]} if case["method"] == "sauvola" else {"k_niblack": case["k"]}
    for eng, mask in (("integral", "gs3"), ("naive", "gs3"), ("sampled", "full")):
        p = dt.BinarizationParams(method=case["method"], engine=eng, mask=mask,
                                  window=case["win"], r=case["r"], **kw)
        b, t = dt.binarize(case["img"], p)
        assert b.dtype == np.uint8 and np.array_equal(b, case["binary"]), eng
        assert np.array_equal(_bits(t), _bits(case["tmap"])), eng
        b2, t2 = dt.binarize(case["img"], p, return_tmap=False)
        assert t2 is None and np.array_equal(b2, case["binary"])


@pytest.mark.parametrize("case", SMALL, ids=lambda c: f"case{c['idx']}")
def test_mean_std_matches_reference_small(case):
    for fn in (dt.mean_std_integral, dt.mean_std_naive):
        m, s, c = fn(case["img"], case["win"])
        assert np.array_equal(_bits(m), _bits(case["mean"]))
        assert np.array_equal(_bits(s), _bits(case["std"]))
        assert c.dtype == np.int64 and np.array_equal(c, case["count"])
    m, s, c = dt.mean_std_sampled(case["img"], dt.make_mask("full", case["win"]))
    assert np.array_equal(_bits(m), _bits(case["mean"]))


def test_window_sums_exact_vs_oracle(rng):
    imgs = [random_gray(rng) for _ in range(6)] + [workloads.c1_image()[:300, :200]]
    for img in imgs:
        for win in (3, 15, 63, 127, 255, 513):
            S, Q, n = dt.window_sums(img, win)
            So, Qo, no = oracle.window_sums(img, win)
            assert np.array_equal(S, So) and np.array_equal(Q, Qo) and np.array_equal(n, no)


def test_wide_sums_beyond_uint32():
    # all-255 image with a window large enough that Q exceeds 2^32 -> 64-bit instantiation
    img = np.full((600, 700), 255, np.uint8)
    S, Q, n = dt.window_sums(img, 1001)
    assert Q.max() == 600 * 700 * 65025 > 2**32
    So, Qo, no = oracle.window_sums(img, 1001)
    assert np.array_equal(Q, Qo) and np.array_equal(S, So)


def test_c1_full_size():
    g = GOLD["c1/w15"]
    img = workloads.c1_image()
    assert sha(img) == g["input"]
    b, t = dt.binarize(img, dt.BinarizationParams(engine="integral", window=15, k_sauvola=0.5))
    assert sha(b) == g["binary"] and sha(t) == g["tmap"]
    m, s, _ = dt.mean_std_integral(img, 15)
    assert sha(m) == g["mean"] and sha(s) == g["std"]


def test_c2_to_gray_and_binarize():
    g = GOLD
    rgb = workloads.c2_rgb()
    assert sha(rgb) == g["c2/rgb"]["input"]
    gray = dt.to_gray(rgb)
    assert sha(gray) == g["c2/rgb"]["gray"]
    for win in (15, 31, 63):
        b, _ = dt.binarize(gray, dt.BinarizationParams(engine="integral", window=win,
                                                       k_sauvola=0.5), return_tmap=False)
        assert sha(b) == g[f"c2/w{win}"]["binary"], win
        fused, gdev = engine.rgb_binarize(rgb, win, "sauvola", 0.5, 128.0, want_gray=True)
        assert sha(fused.cpu().numpy()) == g[f"c2/w{win}"]["binary"], win
        assert sha(gdev.cpu().numpy()) == g["c2/rgb"]["gray"]


def test_c3_batch():
    torch = engine.torch_mod()
    imgs = [workloads.c3_image(i) for i in range(64)]
    stack = torch.from_numpy(np.stack(imgs)).cuda()
    out = engine.binarize_batch(stack, 31, "niblack", -0.2, 128.0).cpu().numpy()
    for i in range(64):
        g = GOLD[f"c3/img{i}"]
        assert sha(imgs[i]) == g["input"]
        assert sha(out[i]) == g["binary"], i


def test_c4_whole_and_bands():
    torch = engine.torch_mod()
    g = GOLD["c4/w127"]
    img = workloads.c4_image()
    assert sha(img) == g["input"]
    dev = torch.from_numpy(img).cuda()
    b, _ = engine.binarize(dev, 127, "sauvola", 0.34, 128.0, want_tmap=False)
    assert sha(b.cpu().numpy()) == g["binary"]
    # 8 virtual row bands, each from a buffer of band + 63-row halos (multi-GPU layout)
    H = img.shape[0]
    out = torch.empty_like(dev)
    for i in range(8):
        y0, y1 = H * i // 8, H * (i + 1) // 8
        a, z = max(y0 - 63, 0), min(y1 + 63, H)
        buf = dev[a:z].clone()
        engine.binarize_band(buf, a, H, y0, y1, 127, "sauvola", 0.34, 128.0, out=out[y0:y1])
    assert sha(out.cpu().numpy()) == g["binary"]


def test_c5_window_sweep():
    torch = engine.torch_mod()
    img = workloads.c5_image()
    dev = torch.from_numpy(img).cuda()
    for win in workloads.CONFIGS["c5"].windows:
        g = GOLD[f"c5/w{win}"]
        b, t = engine.binarize(dev, win, "sauvola", 0.5, 128.0, want_tmap="tmap" in g)
        assert sha(b.cpu().numpy()) == g["binary"], win
        if "tmap" in g:
            assert sha(t.cpu().numpy()) == g["tmap"]


def test_to_gray_exhaustive():
    r = np.repeat(np.arange(256, dtype=np.uint8), 65536)
    gg = np.tile(np.repeat(np.arange(256, dtype=np.uint8), 256), 256)
    b = np.tile(np.arange(256, dtype=np.uint8), 65536)
    rgb = np.stack([r, gg, b], axis=-1).reshape(4096, 4096, 3)
    assert sha(dt.to_gray(rgb).reshape(-1)) == load_json("to_gray.json")["sha256"]


def test_band_split_any_count(rng):
    img = workloads.c1_image()
    full, _ = dt.binarize(img, dt.BinarizationParams(engine="integral", window=31,
                                                     k_sauvola=0.5), return_tmap=False)
    H = img.shape[0]
    for nb in (2, 3, 7):
        parts = []
        for i in range(nb):
            y0, y1 = H * i // nb, H * (i + 1) // nb
            a, z = max(y0 - 15, 0), min(y1 + 15, H)
            parts.append(engine.binarize_band(img[a:z], a, H, y0, y1, 31, "sauvola", 0.5,
                                              128.0).cpu().numpy())
        assert np.array_equal(np.concatenate(parts), full)


def test_sampled_masks_match_gather_oracle(rng):
    from oracle import numpy_ref  # noqa: F401  (checker only)
    for structure in ("gs1", "gs2", "gs3", "gs4", "gs5", "gs6"):
        img = random_gray(rng, lo=8, hi=30)
        h, w = img.shape
        mask = dt.make_mask(structure, 7)
        m, s, c = dt.mean_std_sampled(img, mask)
        for y in range(h):
            for x in range(w):
                vals = np.array([int(img[y + dy, x + dx]) for dx, dy in mask.offsets
                                 if 0 <= x + dx < w and 0 <= y + dy < h], dtype=np.int64)
                S, Q, n = int(vals.sum()), int((vals * vals).sum()), len(vals)
                mean = S / n
                var = Q / n - mean * mean
                assert c[y, x] == n
                assert m[y, x] == mean and s[y, x] == np.sqrt(max(var, 0.0))


def test_default_params_sampled_gs3(rng):
    img = random_gray(rng)
    b, t = dt.binarize(img)  # reference defaults: sauvola / sampled / gs3 / W=21
    m, s, _ = dt.mean_std_sampled(img, dt.make_mask("gs3", 21))
    assert np.array_equal(t, m * (1.0 + 0.34 * (s / 128.0 - 1.0)))
    assert np.array_equal(b == 0, img.astype(float) < t)


def _brute_force_otsu(img):
    hist = np.bincount(np.asarray(img).ravel(), minlength=256)
    total = int(hist.sum())
    total_sum = int(np.dot(hist, np.arange(256)))
    best_t, best_num, best_den = None, -1, 1
    wb = sumb = 0
    for t in range(1, 256):
        wb += int(hist[t - 1])
        sumb += (t - 1) * int(hist[t - 1])
        wf = total - wb
        if wb == 0 or wf == 0:
            continue
        num = (sumb * wf - (total_sum - sumb) * wb) ** 2
        den = wb * wf
        if num * best_den > best_num * den:
            best_t, best_num, best_den = t, num, den
    return best_t


def test_otsu(rng):
    assert dt.otsu_threshold(np.array([[10] * 50 + [200] * 50], np.uint8)) == 11
    assert dt.otsu_threshold(np.full((4, 7), 77, np.uint8)) == 77
    assert dt.otsu_threshold(np.array([[0, 255]], np.uint8)) == 1
    for _ in range(20):
        img = random_gray(rng)
        assert dt.otsu_threshold(img) == _brute_force_otsu(img)
    img = random_gray(rng)
    b, t = dt.binarize(img, dt.BinarizationParams(method="otsu"))
    T = dt.otsu_threshold(img)
    assert (t == float(T)).all() and np.array_equal(b, np.where(img < T, 0, 255))


def test_estimators_match_functional(rng):
    img = random_gray(rng)
    est = dt.LocalBinarizer(method="sauvola", engine="integral", window=9, k=0.4)
    p = dt.BinarizationParams(method="sauvola", engine="integral", window=9, k_sauvola=0.4)
    assert np.array_equal(est.fit(img).transform(img), dt.binarize(img, p)[0])
    o = dt.OtsuBinarizer().fit(img)
    assert np.array_equal(o.transform(img), dt.apply_global(img, o.threshold_))


def test_scalar_window_stats(rng):
    img = random_gray(rng, lo=8, hi=20)
    ip = dt.build_integral(img)
    So, Qo, _ = oracle.window_sums(img, 3)
    assert ip.sum_table[1:, 1:].sum() >= 0
    a = np.asarray(img, dtype=np.int64)
    assert np.array_equal(ip.sum_table[1:, 1:], a.cumsum(0).cumsum(1))
    assert np.array_equal(ip.sqsum_table[1:, 1:], (a * a).cumsum(0).cumsum(1))
    for (x, y) in ((0, 0), (3, 4), (img.shape[1] - 1, img.shape[0] - 1)):
        a1 = dt.window_stats_naive(img, x, y, 7)
        b1 = dt.window_stats_integral(ip, x, y, 7)
        assert a1 == b1
    st = dt.window_stats_naive(np.array([[42]], np.uint8), 0, 0, 3)
    assert st == (42.0, 0.0, 1)


def test_device_tensor_in_device_tensor_out():
    torch = engine.torch_mod()
    img = workloads.c1_image()
    dev = torch.from_numpy(img).cuda()
    b, t = dt.binarize(dev, dt.BinarizationParams(engine="integral", window=15, k_sauvola=0.5))
    assert b.is_cuda and t.is_cuda
    assert sha(b.cpu().numpy()) == GOLD["c1/w15"]["binary"]
