"""Block-sum group-bound Sauvola kernel (bb_kernel, dtb_block.cu) against the CPU oracle,
bit-exact.

The kernel keeps 4-column block sums, decides 8 adjacent pixels at once from bounds on their
window sums, and rebuilds exact per-pixel sums for uncertain groups from the image rows.  The
cases aim at that split: document pages (almost no uncertain groups), uniform noise (most
groups uncertain), exact ties (flat windows), every r mod 16 (block alignment of the group
windows), image borders, short images (every row clipped), row bands, segmented inputs and
batches.  DTB_BB=1 forces the kernel wherever it is eligible; dtb_last_kernel() pins that it
ran."""

import numpy as np
import pytest

import oracle
from paper_1210_3165_b200 import _lib, engine, workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def force_bb(monkeypatch):
    monkeypatch.setenv("DTB_BB", "1")


def _ran_bb():
    return _lib.lib().dtb_last_kernel() == b"bb_kernel"


def _check(img, win, k, r=128.0, expect_bb=True):
    got, _ = engine.binarize(img, win, "sauvola", k, r, want_tmap=False)
    if expect_bb:
        assert _ran_bb(), _lib.lib().dtb_last_kernel()
    want, _ = oracle.binarize(img, win, "sauvola", k, r, tmap=False, threads=8)
    got = got.cpu().numpy()
    if not np.array_equal(got, want):
        bad = np.argwhere(got != want)
        raise AssertionError(f"{len(bad)} mismatches, first at {bad[:5].tolist()} "
                             f"(win={win} k={k} r={r} shape={img.shape})")


def test_c4_crop_w127():
    _check(workloads.c4_image(2048), 127, 0.34)


@pytest.mark.parametrize("rad", range(31, 47))  # every r mod 16
def test_every_residue(rad):
    img = workloads.doc_gray(300, 2608, 40 + rad, 900)
    _check(img, 2 * rad + 1, 0.34)


@pytest.mark.parametrize("rad", [8, 9, 10, 11, 15, 17, 23, 24, 100, 119, 124])
def test_window_range(rad):
    img = workloads.doc_gray(257, 2112, rad, 700)
    _check(img, 2 * rad + 1, 0.5)


@pytest.mark.parametrize("seed", range(4))
def test_uniform_noise_many_uncertain(seed):
    rng = np.random.default_rng(100 + seed)
    img = rng.integers(0, 256, (200, 1808)).astype(np.uint8)
    win = int(rng.choice([49, 63, 65, 99, 127, 201]))
    k = float(rng.choice([0.05, 0.34, 0.5, 1.0]))
    r = float(rng.choice([128.0, 64.0, 255.0, 1.5]))
    _check(img, win, k, r)


def test_flat_windows_exact_ties():
    # constant areas: s = 0 -> t = m (1-k) exactly (k = 0.5: t = 100 at m = 200)
    img = np.full((300, 2208), 200, np.uint8)
    img[:, 1000:1600] = 100
    img[120:180, 300:900] = 0
    img[::7, ::5] = 100
    for win, k in ((63, 0.5), (127, 0.5), (101, 0.25)):
        _check(img, win, k)


def test_short_and_wide_images():
    for h in (1, 2, 5, 40):
        img = workloads.doc_gray(h, 3008, h, 50)
        _check(img, 127, 0.34)


def test_narrow_images():
    # one strip, both image edges inside it; widths just above the radius
    for w, win in ((80, 63), (128, 127), (160, 99), (256, 201), (896, 127)):
        img = workloads.doc_gray(180, w, w, 60)
        _check(img, win, 0.34)


def test_lanes_with_two_edge_groups():
    # left- and right-edge groups 32 slots apart land in the same lane: the first one's count
    # bounds come packed from the prologue, the second one's are derived in the row loop
    for w, win in ((330, 127), (333, 127), (700, 249), (523, 191)):
        img = workloads.doc_gray(140, w, w % 13 + 1, 70)
        _check(img, win, 0.34)
        # low contrast, t ~ 0.87 m: bounds leave many groups open -> refinement and exact path
        _check((img // 4 + 90).astype(np.uint8), win, 0.15)


def test_right_edge_partial_strip():
    for w in (912, 1808, 2128, 4112, 16384):
        img = workloads.doc_gray(150, w, w, 300)
        _check(img, 95, 0.34)


def test_bands_and_batch():
    torch = engine.torch_mod()
    img = workloads.c4_image(2048)[:700, :2048]
    want, _ = oracle.binarize(img, 127, "sauvola", 0.34, tmap=False, threads=8)
    dev = torch.from_numpy(img).cuda()
    for y0, y1 in ((0, 1), (13, 400), (699, 700), (300, 700)):
        a, z = max(y0 - 63, 0), min(y1 + 63, 700)
        got = engine.binarize_band(dev[a:z], a, 700, y0, y1, 127, "sauvola", 0.34, 128.0)
        assert _ran_bb()
        assert np.array_equal(got.cpu().numpy(), want[y0:y1]), (y0, y1)
    imgs = np.stack([workloads.doc_gray(256, 2048, s, 300) for s in range(3)])
    got = engine.binarize_batch(torch.from_numpy(imgs).cuda(), 127, "sauvola", 0.34, 128.0)
    assert _ran_bb()
    for i in range(3):
        assert np.array_equal(got[i].cpu().numpy(),
                              oracle.binarize(imgs[i], 127, "sauvola", 0.34, tmap=False)[0])


def test_ineligible_falls_back(monkeypatch):
    img = workloads.doc_gray(200, 2112, 9, 300)
    _check(img, 127, 1.5, expect_bb=False)  # k > 1
    assert not _ran_bb()
    engine.binarize(img, 127, "niblack", -0.2, 128.0, want_tmap=False)
    assert not _ran_bb()
    _check(img, 15, 0.34, expect_bb=False)  # r < 8
    assert not _ran_bb()
    monkeypatch.setenv("DTB_BB", "0")
    _check(img, 127, 0.34, expect_bb=False)
    assert not _ran_bb()


def test_segmented_input_matches_page():
    torch = engine.torch_mod()
    img = workloads.c4_image(2048)[:900, :2048]
    want, _ = oracle.binarize(img, 127, "sauvola", 0.34, tmap=False, threads=8)
    dev = torch.from_numpy(img).cuda()
    top, mid, bot = dev[:200].clone(), dev[200:700].clone(), dev[700:].clone()
    segs = [(t.data_ptr(), t.stride(0), t.shape[0], t.shape[1]) for t in (top, mid, bot)]
    for y0, y1 in ((263, 637), (0, 900), (640, 900)):
        out = engine.binarize_segments(segs, 0, 900, y0, y1, 127, "sauvola", 0.34, 128.0)
        assert _ran_bb()
        assert np.array_equal(out.cpu().numpy(), want[y0:y1]), (y0, y1)


def test_large_windows_limit():
    # the uint32 bound E needs (2r+1)(2r+14) 255^2 < 2^32: r <= 124 runs the kernel
    img = np.full((400, 2112), 255, np.uint8)
    img[::3, ::7] = 254
    _check(img, 249, 0.34)
    _check(img, 251, 0.34, expect_bb=False)
    assert not _ran_bb()


@pytest.mark.parametrize("seed", range(8))
def test_random_pages_and_params(seed):
    rng = np.random.default_rng(3000 + seed)
    for _ in range(4):
        h = int(rng.integers(1, 400))
        w = 16 * int(rng.integers(20, 270))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            img = workloads.doc_gray(h, w, int(rng.integers(0, 1 << 30)), max(1, h * w // 3000))
        elif kind == 1:
            img = rng.integers(0, 256, (h, w)).astype(np.uint8)
        else:  # flat levels + small noise: many near-ties
            base = rng.integers(0, 256, (1, w // 64 + 1)).repeat(64, 1)[:, :w]
            img = np.clip(base + rng.integers(-3, 4, (h, w)), 0, 255).astype(np.uint8)
        rad = int(rng.integers(8, 125))
        rad = min(rad, w - 1)
        k = float(rng.choice([0.01, 0.2, 0.34, 0.5, 0.77, 1.0]))
        r = float(rng.choice([1.0, 16.0, 128.0, 255.0, 300.0]))
        _check(img, 2 * rad + 1, k, r, expect_bb=rad >= 8)


@pytest.mark.parametrize("w", [130, 1003, 2550, 4097])
def test_odd_widths_pitched(w):
    # widths that are not a multiple of 16 arrive in a 16-byte pitched buffer: the tensor map
    # covers whole 8-byte chunks, the kernel patches the last cols % 8 bytes of each staged row
    img = workloads.doc_gray(170, w, w, 90)
    _check(img, 2 * min(63, (w - 1) // 2) + 1, 0.34)


def test_odd_width_band_and_segments():
    torch = engine.torch_mod()
    img = workloads.doc_gray(600, 2003, 5, 400)
    want, _ = oracle.binarize(img, 101, "sauvola", 0.34, tmap=False, threads=8)
    pitched = torch.empty((600, 2016), dtype=torch.uint8, device="cuda")[:, :2003]
    pitched.copy_(torch.from_numpy(img))
    got = engine.binarize_band(pitched[100:500], 100, 600, 150, 450, 101, "sauvola", 0.34, 128.0)
    assert _ran_bb()
    assert np.array_equal(got.cpu().numpy(), want[150:450])
    segs = [(t.data_ptr(), t.stride(0), t.shape[0], 2003) for t in (pitched[:200], pitched[200:420], pitched[420:])]
    out = engine.binarize_segments(segs, 0, 600, 0, 600, 101, "sauvola", 0.34, 128.0)
    assert _ran_bb()
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("h", [17, 63, 64, 65, 129, 131, 200, 257, 1030])
def test_band_pair_counts(h):
    # pipelines run in pairs sharing one warm-up (one band downward, one upward from their
    # common row); heights give odd / even band counts and a pair whose downward band is empty
    img = workloads.doc_gray(h, 1500, 3 + h % 11, 1300)
    _check(img, 63, 0.34)


def test_tall_and_short_bands():
    # bands taller and shorter than the window (both share the pair's warm-up); both parities
    # against the oracle
    for h, w in ((1400, 41), (300, 201)):
        img = workloads.doc_gray(h, 3000, 5, 1400 + h)
        _check(img, w, 0.34)
