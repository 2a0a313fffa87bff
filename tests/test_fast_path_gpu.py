"""Stress the fast certified-decision kernel (dtb_slide.cu) against the CPU oracle:
many sizes, windows 3..255, both methods, extreme k / R, near-tie-heavy inputs, unaligned
pitches, band offsets and batches.  Bit-exact binary output is required everywhere."""

import numpy as np
import pytest

import oracle
from paper_1210_3165_b200 import engine, workloads

pytestmark = pytest.mark.gpu


def _check(img, win, method, k, r=128.0):
    got, _ = engine.binarize(img, win, method, k, r, want_tmap=False)
    want, _ = oracle.binarize(img, win, method, k, r, tmap=False, threads=8)
    got = got.cpu().numpy()
    if not np.array_equal(got, want):
        bad = np.argwhere(got != want)
        raise AssertionError(f"{len(bad)} mismatches, first at {bad[:5].tolist()} "
                             f"(win={win} {method} k={k} r={r} shape={img.shape})")


@pytest.mark.parametrize("win", [3, 5, 9, 15, 31, 63, 127, 255])
def test_documents_all_windows(win):
    img = workloads.c1_image()
    for method, k in (("sauvola", 0.5), ("sauvola", 0.05), ("sauvola", 0.9), ("niblack", -0.2),
                      ("niblack", 0.0), ("niblack", 0.5)):
        _check(img, win, method, k)


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes(seed):
    rng = np.random.default_rng(seed)
    for _ in range(6):
        h, w = int(rng.integers(1, 700)), int(rng.integers(1, 1500))
        img = rng.integers(0, 256, (h, w)).astype(np.uint8)
        win = int(rng.choice([3, 7, 21, 33, 65, 129, 255]))
        _check(img, win, "sauvola", float(rng.choice([0.34, 0.5, 0.2])),
               float(rng.choice([128.0, 64.0, 200.0])))
        _check(img, win, "niblack", float(rng.choice([-0.2, 0.0, 0.3])))


def test_near_ties_niblack_k0():
    # t == mean exactly: integer-mean windows make f == t ties common
    rng = np.random.default_rng(7)
    img = rng.integers(100, 104, (600, 900)).astype(np.uint8)
    for win in (3, 5, 15, 31):
        _check(img, win, "niblack", 0.0)
        _check(img, win, "sauvola", 1e-9, 1e9)


def test_flat_and_extreme_regions():
    img = np.full((300, 700), 200, np.uint8)
    img[100:140, 200:260] = 0
    img[:, 500:] = 255
    img[250:, :] = 1
    for win in (3, 15, 63, 127):
        _check(img, win, "sauvola", 0.34)
        _check(img, win, "niblack", -0.2)


def test_unaligned_pitch_and_bands():
    torch = engine.torch_mod()
    img = workloads.c5_image()[:1000, :1500]
    wide = torch.zeros((1000, 1523), dtype=torch.uint8, device="cuda")
    wide[:, 7:1507] = torch.from_numpy(img).cuda()
    view = wide[:, 7:1507]  # pitch 1523, base offset 7: scalar-load path
    want, _ = oracle.binarize(img, 63, "sauvola", 0.5, tmap=False)
    got = engine.binarize_band(view, 0, 1000, 0, 1000, 63, "sauvola", 0.5, 128.0)
    assert np.array_equal(got.cpu().numpy(), want)
    for y0, y1 in ((0, 1), (13, 500), (999, 1000), (400, 1000)):
        a, z = max(y0 - 31, 0), min(y1 + 31, 1000)
        got = engine.binarize_band(view[a:z], a, 1000, y0, y1, 63, "sauvola", 0.5, 128.0)
        assert np.array_equal(got.cpu().numpy(), want[y0:y1]), (y0, y1)


def test_batch_matches_single():
    torch = engine.torch_mod()
    imgs = np.stack([workloads.c3_image(i, size=512) for i in range(5)])
    out = engine.binarize_batch(torch.from_numpy(imgs).cuda(), 31, "niblack", -0.2, 128.0)
    for i in range(5):
        assert np.array_equal(out[i].cpu().numpy(),
                              oracle.binarize(imgs[i], 31, "niblack", -0.2, tmap=False)[0])


@pytest.mark.parametrize("method,k,r", [("sauvola", 1e-6, 128.0), ("sauvola", 0.99, 128.0),
                                        ("sauvola", 5.0, 128.0), ("sauvola", 0.34, 1.0),
                                        ("sauvola", 50.0, 2.0), ("sauvola", 0.5, 1e6),
                                        ("niblack", -5.0, 128.0), ("niblack", 5.0, 128.0),
                                        ("niblack", 1e-9, 128.0), ("niblack", -0.2, 128.0)])
@pytest.mark.parametrize("win", [3, 31, 255])
def test_extreme_parameters_match_oracle(method, k, r, win):
    """The certified fp32 decision's tolerance scales with k and R: extreme values only make
    more pixels take the fp64 replay, never a wrong byte."""
    import torch
    img = workloads.doc_gray(300, 1100, 13, 150)
    b, _ = engine.binarize(torch.from_numpy(img).cuda(), win, method, k, r, want_tmap=False)
    ob = oracle.binarize(img, win, method, k, r, tmap=False, threads=8)[0]
    assert np.array_equal(b.cpu().numpy(), ob)
    # and the wide-strip (warp-specialised) kernel on a page wide enough for it
    wide = workloads.doc_gray(160, 3840, 17, 150)
    b, _ = engine.binarize(torch.from_numpy(wide).cuda(), win, method, k, r, want_tmap=False)
    assert np.array_equal(b.cpu().numpy(), oracle.binarize(wide, win, method, k, r, tmap=False,
                                                           threads=8)[0])


@pytest.mark.parametrize("width", [1, 17, 500, 512, 1000, 2048, 2049, 2550, 4096])
def test_edge_padded_single_strip(monkeypatch, width):
    """slide_kernel's edge-padded layout (one strip = the image's own columns, no halo columns;
    DTB_PAD=1 forces it wherever the image fits one strip): every window alignment class
    (rx mod 4, rx mod 32 == 0), windows wider than the image, both methods, short bands."""
    from paper_1210_3165_b200 import _lib
    monkeypatch.setenv("DTB_PAD", "1")
    monkeypatch.setenv("DTB_BB", "0")
    rng = np.random.default_rng(width)
    h = 150 if width > 1000 else 333
    img = rng.integers(0, 256, (h, width)).astype(np.uint8)
    img[: h // 3] = (img[: h // 3] // 64) + 120  # a near-flat region: ties and tiny variances
    for win in (3, 5, 7, 9, 31, 63, 65, 127, 129, 255):
        _check(img, win, "sauvola", 0.34)
        assert _lib.lib().dtb_last_kernel().decode() == "slide_kernel"
        _check(img, win, "niblack", -0.2)


def test_edge_padded_batch_and_bands(monkeypatch):
    torch = engine.torch_mod()
    monkeypatch.setenv("DTB_PAD", "1")
    imgs = np.stack([workloads.c3_image(i, size=512) for i in range(3)])
    got = engine.binarize_batch(torch.from_numpy(imgs).cuda(), 31, "niblack", -0.2, 128.0)
    for i in range(3):
        want, _ = oracle.binarize(imgs[i], 31, "niblack", -0.2, tmap=False)
        assert np.array_equal(got[i].cpu().numpy(), want)
    img = workloads.c5_image()[:700, :1800]
    dev = torch.from_numpy(img).cuda()
    want, _ = oracle.binarize(img, 45, "sauvola", 0.5, tmap=False)
    for y0, y1 in ((0, 1), (13, 400), (699, 700), (300, 700)):
        a, z = max(y0 - 22, 0), min(y1 + 22, 700)
        got = engine.binarize_band(dev[a:z], a, 700, y0, y1, 45, "sauvola", 0.5, 128.0)
        assert np.array_equal(got.cpu().numpy(), want[y0:y1]), (y0, y1)


def test_planner_takes_the_edge_padded_strip_when_it_saves_columns():
    """Default planner rule (DTB_PAD unset): a 2048-wide page at W31 runs one edge-padded strip
    (5 x 512 halo columns -> 2048), C2's 2480-wide page keeps the halo layout (one 2560-column
    strip either way).
    The plan is read from DTB_PRINT_PLAN's stderr line in a fresh process."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import numpy as np, torch\n"
            "from paper_1210_3165_b200 import engine\n"
            "for w in (2048, 2480):\n"
            "    img = np.random.default_rng(w).integers(0, 256, (64, w)).astype(np.uint8)\n"
            "    engine.binarize(img, 31, 'niblack', -0.2, 128.0, want_tmap=False)\n"
            "torch.cuda.synchronize()\n")
    env = dict(os.environ, DTB_PRINT_PLAN="1")
    env.pop("DTB_PAD", None)
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    plans = [ln for ln in res.stderr.splitlines() if ln.startswith("[dtb plan] slide_kernel")]
    assert any("cols=2048" in ln and "strips=1" in ln and "pad=32" in ln for ln in plans), plans
    assert any("cols=2480" in ln and "pad=0" in ln for ln in plans), plans
