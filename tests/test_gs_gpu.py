"""O(1)-per-pixel GS-mask kernel (dtb_gs_stats) against the numpy
oracle (stats.py:133-163 restated) and against the O(|mask|) offset-gather kernel."""

import numpy as np
import pytest

import paper_1210_3165_b200 as dt
from paper_1210_3165_b200 import engine
from oracle import numpy_ref

pytestmark = pytest.mark.gpu

STRUCTS = ("gs1", "gs2", "gs3", "gs4", "gs5", "gs6")


def _doc(rng, h, w):
    img = rng.integers(170, 236, (h, w))
    ink = rng.random((h, w)) < 0.08
    img[ink] = rng.integers(0, 70, int(ink.sum()))
    return img.astype(np.uint8)


@pytest.mark.parametrize("structure", STRUCTS)
@pytest.mark.parametrize("shape,win", [((1, 1), 3), ((3, 200), 5), ((130, 2), 7), ((33, 129), 21),
                                       ((64, 128), 11), ((97, 301), 31), ((40, 40), 81),
                                       ((70, 260), 127)])
def test_gs_stats_match_oracle(rng, structure, shape, win):
    img = _doc(rng, *shape)
    m, s, n = dt.mean_std_sampled(img, dt.make_mask(structure, win))
    om, os_, on = numpy_ref.mean_std_sampled(img, structure, win)
    assert np.array_equal(n, on)
    assert np.array_equal(m.view(np.uint64), om.view(np.uint64))
    assert np.array_equal(s.view(np.uint64), os_.view(np.uint64))


@pytest.mark.parametrize("structure", STRUCTS)
@pytest.mark.parametrize("method,k", [("sauvola", 0.34), ("niblack", -0.2), ("sauvola", 0.5)])
def test_gs_binarize_matches_gather_kernel(rng, structure, method, k):
    import torch
    img = torch.from_numpy(_doc(rng, 517, 1031)).cuda()
    for win in (3, 15, 41, 101):
        offs = dt.make_mask(structure, win).offsets
        b1, t1 = engine.gs(img, structure, win, method, k, 128.0)
        b2, t2 = engine.sampled(img, offs, method, k, 128.0)
        assert torch.equal(b1, b2), (structure, win)
        assert torch.equal(t1.view(torch.int64), t2.view(torch.int64)), (structure, win)
        b3, t3 = engine.gs(img, structure, win, method, k, 128.0, want_tmap=False)
        assert t3 is None and torch.equal(b3, b1)


def test_gs_strided_device_input_and_default_params(rng):
    import torch
    big = torch.from_numpy(_doc(rng, 300, 700)).cuda()
    view = big[7:290, 13:650]  # row pitch 700, unaligned origin
    b, t = dt.binarize(view)  # reference defaults: sauvola / sampled / gs3 / W=21
    host = view.cpu().numpy()
    om, os_, _ = numpy_ref.mean_std_sampled(host, "gs3", 21)
    tm = numpy_ref.threshold_map(om, os_, "sauvola", 0.34)
    assert np.array_equal(t.cpu().numpy().view(np.uint64), tm.view(np.uint64))
    assert np.array_equal(b.cpu().numpy(), np.where(host < tm, 0, 255).astype(np.uint8))


def test_gs_huge_window_falls_back_to_gather(rng):
    img = _doc(rng, 20, 30)
    m, s, n = dt.mean_std_sampled(img, dt.make_mask("gs3", 601))  # tile > shared memory
    om, os_, on = numpy_ref.mean_std_sampled(img, "gs3", 601)
    assert np.array_equal(n, on) and np.array_equal(m, om) and np.array_equal(s, os_)


@pytest.mark.parametrize("structure", STRUCTS)
def test_gs_fast_path_near_ties(rng, structure):
    """Binary-only (certified fp32) path on images built to put f at or near t."""
    import torch
    cases = [(rng.choice([100, 101], (150, 290)).astype(np.uint8), "niblack", 0.0),
             (rng.choice([0, 255], (150, 290)).astype(np.uint8), "niblack", 0.0),
             (rng.choice([60, 61, 62], (150, 290)).astype(np.uint8), "sauvola", 0.5),
             (np.full((150, 290), 77, np.uint8), "sauvola", 0.34),
             (rng.integers(0, 256, (150, 290)).astype(np.uint8), "niblack", -0.2)]
    for img, method, k in cases:
        for win in (3, 9, 21):
            b, _ = engine.gs(torch.from_numpy(img).cuda(), structure, win, method, k, 128.0,
                             want_tmap=False)
            om, os_, _ = numpy_ref.mean_std_sampled(img, structure, win)
            tm = numpy_ref.threshold_map(om, os_, method, k)
            want = np.where(img.astype(np.float64) < tm, 0, 255).astype(np.uint8)
            assert np.array_equal(b.cpu().numpy(), want), (method, k, win)


@pytest.mark.parametrize("structure", STRUCTS)
@pytest.mark.parametrize("win", [3, 21, 63, 127])
def test_gs_bands_stitch_to_whole_page(rng, structure, win):
    """dtb_gs_band over row bands whose buffers hold only the band + r-row halos."""
    import torch
    h, w = 517, 700
    img = torch.from_numpy(_doc(rng, h, w)).cuda()
    want, _ = engine.gs(img, structure, win, "sauvola", 0.34, 128.0, want_tmap=False)
    r = win // 2
    cuts = [0, 1, 40, 41, 200, 333, 516, 517]
    for y0, y1 in zip(cuts[:-1], cuts[1:]):
        a, z = max(y0 - r, 0), min(y1 + r, h)
        buf = img[a:z].clone()
        got = engine.gs_band(buf, a, h, y0, y1, structure, win, "sauvola", 0.34, 128.0)
        assert torch.equal(got, want[y0:y1]), (y0, y1)


def test_default_params_host_tensor_streamed(rng):
    """binarize(pinned host tensor) with the reference defaults (gs3 W=21) streams row
    chunks through dtb_gs_band and equals the device result."""
    import torch
    img = _doc(rng, 1500, 1234)
    want, _ = dt.binarize(torch.from_numpy(img).cuda(), return_tmap=False)
    host = torch.from_numpy(img).pin_memory()
    got, t = dt.binarize(host, return_tmap=False)
    assert t is None and torch.equal(got, want.cpu())
