"""PNM page pipeline: pinned readinto -> H2D -> to_gray/binarize ->
D2H -> P5, overlapped across pages; outputs byte-identical to the reference CLI's recipe
(cli.py:85-93: read_pnm, to_gray for RGB, binarize, write_pnm) computed by the oracle."""

import numpy as np
import pytest

import paper_1210_3165_b200 as dt
from oracle import numpy_ref
from paper_1210_3165_b200 import pipeline

pytestmark = pytest.mark.gpu


def _expected(img, params):
    gray = numpy_ref.to_gray(img) if img.ndim == 3 else img
    if params.method == "otsu":
        t = numpy_ref.otsu_threshold(gray)
        b = np.where(gray < t, 0, 255).astype(np.uint8)
    elif params.full_window:
        b, _ = numpy_ref.binarize(gray, params.window, params.method, params.k, params.r)
    else:
        m, s, _ = numpy_ref.mean_std_sampled(gray, params.mask, params.window)
        tm = numpy_ref.threshold_map(m, s, params.method, params.k, params.r)
        b = np.where(gray.astype(np.float64) < tm, 0, 255).astype(np.uint8)
    h, w = b.shape
    return f"P5\n{w} {h}\n255\n".encode() + b.tobytes()


def _ascii(img):
    magic = "P3" if img.ndim == 3 else "P2"
    h, w = img.shape[:2]
    body = " ".join(str(int(v)) for v in img.reshape(-1))
    return f"{magic}\n# a comment\n{w} {h}\n255\n{body}\n".encode()


def _pages(rng):
    pages = []
    for i, (h, w) in enumerate([(300, 417), (64, 64), (517, 1031), (33, 20), (800, 600)]):
        g = rng.integers(150, 230, (h, w)).astype(np.uint8)
        g[rng.random((h, w)) < 0.07] = 30
        if i % 2:
            rgb = np.stack([g, np.clip(g.astype(int) + 9, 0, 255), g // 2], -1).astype(np.uint8)
            pages.append((rgb, b"P6\n#c\n%d %d\n255\n" % (w, h) + rgb.tobytes()))
        else:
            pages.append((g, b"P5 %d %d 255\n" % (w, h) + g.tobytes()))
    small = rng.integers(0, 256, (9, 13)).astype(np.uint8)
    pages.append((small, _ascii(small)))
    rgb = rng.integers(0, 256, (7, 5, 3)).astype(np.uint8)
    pages.append((rgb, _ascii(rgb)))
    return pages


@pytest.mark.parametrize("params", [
    dt.BinarizationParams(),  # reference defaults: sauvola / sampled / gs3 / W=21
    dt.BinarizationParams(engine="integral", window=31, k_sauvola=0.5),
    dt.BinarizationParams(method="niblack", engine="naive", window=15),
    dt.BinarizationParams(method="otsu"),
    dt.BinarizationParams(engine="sampled", mask="gs6", window=9),
], ids=["default", "integral", "niblack", "otsu", "gs6"])
@pytest.mark.parametrize("slots", [1, 2, 3])
def test_pipeline_outputs_match_oracle(tmp_path, rng, params, slots):
    pages = _pages(rng)
    pairs = []
    for i, (_, data) in enumerate(pages):
        src, dst = tmp_path / f"in{i}.pnm", tmp_path / f"out{i}.pgm"
        src.write_bytes(data)
        pairs.append((str(src), str(dst)))
    st = pipeline.binarize_files(pairs, params, slots=slots)
    assert st.pages == len(pages)
    for (img, _), (_, dst) in zip(pages, pairs):
        assert open(dst, "rb").read() == _expected(img, params)
        assert dt.read_pnm(open(dst, "rb").read()).shape == img.shape[:2]


def test_pipeline_errors_match_read_pnm(tmp_path):
    bad = b"P5\n4 4\n255\n" + bytes(10)  # truncated payload
    src = tmp_path / "bad.pgm"
    src.write_bytes(bad)
    with pytest.raises(dt.PnmError) as e1:
        pipeline.binarize_files([(str(src), str(tmp_path / "o.pgm"))])
    with pytest.raises(dt.PnmError) as e2:
        dt.read_pnm(bad)
    assert str(e1.value) == str(e2.value)
    src.write_bytes(b"P5\n4 4\n65535\n" + bytes(32))
    with pytest.raises(dt.PnmError, match="unsupported maxval 65535"):
        pipeline.binarize_files([(str(src), str(tmp_path / "o.pgm"))])
