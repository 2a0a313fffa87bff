"""Host-tensor binarize with H2D / compute / D2H overlapped by row chunks (engine.host_streamed):
identical to the device path for any chunking, pinned or pageable input, with or without out=."""

import numpy as np
import pytest
import torch

import paper_1210_3165_b200 as dt
from paper_1210_3165_b200 import engine, workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("h,w,win,method,k", [(512, 512, 15, "sauvola", 0.5),
                                               (1000, 777, 127, "sauvola", 0.34),
                                               (333, 2048, 31, "niblack", -0.2),
                                               (7, 40, 3, "sauvola", 0.5)])
@pytest.mark.parametrize("pinned", [True, False])
def test_host_tensor_binarize_matches_device(h, w, win, method, k, pinned):
    img = workloads.doc_gray(h, w, 5, max(4, h * w // 3000))
    want, _ = engine.binarize(torch.from_numpy(img).cuda(), win, method, k, 128.0, want_tmap=False)
    host = torch.from_numpy(img)
    if pinned:
        host = host.pin_memory()
    kw = {"k_sauvola": k} if method == "sauvola" else {"k_niblack": k}
    p = dt.BinarizationParams(method=method, engine="integral", window=win, **kw)
    b, t = dt.binarize(host, p, return_tmap=False)
    assert t is None and not b.is_cuda
    assert torch.equal(b, want.cpu())
    out = torch.empty((h, w), dtype=torch.uint8).pin_memory()
    b2, _ = dt.binarize(host, p, return_tmap=False, out=out)
    assert b2.data_ptr() == out.data_ptr() and torch.equal(out, want.cpu())


@pytest.mark.parametrize("chunk", [1, 17, 64, 200, 5000])
def test_host_streamed_chunking(chunk):
    """Chunks thinner than the window radius: a chunk's compute waits for later chunks."""
    img = workloads.doc_gray(900, 640, 9, 200)
    want, _ = engine.binarize(torch.from_numpy(img).cuda(), 127, "sauvola", 0.34, 128.0,
                              want_tmap=False)
    host = torch.from_numpy(img).pin_memory()

    def band(dev_in, y0, y1, dev_out):
        engine.binarize_band(dev_in, 0, dev_in.shape[0], y0, y1, 127, "sauvola", 0.34, 128.0,
                             out=dev_out)
    got = engine.host_streamed(host, band, 63, chunk_rows=chunk)
    assert torch.equal(got, want.cpu())
