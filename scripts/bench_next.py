"""Device timings for the §8 'next' rows on a B200 (CUDA events, L2 flushed per rep).

f1: GS-mask engine -- O(1) tiled kernel (dtb_gs_stats) vs the O(|mask|) gather kernel
    (dtb_sampled_stats), binarize without tmap, on the 4096^2 C5 page.
f2: sweep() over the default 5 x 6 grid (sampled/gs3) and evaluate() on the same page.

    python scripts/bench_next.py [--reps 5] > gpurun_out/next.json
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1210_3165_b200 as dt  # noqa: E402
from paper_1210_3165_b200 import engine, workloads  # noqa: E402

_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
    _flush.zero_()


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--gather", action="store_true", help="also time the gather kernel")
    a = ap.parse_args()
    img = torch.from_numpy(workloads.c5_image()).cuda()
    px = img.numel()
    rows = []
    for st in ("gs1", "gs2", "gs3", "gs4", "gs5", "gs6"):
        for w in (3, 21, 41, 127):
            ms = timed(lambda: engine.gs(img, st, w, "sauvola", 0.34, 128.0, want_tmap=False),
                       a.reps)
            row = {"structure": st, "win": w, "gs_ms": round(ms, 4),
                   "gs_gpx_s": round(px / ms / 1e6, 2)}
            if a.gather and (w <= 41 or st in ("gs3",)):
                offs = dt.make_mask(st, w).offsets
                mg = timed(lambda: engine.sampled(img, offs, "sauvola", 0.34, 128.0,
                                                  want_tmap=False), max(1, a.reps // 2))
                row["gather_ms"] = round(mg, 4)
                b1, _ = engine.gs(img, st, w, "sauvola", 0.34, 128.0, want_tmap=False)
                b2, _ = engine.sampled(img, offs, "sauvola", 0.34, 128.0, want_tmap=False)
                row["identical"] = bool(torch.equal(b1, b2))
            rows.append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
    # f2: sweep + evaluate on a page with ground truth = the full-window W=127 binarization
    gt, _ = engine.binarize(img, 127, "sauvola", 0.34, 128.0, want_tmap=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = dt.sweep(img, gt)
    torch.cuda.synchronize()
    sweep_s = time.perf_counter() - t0
    pred, _ = engine.gs(img, "gs3", 21, "sauvola", 0.34, 128.0, want_tmap=False)
    ev_ms = timed(lambda: dt.evaluate(pred, gt), a.reps)
    # f4: PNM page pipeline, 12 A4/300dpi RGB pages (C2 shape, P6 files), reference-CLI
    # default params (sauvola / sampled gs3 / W=21); files in a temp dir, page cache warm.
    import tempfile
    from paper_1210_3165_b200 import pipeline
    rgb = workloads.c2_rgb()
    h, w = rgb.shape[:2]
    data = b"P6\n%d %d\n255\n" % (w, h) + rgb.tobytes()
    pipe = {}
    with tempfile.TemporaryDirectory() as td:
        pairs = []
        for i in range(12):
            src = os.path.join(td, f"p{i}.ppm")
            with open(src, "wb") as fh:
                fh.write(data)
            pairs.append((src, os.path.join(td, f"o{i}.pgm")))
        for slots in (1, 2, 3):
            pipeline.binarize_files(pairs[:2], slots=slots)  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st = pipeline.binarize_files(pairs, slots=slots)
            torch.cuda.synchronize()
            dt_s = time.perf_counter() - t0
            pipe[f"slots{slots}"] = {"pages_per_s": round(st.pages / dt_s, 2),
                                     "mpx_per_s": round(st.pixels / dt_s / 1e6, 1),
                                     "file_mb_per_s": round((st.bytes_in + st.bytes_out) / dt_s / 1e6, 1)}
    out = {"gpu": torch.cuda.get_device_name(0), "page": list(img.shape),
           "pipeline_c2_pages": pipe,
           "l2": "flushed (512 MiB memset) before every rep", "gs": rows,
           "sweep_default_grid_s": round(sweep_s, 4), "sweep_best": list(res.best),
           "evaluate_ms_incl_host_sync": round(ev_ms, 4)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
