"""Per-config results table for all five BASELINE configs (GPU box).

For every config: the fused kernel's device time (CUDA events, median of reps, L2 flushed
between reps with a 512 MiB memset), Mpixel/s, achieved algorithmic GB/s vs the measured
HBM peak, and bit-exactness of the output against the golden hash produced by the
reference (tests/golden/configs.json).  C5 is swept over all 16 window sizes.

    python scripts/config_table.py [--reps 10] > gpurun_out/config_table.json
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1210_3165_b200 import engine, workloads  # noqa: E402

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
    _flush.zero_()


def timed(fn, reps):
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


_audit_fn = None


def audit(fn):
    """Run fn once with the fp32-epilogue audit on: (replayed in fp64, would-flip, max gap)."""
    import struct
    from paper_1210_3165_b200 import _lib
    c = torch.zeros(3, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().dtb_set_fp32_audit(c.data_ptr()), "audit")
    fn()
    torch.cuda.synchronize()
    _lib.check(_lib.lib().dtb_set_fp32_audit(None), "audit")
    rep, flip, gap = (int(v) for v in c.cpu().tolist())
    return {"replayed_fp64": rep, "fp32_would_flip": flip,
            "max_gap_of_would_flip": struct.unpack("<f", struct.pack("<I", gap & 0xFFFFFFFF))[0]}


def _lk():
    from paper_1210_3165_b200 import _lib
    return _lib.lib().dtb_last_kernel().decode()


def row(name, px, ms, alg_bytes, exact, fn=None, kernel=None):
    from paper_1210_3165_b200 import _lib
    gbs = alg_bytes / (ms / 1e3) / 1e9
    # dtb_last_kernel names the last BINARIZATION kernel: rows of other kernels pass theirs
    out = {"config": name, "kernel": kernel or _lib.lib().dtb_last_kernel().decode(), "pixels": int(px), "kernel_ms": round(ms, 4),
           "mpix_per_s": round(px / (ms / 1e3) / 1e6, 1), "alg_bytes": int(alg_bytes),
           "achieved_gbs": round(gbs, 1), "roofline_frac": round(gbs / PEAK, 4),
           "bit_exact_vs_reference": exact}
    if fn is not None:
        # north_star: the fp32 epilogue reported separately -- output flips are 0 by
        # construction (uncertain pixels are replayed in fp64; the hash check above proves it)
        out["fp32_epilogue"] = dict(audit(fn), flipped_in_output=0 if exact else None)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-audit", action="store_true")
    a = ap.parse_args()
    if a.no_audit:
        global audit
        audit = lambda fn: {}  # noqa: E731
    cfg = workloads.CONFIGS
    out = []
    # C1
    img = torch.from_numpy(workloads.c1_image()).cuda()
    ms = timed(lambda: engine.binarize(img, 15, "sauvola", 0.5, 128.0, want_tmap=False), a.reps)
    b, _ = engine.binarize(img, 15, "sauvola", 0.5, 128.0, want_tmap=False)
    out.append(row("c1 512^2 W15", img.numel(), ms, 2 * img.numel(),
                   sha(b.cpu().numpy()) == GOLD["c1/w15"]["binary"],
                   lambda: engine.binarize(img, 15, "sauvola", 0.5, 128.0, want_tmap=False)))
    # C2: to_gray + binarize at 3 windows
    rgb = torch.from_numpy(workloads.c2_rgb()).cuda()
    gray = engine.to_gray(rgb)
    ms = timed(lambda: engine.to_gray(rgb), a.reps)
    out.append(row("c2 to_gray 3508x2480", gray.numel(), ms, 4 * gray.numel(),
                   sha(gray.cpu().numpy()) == GOLD["c2/rgb"]["gray"], kernel="to_gray_kernel"))
    for w in cfg["c2"].windows:
        ms = timed(lambda: engine.binarize(gray, w, "sauvola", 0.5, 128.0, want_tmap=False), a.reps)
        b, _ = engine.binarize(gray, w, "sauvola", 0.5, 128.0, want_tmap=False)
        out.append(row(f"c2 W{w}", gray.numel(), ms, 2 * gray.numel(),
                       sha(b.cpu().numpy()) == GOLD[f"c2/w{w}"]["binary"],
                       lambda: engine.binarize(gray, w, "sauvola", 0.5, 128.0, want_tmap=False)))
        ms = timed(lambda: engine.rgb_binarize(rgb, w, "sauvola", 0.5, 128.0), a.reps)
        b = engine.rgb_binarize(rgb, w, "sauvola", 0.5, 128.0)
        out.append(row(f"c2 rgb->binary W{w}", gray.numel(), ms, 4 * gray.numel(),
                       sha(b.cpu().numpy()) == GOLD[f"c2/w{w}"]["binary"],
                       kernel="to_gray_kernel + " + _lk()))
    del rgb, gray
    # C3 batch
    stack = torch.from_numpy(np.stack([workloads.c3_image(i) for i in range(64)])).cuda()
    ms = timed(lambda: engine.binarize_batch(stack, 31, "niblack", -0.2, 128.0), a.reps)
    o = engine.binarize_batch(stack, 31, "niblack", -0.2, 128.0).cpu().numpy()
    ok = all(sha(o[i]) == GOLD[f"c3/img{i}"]["binary"] for i in range(64))
    out.append(row("c3 64x2048^2 niblack W31", stack.numel(), ms, 2 * stack.numel(), ok,
                   lambda: engine.binarize_batch(stack, 31, "niblack", -0.2, 128.0)))
    del stack
    # C4
    img = torch.from_numpy(workloads.c4_image()).cuda()
    ms = timed(lambda: engine.binarize(img, 127, "sauvola", 0.34, 128.0, want_tmap=False), a.reps)
    b, _ = engine.binarize(img, 127, "sauvola", 0.34, 128.0, want_tmap=False)
    out.append(row("c4 16384^2 W127", img.numel(), ms, 2 * img.numel(),
                   sha(b.cpu().numpy()) == GOLD["c4/w127"]["binary"],
                   lambda: engine.binarize(img, 127, "sauvola", 0.34, 128.0, want_tmap=False)))
    del img, b
    # C5 sweep
    img = torch.from_numpy(workloads.c5_image()).cuda()
    for w in cfg["c5"].windows:
        ms = timed(lambda: engine.binarize(img, w, "sauvola", 0.5, 128.0, want_tmap=False), a.reps)
        b, _ = engine.binarize(img, w, "sauvola", 0.5, 128.0, want_tmap=False)
        out.append(row(f"c5 4096^2 W{w}", img.numel(), ms, 2 * img.numel(),
                       sha(b.cpu().numpy()) == GOLD[f"c5/w{w}"]["binary"],
                       lambda: engine.binarize(img, w, "sauvola", 0.5, 128.0, want_tmap=False)))
    print(json.dumps({"gpu": torch.cuda.get_device_name(0), "peak_gbs": PEAK,
                      "l2": "flushed (512 MiB memset) before every rep", "rows": out}, indent=1))


if __name__ == "__main__":
    main()
