"""Warm-up cost probe: time the C4 kernel on 16384 vs 32768 vs 65536 rows (same width, one
wave of CTAs each, so band height scales with the page) -> per-pixel time vs band height."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_3165_b200 import engine, workloads
img = workloads.c4_image()
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
for reps in (1, 2, 4):
    page = torch.from_numpy(np.concatenate([img] * reps)).cuda()
    out = torch.empty_like(page)
    def run():
        engine.binarize_band(page, 0, page.shape[0], 0, page.shape[0], 127, "sauvola", 0.34, 128.0, out=out)
    run(); torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    print(f"rows {page.shape[0]}: {ms:.4f} ms, {ms / reps:.4f} ms per 16384 rows", flush=True)
    del page, out
