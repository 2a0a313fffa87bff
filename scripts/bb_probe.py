"""Probe: bb_kernel time and exact-path group count on a BASELINE page (scripts/, not product)."""
import ctypes, sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1210_3165_b200 import _lib, engine, workloads

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
win = int(sys.argv[2]) if len(sys.argv) > 2 else 127
img = workloads.c4_image() if cfg == "c4" else workloads.c5_image()
k = 0.34 if cfg == "c4" else 0.5
dev = torch.from_numpy(img).cuda()
out = torch.empty_like(dev)
L = _lib.lib()
cnt = ctypes.c_uint64(0)
for rep in range(3):
    L.dtb_debug_bb_exact(ctypes.byref(cnt), 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    got, _ = engine.binarize(dev, win, "sauvola", k, 128.0, want_tmap=False, out=out) if False else engine.binarize(dev, win, "sauvola", k, 128.0, want_tmap=False)
    e1.record(); torch.cuda.synchronize()
    L.dtb_debug_bb_exact(ctypes.byref(cnt), 1)
    print(cfg, win, L.dtb_last_kernel().decode(), "ms=%.4f" % e0.elapsed_time(e1), "exact_groups", cnt.value, flush=True)
