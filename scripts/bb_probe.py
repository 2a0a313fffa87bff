"""Probe (scripts/, not product): kernel time of one BASELINE page / window (mean of 20
back-to-back launches between CUDA events, after warm-up), exact-path group count, and the
output's hash against the reference golden.

    python scripts/bb_probe.py [c4|c5] [window]
"""
import ctypes
import hashlib
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1210_3165_b200 import _lib, engine, workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
win = int(sys.argv[2]) if len(sys.argv) > 2 else 127
img = workloads.c4_image() if cfg == "c4" else workloads.c5_image()
k = 0.34 if cfg == "c4" else 0.5
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json"))).get(f"{cfg}/w{win}", {}).get("binary")
dev = torch.from_numpy(img).cuda()
out = torch.empty_like(dev)
L = _lib.lib()
cnt = ctypes.c_uint64(0)
run = lambda: engine.binarize(dev, win, "sauvola", k, 128.0, want_tmap=False, out=out)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
L.dtb_debug_bb_exact(ctypes.byref(cnt), 1)
run()
torch.cuda.synchronize()
L.dtb_debug_bb_exact(ctypes.byref(cnt), 1)
ok = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest() == gold if gold else None
n = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(2_000_000)  # keep the GPU busy while the launches queue up
e0.record()
for _ in range(n):
    run()
e1.record()
torch.cuda.synchronize()
print(cfg, win, L.dtb_last_kernel().decode(), "ms=%.4f" % (e0.elapsed_time(e1) / n),
      "exact_groups", cnt.value, "golden", ok, flush=True)
