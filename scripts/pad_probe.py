"""Probe (scripts/, not product): edge-padded single-strip layout of slide_kernel against the
halo layout, alternating DTB_PAD / DTB_PAD_V inside one process (C3, C2 page, C5 windows)."""
import os, statistics, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1210_3165_b200 import engine, workloads, _lib
flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
def timed(fn, reps=7):
    ts = []
    for i in range(reps):
        flush.zero_(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.median(ts[2:])
modes = [("0", "16"), ("1", "16")]
def ab(name, fn):
    res = {}
    for rnd in range(2):
        for pad, v in modes:
            os.environ["DTB_PAD"], os.environ["DTB_PAD_V"] = pad, v
            t = timed(fn)
            res.setdefault((pad, v), []).append(t)
    print(name, " ".join("pad=%s,V=%s: %.4f" % (k[0], k[1], min(v)) for k, v in res.items()), flush=True)
os.environ["DTB_BB"] = "0"
stack = torch.from_numpy(np.stack([workloads.c3_image(i) for i in range(64)])).cuda()
out = torch.empty_like(stack)
ab("c3 W31 niblack", lambda: engine.binarize_batch(stack, 31, "niblack", -0.2, 128.0, out=out))
page = torch.from_numpy(workloads.c5_image()).cuda(); pout = torch.empty_like(page)
for w in (3, 19, 35, 51, 67):
    ab("c5 4096^2 W%d" % w, lambda: engine.binarize(page, w, "sauvola", 0.34, 128.0, want_tmap=False, out=pout))
c2 = page[:3508, :2480].contiguous(); c2o = torch.empty_like(c2)
for w in (15, 31, 63):
    ab("c2 3508x2480 W%d" % w, lambda: engine.binarize(c2, w, "sauvola", 0.34, 128.0, want_tmap=False, out=c2o))
