"""Probe (scripts/, not product): the reference's default contract on C4 -- binary + fp64 tmap --
kernel time and golden hashes."""
import hashlib, json, os, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1210_3165_b200 import _lib, engine, workloads
img = workloads.c4_image()
dev = torch.from_numpy(img).cuda()
out = torch.empty_like(dev)
tm = torch.empty(img.shape, dtype=torch.float64, device="cuda")
res = engine.binarize(dev, 127, "sauvola", 0.34, 128.0, want_tmap=True, out=out, tmap_out=tm)
torch.cuda.synchronize()
print("kernel", _lib.lib().dtb_last_kernel().decode())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 5
e0.record()
for _ in range(n):
    res = engine.binarize(dev, 127, "sauvola", 0.34, 128.0, want_tmap=True, out=out, tmap_out=tm)
e1.record(); torch.cuda.synchronize()
print("binary+tmap ms %.4f" % (e0.elapsed_time(e1) / n))
gold = json.load(open("tests/golden/configs.json")).get("c4/w127", {})
b = res[0] if isinstance(res, (tuple, list)) else res
print("binary golden", hashlib.sha256(b.cpu().numpy().tobytes()).hexdigest() == gold.get("binary"))
