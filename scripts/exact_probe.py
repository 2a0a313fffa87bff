"""Probe (scripts/, not product): exact-path group counts of bb_kernel on row crops of the C4 page."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1210_3165_b200 import _lib, engine, workloads
img = workloads.c4_image()
L = _lib.lib()
cnt = ctypes.c_uint64(0)
def count(a):
    dev = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    L.dtb_debug_bb_exact(ctypes.byref(cnt), 1)
    engine.binarize(dev, 127, "sauvola", 0.34, 128.0, want_tmap=False)
    torch.cuda.synchronize()
    L.dtb_debug_bb_exact(ctypes.byref(cnt), 1)
    return cnt.value, L.dtb_last_kernel().decode()
for (a, b) in ((0, 512), (512, 1024), (8000, 8512), (15360, 15872), (15872, 16384), (16000, 16384)):
    print("rows", a, b, count(img[a:b]))
for c0 in range(0, 16384, 2048):
    print("rows 15872-16384 cols", c0, c0 + 2048, count(img[15872:16384, c0:c0 + 2048]))
for (a, b) in ((14000, 16384), (8192, 16384), (4096, 16384), (1024, 16384), (0, 16384)):
    print("rows", a, b, count(img[a:b]))
