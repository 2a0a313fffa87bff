"""Probe (scripts/, not product): host-side cost of one small binarize call -- the Python wrapper
against the bare C-ABI call -- and the device-side time of the same launches back to back."""
import cProfile, pstats, sys, time
import torch
sys.path.insert(0, '.')
from paper_1210_3165_b200 import _lib, engine, workloads
from paper_1210_3165_b200.engine import METHOD_CODES
img = torch.from_numpy(workloads.c1_image()).cuda()
out = torch.empty_like(img)
lib = _lib.lib()
N = 3000
def wrapped():
    engine.binarize(img, 15, "sauvola", 0.5, 128.0, want_tmap=False, out=out)
def raw():
    lib.dtb_binarize(img.data_ptr(), img.stride(0), img.shape[0], img.shape[1], 0, img.shape[0], 0,
                     img.shape[0], out.data_ptr(), out.stride(0), None, 0, 15, METHOD_CODES["sauvola"],
                     0.5, 128.0, None)
for name, fn in (("wrapper", wrapped), ("raw C-ABI", raw)):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(N): fn()
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print("%-10s host %.2f us/call   device %.2f us/call" % (name, (t1 - t0) / N * 1e6, e0.elapsed_time(e1) / N * 1e3))
pr = cProfile.Profile(); pr.enable()
for _ in range(N): wrapped()
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
