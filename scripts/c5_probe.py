"""C5 (4096^2, W3..W243) timing probe (GPU box): each window's kernel time under three L2
states -- dirty flush (512 MiB memset: the evicted dirty lines are written back during the
timed kernel), clean flush (memset, then a 512 MiB read of another buffer), and warm (no
flush) -- plus an empty-launch floor.  Plans print with DTB_PRINT_PLAN=1.

    python scripts/c5_probe.py [--windows 3,67,131,243] [--bb 0|1|2]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1210_3165_b200 import _lib, engine, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--windows", default="3,19,67,115,131,243")
ap.add_argument("--reps", type=int, default=12)
ap.add_argument("--bb", default=None)
a = ap.parse_args()
if a.bb is not None:
    os.environ["DTB_BB"] = a.bb

img = torch.from_numpy(workloads.c5_image()).cuda()
out = torch.empty_like(img)
dirty = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(512 << 20 // 4, dtype=torch.int32, device="cuda")
acc = torch.empty((), dtype=torch.int64, device="cuda")


def flush(mode):
    if mode in ("dirty", "clean"):
        dirty.zero_()
    if mode == "clean":
        acc.copy_(clean.sum(dtype=torch.int64))


def timed(fn, mode):
    ts = []
    for _ in range(a.reps):
        flush(mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts[2:]), 4)


rows = []
noop = torch.empty(1, device="cuda")
rows.append({"what": "empty torch launch", "warm": timed(lambda: noop.add_(0), "none")})
for w in [int(x) for x in a.windows.split(",")]:
    fn = lambda: engine.binarize(img, w, "sauvola", 0.5, 128.0, want_tmap=False, out=out)  # noqa: E731
    fn()
    r = {"window": w, "kernel": _lib.lib().dtb_last_kernel().decode()}
    for mode in ("dirty", "clean", "none"):
        r[mode] = timed(fn, mode)
    r["clean_gbs"] = round(2 * img.numel() / (r["clean"] / 1e3) / 1e9, 1)
    rows.append(r)
    print(json.dumps(r), flush=True)
print(json.dumps(rows[0]))
