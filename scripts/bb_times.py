"""Per-CTA timeline of one bb_kernel launch (dtb_debug_bb_times): warm-up and main-phase
durations, and which pipelines finish last.  scripts/, analysis only.

    python scripts/bb_times.py [page|band] [bands=8]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1210_3165_b200 import _lib, engine, workloads  # noqa: E402
from paper_1210_3165_b200 import distributed as D  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "page"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
img = workloads.c4_image()
H, Wd = img.shape
L = _lib.lib()
buf = torch.zeros(4 * 16384, dtype=torch.int64, device='cuda')
if mode == "page":
    dev = torch.from_numpy(img).cuda()
    run = lambda: engine.binarize(dev, 127, "sauvola", 0.34, 128.0, want_tmap=False)  # noqa: E731
elif mode == "bandbuf":  # the band and its halos in one buffer (single-buffer kernel)
    y0, y1 = D.band_bounds(H, nb, nb // 2)
    ha, hz = D.halo_bounds(H, y0, y1, 63)
    bb = torch.from_numpy(np.ascontiguousarray(img[ha:hz])).cuda()
    out = torch.empty((y1 - y0, Wd), dtype=torch.uint8, device='cuda')
    run = lambda: engine.binarize_band(bb, ha, H, y0, y1, 127, "sauvola", 0.34, 128.0, out=out)  # noqa: E731
else:
    y0, y1 = D.band_bounds(H, nb, nb // 2)
    ha, hz = D.halo_bounds(H, y0, y1, 63)
    segs_t = [torch.from_numpy(np.ascontiguousarray(img[a:b])).cuda() for a, b in ((ha, y0), (y0, y1), (y1, hz))]
    segs = [(t.data_ptr(), t.stride(0), t.shape[0], Wd) for t in segs_t]
    out = torch.empty((y1 - y0, Wd), dtype=torch.uint8, device='cuda')
    run = lambda: engine.binarize_segments(segs, ha, H, y0, y1, 127, "sauvola", 0.34, 128.0, out=out)  # noqa: E731
run()
L.dtb_debug_bb_times(buf.data_ptr(), 16384)
run()
torch.cuda.synchronize()
L.dtb_debug_bb_times(None, 0)
traw = buf.view(-1, 4).cpu().numpy()
t = traw.astype(np.float64)
t[:, 2] = (traw[:, 2] & 0xFFFF)
n = int((t[:, 1] > 0).sum())
t = t[:n]
t0 = t[:, 0].min()
st, en, wu = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 3] - t0) / 1e3
dur, warm = en - st, wu - st
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(2_000_000)
e0.record()
for _ in range(10):
    run()
e1.record()
torch.cuda.synchronize()
print(mode, "kernel ms %.4f" % (e0.elapsed_time(e1) / 10), L.dtb_last_kernel().decode())
print(mode, "ctas", n, "span us %.1f" % en.max(), "start max %.1f" % st.max())
for name, v in (("duration", dur), ("warm-up", warm), ("main", en - wu)):
    print("%-9s us: min %.1f p50 %.1f p90 %.1f max %.1f" % (name, v.min(), np.median(v), np.percentile(v, 90), v.max()))
# CTA -> strip (the launch plan: DTB_PLAN="strips pairs edge_pairs", from DTB_PRINT_PLAN=1's line)
import os
plan = [int(v) for v in os.environ.get("DTB_PLAN", "20 59 0").split()]
ns, npairs, npairs_e = plan
cta = np.arange(n) // 2  # pipelines 2c, 2c+1 share CTA c
if npairs_e == 0:
    strip = cta % ns
    band = 2 * ((cta // ns) % npairs) + (np.arange(n) % 2 == 0)
else:
    n_edge = 2 * npairs_e  # the edge strips' CTAs come first
    strip = np.where(cta < n_edge, np.where(cta % 2 == 1, ns - 1, 0), 1 + (cta - n_edge) % (ns - 2))
    band = np.where(cta < n_edge, 2 * (cta // 2), 2 * ((cta - n_edge) // (ns - 2))) + (np.arange(n) % 2 == 0)
for s_ in range(ns):
    m = strip == s_
    print("strip %2d n %4d dur mean %.1f max %.1f  warm mean %.1f  exact %d" % (s_, m.sum(), dur[m].mean(), dur[m].max(), warm[m].mean(), t[m, 2].sum()))
mi = (strip > 0) & (strip < ns - 1)
bmax = band[mi].max() + 1
for q in range(8):
    m = mi & (band * 8 // bmax == q)
    if m.any():
        print("interior bands octile %d: dur mean %.1f p90 %.1f max %.1f exact %d" % (q, dur[m].mean(), np.percentile(dur[m], 90), dur[m].max(), t[m, 2].sum()))
order = np.argsort(-en)[:8]
for i in order:
    print("cta %5d strip %2d band %3d start %.1f warm_end %.1f end %.1f exact %d last exact y %d g %d" % (i // 2, strip[i], band[i], st[i], wu[i], en[i], t[i, 2], (traw[i, 2] >> 16) & 0xFFFFFF, traw[i, 2] >> 40))
