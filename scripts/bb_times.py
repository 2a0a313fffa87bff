"""Per-CTA timeline of one bb_kernel launch (dtb_debug_bb_times): which pipelines finish last."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1210_3165_b200 import _lib, engine, workloads

img = workloads.c4_image()
dev = torch.from_numpy(img).cuda()
L = _lib.lib()
buf = torch.zeros(4 * 8192, dtype=torch.int64, device='cuda')
engine.binarize(dev, 127, "sauvola", 0.34, 128.0, want_tmap=False)
L.dtb_debug_bb_times(buf.data_ptr(), 8192)
engine.binarize(dev, 127, "sauvola", 0.34, 128.0, want_tmap=False)
torch.cuda.synchronize()
L.dtb_debug_bb_times(None, 0)
t = buf.view(-1, 4).cpu().numpy().astype(np.float64)
n = int((t[:, 1] > 0).sum())
t = t[:n]
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 19
print("ctas", n, "span us %.1f" % en.max(), "start max %.1f" % st.max())
dur = en - st
print("duration us: min %.1f p50 %.1f p90 %.1f max %.1f" % (dur.min(), np.median(dur), np.percentile(dur, 90), dur.max()))
strip = np.arange(n) % ns
band = np.arange(n) // ns
for s_ in range(ns):
    m = strip == s_
    print("strip %2d mean %.1f max %.1f exact %d" % (s_, dur[m].mean(), dur[m].max(), t[m, 2].sum()))
order = np.argsort(-en)[:15]
for i in order:
    print("cta %5d strip %2d band %3d start %.1f end %.1f dur %.1f exact %d" % (i, strip[i], band[i], st[i], en[i], dur[i], t[i, 2]))
