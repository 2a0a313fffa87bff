import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_3165_b200 import engine, workloads
mode, w = sys.argv[1], int(sys.argv[2])
img = torch.from_numpy(workloads.c5_image()).cuda()
outs = []
for rep in range(3):
    b, _ = engine.binarize(img, w, "sauvola", 0.5, 128.0, want_tmap=False)
    outs.append(b.cpu().numpy())
if mode == "save":
    np.save("/tmp/ref_c5.npy", outs[0])
else:
    ref = np.load("/tmp/ref_c5.npy")
    for o in outs:
        bad = np.argwhere(o != ref)
        if len(bad) == 0:
            print("identical"); continue
        ys, xs = bad[:, 0], bad[:, 1]
        print(f"{len(bad)} px differ; rows {ys.min()}..{ys.max()} ({len(np.unique(ys))} rows), cols {xs.min()}..{xs.max()} ({len(np.unique(xs))} cols)")
        print("  first rows:", np.unique(ys)[:12], " first cols:", np.unique(xs)[:12])
