"""One GS-kernel binarization of the 4096^2 C5 page (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1210_3165_b200 import engine, workloads  # noqa: E402

st = sys.argv[1] if len(sys.argv) > 1 else "gs3"
w = int(sys.argv[2]) if len(sys.argv) > 2 else 21
img = torch.from_numpy(workloads.c5_image()).cuda()
for _ in range(3):
    b, _ = engine.gs(img, st, w, "sauvola", 0.34, 128.0, want_tmap=False)
torch.cuda.synchronize()
print("ok", int((b == 0).sum()))
