"""Small cases through both fast kernels (classic + warp-specialized) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1210_3165_b200 import engine, workloads
import oracle

img = workloads.c1_image()
wide = np.ascontiguousarray(np.concatenate([img, img[:, :200]], axis=1))  # 712 wide -> 2 column warps
for arr, win, meth, k in ((img, 15, "sauvola", 0.5), (wide, 63, "niblack", -0.2), (img[:100, :300], 31, "sauvola", 0.34)):
    b, _ = engine.binarize(arr, win, meth, k, 128.0, want_tmap=False)
    ok = np.array_equal(b.cpu().numpy(), oracle.binarize(arr, win, meth, k, tmap=False)[0])
    print(arr.shape, win, meth, "exact" if ok else "MISMATCH")
stack = torch.from_numpy(np.stack([workloads.c3_image(i, size=256) for i in range(3)])).cuda()
engine.binarize_batch(stack, 31, "niblack", -0.2, 128.0)
torch.cuda.synchronize()
print("done")
