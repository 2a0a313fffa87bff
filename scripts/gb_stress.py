"""One-off stress of the group-bound kernel against the C oracle (GPU box):
python scripts/gb_stress.py N -> prints the number of bit-exact cases out of N."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DTB_GB"] = "1"
import oracle  # noqa: E402
from paper_1210_3165_b200 import _lib, engine, workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
ok = ran = 0
rng = np.random.default_rng(777)
for i in range(n):
    h = int(rng.integers(1, 900))
    w = 16 * int(rng.integers(96, 400))
    kind = int(rng.integers(0, 3))
    if kind == 0:
        img = workloads.doc_gray(h, w, int(rng.integers(0, 1 << 30)), max(1, h * w // 3000))
    elif kind == 1:
        img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    else:
        base = rng.integers(0, 256, (1, w // 64 + 1)).repeat(64, 1)[:, :w]
        img = np.clip(base + rng.integers(-3, 4, (h, w)), 0, 255).astype(np.uint8)
    win = int(2 * rng.integers(1, 128) + 1)
    k = float(rng.uniform(0.005, 1.0))
    r = float(rng.uniform(0.5, 400.0))
    got, _ = engine.binarize(img, win, "sauvola", k, r, want_tmap=False)
    ran += _lib.lib().dtb_last_kernel() == b"gb_kernel"
    want, _ = oracle.binarize(img, win, "sauvola", k, r, tmap=False, threads=16)
    if np.array_equal(got.cpu().numpy(), want):
        ok += 1
    else:
        print("MISMATCH", i, img.shape, win, k, r, kind, flush=True)
print(f"{ok}/{n} bit-exact, {ran} on gb_kernel")
