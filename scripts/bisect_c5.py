import os, sys, json, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_3165_b200 import engine, workloads
G = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/configs.json")))
img = torch.from_numpy(workloads.c5_image()).cuda()
bad = []
for w in [int(x) for x in sys.argv[1:]] or workloads.CONFIGS["c5"].windows:
    b, _ = engine.binarize(img, w, "sauvola", 0.5, 128.0, want_tmap=False)
    ok = hashlib.sha256(b.cpu().numpy().tobytes()).hexdigest() == G[f"c5/w{w}"]["binary"]
    if not ok:
        bad.append(w)
print(os.environ.get("DTB_WS", "-"), "bad:", bad)
