"""Generate golden fixtures by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--skip-big]

Writes (all committed; nothing here reads /root/reference at test time):

* small.npz      -- ~80 small cases: input, params, and the reference's
                    binarize(engine="integral") binary + tmap, mean_std_integral
                    mean/std/count; each case also checked naive == integral.
* to_gray.json   -- sha256 of the reference to_gray over all 2^24 RGB triples
                    (r-major order), plus every triple where it differs from
                    exact integer half-up rounding (the fp64 tie cases).
* configs.json   -- per BASELINE config: sha256 of the generated input and of
                    the reference's binary output (and tmap for c1/c5), at
                    FULL size.  c4 takes ~90 s and ~21 GB RSS.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import docthresh as ref  # noqa: E402  (the reference, via PYTHONPATH)

from paper_1210_3165_b200 import workloads  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_binarize(img, win, method, k, r, engine="integral"):
    kw = {"k_sauvola": k} if method == "sauvola" else {"k_niblack": k}
    p = ref.BinarizationParams(method=method, engine=engine, window=win, r=r, **kw)
    return ref.binarize(img, p)


def small_cases(rng):
    cases = []
    # edge shapes
    for h, w in [(1, 1), (1, 9), (9, 1), (2, 2), (3, 40), (40, 3), (1, 64), (64, 1)]:
        cases.append((rng.integers(0, 256, (h, w)).astype(np.uint8), 3))
        cases.append((rng.integers(0, 256, (h, w)).astype(np.uint8), 15))
    # windows larger than the image
    for win in (63, 127, 255):
        cases.append((rng.integers(0, 256, (int(rng.integers(5, 40)), int(rng.integers(5, 40))))
                      .astype(np.uint8), win))
    # constant and extreme images
    cases.append((np.full((17, 23), 120, np.uint8), 5))
    cases.append((np.full((9, 9), 0, np.uint8), 3))
    cases.append((np.full((9, 9), 255, np.uint8), 7))
    ext = np.zeros((16, 16), np.uint8)
    ext[:, 8:] = 255
    cases.append((ext, 9))
    chk = ((np.indices((20, 20)).sum(0) % 2) * 255).astype(np.uint8)
    cases.append((chk, 3))
    # random sizes / windows like the reference's own tests (conftest.py:10-16)
    for _ in range(40):
        h, w = int(rng.integers(8, 65)), int(rng.integers(8, 65))
        win = int(rng.choice([3, 5, 7, 9, 15, 21, 31, 41, 63]))
        cases.append((rng.integers(0, 256, (h, w)).astype(np.uint8), win))
    # document-like crops (low noise -> many near-ties)
    doc = workloads.c1_image()
    for _ in range(8):
        y, x = int(rng.integers(0, 400)), int(rng.integers(0, 400))
        h, w = int(rng.integers(16, 100)), int(rng.integers(16, 100))
        cases.append((np.ascontiguousarray(doc[y:y + h, x:x + w]),
                      int(rng.choice([3, 15, 31, 63]))))
    return cases


def make_small(rng):
    out = {}
    meta = []
    for i, (img, win) in enumerate(small_cases(rng)):
        if i % 3 == 0:
            method, k, r = "niblack", float(rng.choice([-0.2, -0.5, 0.0, 0.3])), 128.0
        else:
            method = "sauvola"
            k = float(rng.choice([0.34, 0.5, 0.05, 0.9, 0.2]))
            r = float(rng.choice([128.0, 64.0, 100.0, 256.0]))
        binary, tmap = ref_binarize(img, win, method, k, r, "integral")
        b2, t2 = ref_binarize(img, win, method, k, r, "naive")
        assert np.array_equal(binary, b2) and np.array_equal(tmap, t2), i
        mean, std, count = ref.mean_std_integral(img, win)
        out[f"img{i}"] = img
        out[f"binary{i}"] = binary
        out[f"tmap{i}"] = tmap
        out[f"mean{i}"] = mean
        out[f"std{i}"] = std
        out[f"count{i}"] = count.astype(np.int32)
        meta.append({"win": win, "method": method, "k": k, "r": r})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print(f"small.npz: {len(meta)} cases")


def make_to_gray():
    r = np.repeat(np.arange(256, dtype=np.uint8), 65536)
    g = np.tile(np.repeat(np.arange(256, dtype=np.uint8), 256), 256)
    b = np.tile(np.arange(256, dtype=np.uint8), 65536)
    rgb = np.stack([r, g, b], axis=-1).reshape(4096, 4096, 3)
    gray = ref.to_gray(rgb).reshape(-1)
    x = 299 * r.astype(np.int64) + 587 * g.astype(np.int64) + 114 * b.astype(np.int64)
    exact = (x + 500) // 1000
    diff = np.nonzero(gray != exact)[0]
    ties = int(np.count_nonzero(x % 1000 == 500))
    doc = {
        "order": "index = r*65536 + g*256 + b",
        "sha256": sha(gray),
        "n_exact_half_ties": ties,
        "differs_from_integer_half_up": [[int(r[i]), int(g[i]), int(b[i]), int(gray[i])]
                                         for i in diff],
    }
    with open(os.path.join(HERE, "to_gray.json"), "w") as f:
        json.dump(doc, f)
    print(f"to_gray.json: {len(diff)} triples differ from integer half-up ({ties} ties)")


def make_configs(skip_big: bool):
    path = os.path.join(HERE, "configs.json")
    doc = json.load(open(path)) if os.path.exists(path) else {}
    cfg = workloads.CONFIGS

    def run(key, img, win, c, with_tmap=False):
        t0 = time.time()
        b, t = ref_binarize(img, win, c.method, c.k, c.r)
        entry = {"input": sha(img), "shape": list(img.shape), "win": win,
                 "method": c.method, "k": c.k, "r": c.r, "binary": sha(b),
                 "ink_fraction": float((b == 0).mean())}
        if with_tmap:
            entry["tmap"] = sha(t)
        doc[key] = entry
        print(f"{key}: {time.time() - t0:.1f}s", flush=True)
        with open(path, "w") as f:
            json.dump(doc, f, indent=1)

    c1 = workloads.c1_image()
    run("c1/w15", c1, 15, cfg["c1"], with_tmap=True)
    mean, std, count = ref.mean_std_integral(c1, 15)
    doc["c1/w15"]["mean"] = sha(mean)
    doc["c1/w15"]["std"] = sha(std)
    rgb = workloads.c2_rgb()
    gray = ref.to_gray(rgb)
    doc["c2/rgb"] = {"input": sha(rgb), "gray": sha(gray)}
    for win in cfg["c2"].windows:
        run(f"c2/w{win}", gray, win, cfg["c2"])
    if skip_big:
        return
    for win in cfg["c5"].windows:
        run(f"c5/w{win}", workloads.c5_image(), win, cfg["c5"], with_tmap=(win == 35))
    for i in range(64):
        run(f"c3/img{i}", workloads.c3_image(i), 31, cfg["c3"])
    run("c4/w127", workloads.c4_image(), 127, cfg["c4"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-big", action="store_true")
    ap.add_argument("--only", choices=["small", "to_gray", "configs"])
    a = ap.parse_args()
    rng = np.random.default_rng(20261019)
    if a.only in (None, "small"):
        make_small(rng)
    if a.only in (None, "to_gray"):
        make_to_gray()
    if a.only in (None, "configs"):
        make_configs(a.skip_big)


if __name__ == "__main__":
    main()
