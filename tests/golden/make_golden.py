"""Generate golden fixtures by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--skip-big]

Writes (all committed; nothing here reads /root/reference at test time):

* small.npz      -- ~80 small cases: input, params, and the reference's
                    binarize(engine="integral") binary + tmap, mean_std_integral
                    mean/std/count; each case also checked naive == integral.
* to_gray.json   -- sha256 of the reference to_gray over all 2^24 RGB triples
                    (r-major order), plus every triple where it differs from
                    exact integer half-up rounding (the fp64 tie cases).
* sampled.npz    -- GS-mask ("sampled" engine) cases: input, structure, W and sha256 of
                    the reference's mean_std_sampled mean/std/count and of
                    binarize(engine="sampled") binary/tmap.
* metrics.npz    -- evaluate() counts/ratios on random bi-level pairs and full sweep()
                    grids (cells + best) on gen_synthetic pages (§8 row f2).
* otsu.npz       -- images + the reference's otsu_threshold T (§8 row f3).
* acceptance.npz -- the reference acceptance suite's AC5 corpus with its Otsu F-measure and
                    best (W, k, FM) sweep cells for the naive engine and gs1..gs6.
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


STRUCTS = ("gs1", "gs2", "gs3", "gs4", "gs5", "gs6")


def make_sampled(rng):
    out, meta = {}, []
    shapes = [(1, 1), (1, 17), (17, 1), (5, 5), (24, 37), (40, 33), (64, 64), (9, 130)]
    i = 0
    for st in STRUCTS:
        for (h, w) in shapes:
            for win in (3, 7, 21):
                img = rng.integers(0, 256, (h, w)).astype(np.uint8)
                if i % 5 == 0:  # document-like: mostly light, few dark strokes
                    img = np.where(rng.random((h, w)) < 0.1, rng.integers(0, 60, (h, w)),
                                   rng.integers(170, 230, (h, w))).astype(np.uint8)
                mask = ref.make_mask(st, win)
                mean, std, count = ref.mean_std_sampled(img, mask)
                method = "sauvola" if i % 2 == 0 else "niblack"
                k = 0.34 if method == "sauvola" else -0.2
                kw = {"k_sauvola": k} if method == "sauvola" else {"k_niblack": k}
                b, t = ref.binarize(img, ref.BinarizationParams(
                    method=method, engine="sampled", mask=st, window=win, **kw))
                out[f"img{i}"] = img
                meta.append({"structure": st, "win": win, "method": method, "k": k,
                             "mean": sha(mean), "std": sha(std),
                             "count": sha(count.astype(np.int64)),
                             "binary": sha(b), "tmap": sha(t)})
                i += 1
    # the reference's default parameters (sauvola / sampled / gs3 / W=21) on a larger page
    img = workloads.doc_gray(300, 410, 7, 40)
    b, t = ref.binarize(img)
    out[f"img{i}"] = img
    meta.append({"structure": "gs3", "win": 21, "method": "sauvola", "k": 0.34,
                 "binary": sha(b), "tmap": sha(t), "default_params": True})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "sampled.npz"), **out)
    print(f"sampled.npz: {len(meta)} cases")


def make_metrics(rng):
    from docthresh.bench import SyntheticSpec, gen_synthetic
    out, meta = {}, {"evaluate": [], "sweep": []}
    for i in range(12):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        fr = float(rng.choice([0.0, 0.05, 0.3, 0.9, 1.0]))
        pred = np.where(rng.random((h, w)) < fr, 0, 255).astype(np.uint8)
        gt = np.where(rng.random((h, w)) < 0.3, 0, 255).astype(np.uint8)
        if i % 4 == 3:
            gt = pred.copy()
        rep = ref.evaluate(pred, gt)
        out[f"pred{i}"], out[f"gt{i}"] = pred, gt
        meta["evaluate"].append([rep.tp, rep.tn, rep.fp, rep.fn, rep.recall, rep.precision,
                                 rep.f_measure])
    pages = [gen_synthetic(), gen_synthetic(SyntheticSpec(width=300, height=180, noise_seed=3,
                                                          noise_amplitude=20))]
    for p, (img, gt) in enumerate(pages):
        out[f"page{p}"], out[f"page_gt{p}"] = img, gt
    cases = [
        (0, "sauvola", "sampled", "gs3", None, None, 128.0),
        (0, "sauvola", "naive", "gs3", [21], [0.34], 128.0),
        (0, "sauvola", "sampled", "gs2", [11, 21], [0.2, 0.4], 128.0),
        (0, "niblack", "integral", "gs3", [11, 21], [-0.5, -0.2], 128.0),
        (0, "otsu", "sampled", "gs3", [3, 5], [0.1], 128.0),
        (1, "sauvola", "integral", "gs3", [41, 3, 15], [0.5, 0.05, 0.2, 0.34], 100.0),
        (1, "niblack", "sampled", "gs5", [7, 31], [-0.3, 0.0, 0.2], 128.0),
        (1, "sauvola", "sampled", "gs6", [9], [0.1, 0.3], 64.0),
        (1, "sauvola", "sampled", "full", [9, 13], [0.25], 128.0),
    ]
    for page, method, eng, mask, wg, kg, r in cases:
        img, gt = pages[page]
        kw = {}
        if wg is not None:
            kw = {"w_grid": wg, "k_grid": kg}
        res = ref.sweep(img, gt, method=method, engine=eng, mask=mask, r=r, **kw)
        meta["sweep"].append({"page": page, "method": method, "engine": eng, "mask": mask,
                              "w_grid": wg, "k_grid": kg, "r": r,
                              "cells": [[c.w, c.k, c.f_measure] for c in res.cells],
                              "best": [res.best.w, res.best.k, res.best.f_measure],
                              "csv": res.to_csv()})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    print(f"metrics.npz: {len(meta['evaluate'])} evaluate, {len(meta['sweep'])} sweep cases")


def make_otsu(rng):
    """otsu.npz: images and the reference's otsu_threshold (threshold.py:55-88) for each."""
    out, ts = {}, []
    imgs = [np.full((4, 7), 77, np.uint8), np.array([[0, 255]], np.uint8),
            np.array([[10] * 50 + [200] * 50], np.uint8), np.zeros((1, 1), np.uint8)]
    for _ in range(10):
        h, w = int(rng.integers(1, 200)), int(rng.integers(1, 200))
        imgs.append(rng.integers(0, 256, (h, w)).astype(np.uint8))
    for _ in range(6):  # bimodal pages, the case Otsu is for
        h, w = int(rng.integers(50, 300)), int(rng.integers(50, 300))
        lo, hi = int(rng.integers(10, 90)), int(rng.integers(150, 240))
        a = np.where(rng.random((h, w)) < rng.uniform(0.05, 0.5), lo, hi)
        imgs.append(np.clip(a + rng.normal(0, rng.uniform(1, 30), (h, w)), 0, 255).astype(np.uint8))
    imgs.append(workloads.doc_gray(700, 500, 11, 300))
    for _ in range(4):  # few-level images: many exact variance ties
        vals = rng.choice(256, int(rng.integers(2, 5)), replace=False)
        imgs.append(rng.choice(vals, (int(rng.integers(3, 60)), int(rng.integers(3, 60)))).astype(np.uint8))
    for i, img in enumerate(imgs):
        out[f"img{i}"] = img
        ts.append(int(ref.otsu_threshold(img)))
    out["t"] = np.array(ts, np.int32)
    np.savez_compressed(os.path.join(HERE, "otsu.npz"), **out)
    print(f"otsu.npz: {len(ts)} images")


def make_acceptance():
    """acceptance.npz: the reference acceptance suite's AC5 corpus (synthetic_corpus(10)) with
    the reference's Otsu F-measure and best sweep cells (naive engine and each GS structure,
    default grids) per page (test_acceptance.py:165-199)."""
    from docthresh.bench import synthetic_corpus
    out, meta = {}, []
    for i, (img, gt) in enumerate(synthetic_corpus(10)):
        out[f"img{i}"], out[f"gt{i}"] = img, gt
        otsu_fm = ref.evaluate(ref.apply_global(img, ref.otsu_threshold(img)), gt).f_measure
        naive = ref.sweep(img, gt, method="sauvola", engine="naive").best
        gs = {}
        for st in STRUCTS:
            b = ref.sweep(img, gt, method="sauvola", engine="sampled", mask=st).best
            gs[st] = [b.w, b.k, b.f_measure]
        meta.append({"otsu_fm": otsu_fm, "naive": [naive.w, naive.k, naive.f_measure], "gs": gs})
        print(f"acceptance page {i}", flush=True)
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "acceptance.npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-big", action="store_true")
    ap.add_argument("--only", choices=["small", "to_gray", "configs", "sampled", "metrics", "otsu", "acceptance"])
    a = ap.parse_args()
    rng = np.random.default_rng(20261019)
    if a.only in (None, "small"):
        make_small(rng)
    if a.only in (None, "to_gray"):
        make_to_gray()
    if a.only in (None, "sampled"):
        make_sampled(np.random.default_rng(20261020))
    if a.only in (None, "metrics"):
        make_metrics(np.random.default_rng(20261021))
    if a.only in (None, "otsu"):
        make_otsu(np.random.default_rng(20261022))
    if a.only in (None, "acceptance"):
        make_acceptance()
    if a.only in (None, "configs"):
        make_configs(a.skip_big)


if __name__ == "__main__":
    main()
