"""Seeded synthetic document images for the five BASELINE.json configurations.

BASELINE.json only says "seeded synthetic"; this module fixes the recipe
 so that the bench, the GPU parity tests and the golden
fixtures generated from the reference (tests/golden/make_golden.py) all see
byte-identical inputs.  The reference's own generator (bench.py:86-102 in the
reference package) is a different, ±5-uniform-noise design and is not used.

Recipe (gray):  linear illumination ramp (along x, or diagonal), dark
axis-aligned rectangular strokes, additive float32 Gaussian noise, then
``np.rint`` and ``clip(0, 255)``.  Draw order: stroke parameters, then noise.

These are test/bench inputs, not part of the binarization path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED_BASE = 1210_3165


def _draw_strokes(img: np.ndarray, rng: np.random.Generator, n: int,
                  thick: tuple[int, int], length: tuple[int, int],
                  ink: tuple[float, float], channels: int = 0) -> None:
    h, w = img.shape[:2]
    horiz = rng.random(n) < 0.5
    t = rng.integers(thick[0], thick[1] + 1, n)
    ln = rng.integers(length[0], length[1] + 1, n)
    y0 = rng.integers(0, h, n)
    x0 = rng.integers(0, w, n)
    if channels:
        val = rng.uniform(ink[0], ink[1], (n, channels)).astype(np.float32)
    else:
        val = rng.uniform(ink[0], ink[1], n).astype(np.float32)
    hh = np.where(horiz, t, ln)
    ww = np.where(horiz, ln, t)
    for i in range(n):
        img[y0[i]:y0[i] + hh[i], x0[i]:x0[i] + ww[i]] = val[i]


def _finish(img: np.ndarray, rng: np.random.Generator, sigma: float) -> np.ndarray:
    img += rng.standard_normal(img.shape, dtype=np.float32) * np.float32(sigma)
    np.rint(img, out=img)
    np.clip(img, 0, 255, out=img)
    return img.astype(np.uint8)


def doc_gray(h: int, w: int, seed: int, n_strokes: int, ramp=(150.0, 230.0),
             diagonal: bool = False, sigma: float = 8.0) -> np.ndarray:
    """One gray (h, w) uint8 synthetic page (BASELINE configs 1, 3, 4, 5)."""
    rng = np.random.default_rng(seed)
    x = np.linspace(0.0, 1.0, w, dtype=np.float32)
    if diagonal:
        y = np.linspace(0.0, 1.0, h, dtype=np.float32)
        frac = (x[None, :] + y[:, None]) * np.float32(0.5)
    else:
        frac = np.broadcast_to(x[None, :], (h, w))
    img = np.float32(ramp[0]) + np.float32(ramp[1] - ramp[0]) * frac
    img = np.ascontiguousarray(img, dtype=np.float32)
    _draw_strokes(img, rng, n_strokes, (2, 4), (8, 40), (20.0, 60.0))
    return _finish(img, rng, sigma)


def doc_rgb(h: int, w: int, seed: int, n_strokes: int, sigma: float = 10.0) -> np.ndarray:
    """(h, w, 3) uint8 page with a per-channel bilinear illumination field (config 2)."""
    rng = np.random.default_rng(seed)
    corners = rng.uniform(140.0, 235.0, (3, 2, 2)).astype(np.float32)
    y = np.linspace(0.0, 1.0, h, dtype=np.float32)[:, None]
    x = np.linspace(0.0, 1.0, w, dtype=np.float32)[None, :]
    img = np.empty((h, w, 3), dtype=np.float32)
    for c in range(3):
        (a, b), (cc, d) = corners[c]
        img[:, :, c] = (a * (1 - y) * (1 - x) + b * (1 - y) * x
                        + cc * y * (1 - x) + d * y * x)
    _draw_strokes(img, rng, n_strokes, (2, 5), (8, 40), (10.0, 70.0), channels=3)
    return _finish(img, rng, sigma)


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration: input recipe plus method parameters."""

    name: str
    method: str
    windows: tuple
    k: float
    r: float = 128.0
    description: str = ""


# BASELINE.json "configs" in order.  k for Niblack is k_niblack; k_sauvola then
# stays at its default 0.34 so that the reference's validate() accepts it.
CONFIGS = {
    "c1": Config("c1", "sauvola", (15,), 0.5, 128.0, "512x512 gray, Sauvola W=15 k=0.5 R=128"),
    "c2": Config("c2", "sauvola", (15, 31, 63), 0.5, 128.0,
                 "3508x2480 RGB page -> to_gray -> Sauvola k=0.5 R=128, W in {15,31,63}"),
    "c3": Config("c3", "niblack", (31,), -0.2, 128.0, "64 x 2048x2048 gray, Niblack W=31 k=-0.2"),
    "c4": Config("c4", "sauvola", (127,), 0.34, 128.0,
                 "16384x16384 gray, Sauvola W=127 k=0.34 R=128, row bands with 63-row halo"),
    "c5": Config("c5", "sauvola", tuple(range(3, 256, 16)), 0.5, 128.0,
                 "4096x4096 gray (sigma 12), Sauvola k=0.5 R=128, W=3,19,...,243"),
}


def c1_image() -> np.ndarray:
    return doc_gray(512, 512, SEED_BASE + 1, 400)


def c2_rgb() -> np.ndarray:
    return doc_rgb(3508, 2480, SEED_BASE + 2, 6000)


def c3_image(i: int, size: int = 2048) -> np.ndarray:
    scale = (size * size) / (512 * 512)
    return doc_gray(size, size, SEED_BASE + 300 + i, int(round(400 * scale)))


def c4_image(size: int = 16384) -> np.ndarray:
    scale = (size * size) / (512 * 512)
    return doc_gray(size, size, SEED_BASE + 4, int(round(400 * scale)),
                    ramp=(120.0, 240.0), diagonal=True)


def c5_image(size: int = 4096) -> np.ndarray:
    scale = (size * size) / (512 * 512)
    return doc_gray(size, size, SEED_BASE + 5, int(round(400 * scale)), sigma=12.0)
