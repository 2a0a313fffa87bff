"""numpy restatement of the reference hot path (test infrastructure only).

Small sizes only; used to cross-check the C oracle and for the naive engine.
Each function cites the reference lines it restates
(/root/reference/pkg/src/docthresh).
"""

from __future__ import annotations

import numpy as np


def to_gray(rgb):
    """pnm.py:34-38."""
    rgb = np.asarray(rgb)
    acc = 0.299 * rgb[:, :, 0] + 0.587 * rgb[:, :, 1] + 0.114 * rgb[:, :, 2]
    return np.clip(np.floor(acc + 0.5), 0, 255).astype(np.uint8)


def window_sums_integral(img, w):
    """stats.py:82-91 (build_integral) + stats.py:177-189 (rect sums, count)."""
    img = np.asarray(img, dtype=np.uint8)
    h, iw = img.shape
    a = img.astype(np.int64)
    s = np.zeros((h + 1, iw + 1), dtype=np.int64)
    sq = np.zeros((h + 1, iw + 1), dtype=np.int64)
    s[1:, 1:] = a.cumsum(axis=0).cumsum(axis=1)
    sq[1:, 1:] = (a * a).cumsum(axis=0).cumsum(axis=1)
    r = w // 2
    ys, xs = np.arange(h), np.arange(iw)
    y0, y1 = np.maximum(ys - r, 0), np.minimum(ys + r, h - 1) + 1
    x0, x1 = np.maximum(xs - r, 0), np.minimum(xs + r, iw - 1) + 1
    S = s[np.ix_(y1, x1)] - s[np.ix_(y0, x1)] - s[np.ix_(y1, x0)] + s[np.ix_(y0, x0)]
    Q = sq[np.ix_(y1, x1)] - sq[np.ix_(y0, x1)] - sq[np.ix_(y1, x0)] + sq[np.ix_(y0, x0)]
    n = np.outer(y1 - y0, x1 - x0)
    return S, Q, n


def window_sums_naive(img, w):
    """stats.py:133-147 with the full mask (masks.py:98-114): W^2 shifted adds."""
    img = np.asarray(img, dtype=np.uint8)
    h, iw = img.shape
    f = img.astype(np.float64)
    total = np.zeros((h, iw))
    total_sq = np.zeros((h, iw))
    count = np.zeros((h, iw))
    r = w // 2
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            ya, yb = max(0, -dy), min(h, h - dy)
            xa, xb = max(0, -dx), min(iw, iw - dx)
            if ya >= yb or xa >= xb:
                continue
            total[ya:yb, xa:xb] += f[ya + dy:yb + dy, xa + dx:xb + dx]
            total_sq[ya:yb, xa:xb] += f[ya + dy:yb + dy, xa + dx:xb + dx] ** 2
            count[ya:yb, xa:xb] += 1.0
    return total, total_sq, count


def finish(S, Q, n):
    """stats.py:50-54."""
    S = np.asarray(S).astype(np.float64)
    Q = np.asarray(Q).astype(np.float64)
    n = np.asarray(n).astype(np.float64)
    mean = S / n
    var = Q / n - mean * mean
    return mean, np.sqrt(np.maximum(var, 0.0))


def binarize(img, w, method, k, r=128.0):
    """threshold.py:143-147 over the integral-engine statistics."""
    img = np.asarray(img, dtype=np.uint8)
    mean, std = finish(*window_sums_integral(img, w))
    if method == "sauvola":
        tmap = mean * (1.0 + k * (std / r - 1.0))
    else:
        tmap = mean + k * std
    return np.where(img.astype(np.float64) < tmap, 0, 255).astype(np.uint8), tmap
