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


def mask_offsets(structure, w):
    """masks.py:28-64 + 98-114: GS-1..GS-6 / full offsets, row-major (dy outer, dx inner)."""
    r = w // 2

    def member(dx, dy):
        cross = dx == 0 or dy == 0
        xx = dx == dy or dx == -dy
        ring = max(abs(dx), abs(dy)) == r
        return {"gs1": cross, "gs2": xx, "gs3": cross or xx, "gs4": dy == 0 or xx,
                "gs5": ring or (dx == 0 and dy == 0), "gs6": cross or ring,
                "full": True}[structure]

    return [(dx, dy) for dy in range(-r, r + 1) for dx in range(-r, r + 1) if member(dx, dy)]


def sampled_sums(img, offsets):
    """stats.py:133-147 _accumulate, in exact integers: (S, Q, count) over in-bounds offsets."""
    img = np.asarray(img, dtype=np.int64)
    h, w = img.shape
    S = np.zeros((h, w), np.int64)
    Q = np.zeros((h, w), np.int64)
    n = np.zeros((h, w), np.int64)
    for dx, dy in offsets:
        y0, y1 = max(0, -dy), min(h, h - dy)
        x0, x1 = max(0, -dx), min(w, w - dx)
        if y0 >= y1 or x0 >= x1:
            continue
        v = img[y0 + dy:y1 + dy, x0 + dx:x1 + dx]
        S[y0:y1, x0:x1] += v
        Q[y0:y1, x0:x1] += v * v
        n[y0:y1, x0:x1] += 1
    return S, Q, n


def mean_std_sampled(img, structure, w):
    """stats.py:150-163 (fp64 sums of integers are exact, so integer sums give the same bits)."""
    S, Q, n = sampled_sums(img, mask_offsets(structure, w))
    mean, std = finish(S, Q, n)
    return mean, std, n


def threshold_map(mean, std, method, k, r=128.0):
    """threshold.py:143-147 / metrics.py:126-129."""
    if method == "sauvola":
        return mean * (1.0 + k * (std / r - 1.0))
    return mean + k * std


def evaluate_counts(pred, gt):
    """metrics.py:52-61 -> (tp, tn, fp, fn, recall, precision, f_measure)."""
    pf = np.asarray(pred) == 0
    gf = np.asarray(gt) == 0
    tp = int(np.count_nonzero(pf & gf))
    fp = int(np.count_nonzero(pf & ~gf))
    fn = int(np.count_nonzero(~pf & gf))
    tn = pf.size - tp - fp - fn
    recall = tp / (tp + fn) if tp + fn else 0.0
    precision = tp / (tp + fp) if tp + fp else 0.0
    fm = 2 * recall * precision / (recall + precision) if recall + precision else 0.0
    return tp, tn, fp, fn, recall, precision, fm


def sweep(img, gt, method, engine, mask, w_grid, k_grid, r=128.0):
    """metrics.py:105-136 for sauvola/niblack: ([(w, k, fm)], best) with the strict-> tie rule."""
    img = np.asarray(img, dtype=np.uint8)
    ws = sorted(int(w) for w in w_grid)
    ks = sorted(float(k) for k in k_grid)
    cells, best = [], None
    for w in ws:
        if engine in ("naive", "integral") or mask == "full":
            mean, std = finish(*window_sums_integral(img, w))
        else:
            mean, std, _ = mean_std_sampled(img, mask, w)
        for k in ks:
            tmap = threshold_map(mean, std, method, k, r)
            pred = np.where(img.astype(np.float64) < tmap, 0, 255)
            cell = (w, k, evaluate_counts(pred, gt)[6])
            cells.append(cell)
            if best is None or cell[2] > best[2]:
                best = cell
    return cells, best


def otsu_threshold(img):
    """threshold.py:55-88: Otsu T with the strict-> smallest-T tie rule, Python arithmetic."""
    img = np.asarray(img, dtype=np.uint8)
    hist = np.bincount(img.ravel(), minlength=256).astype(np.int64)
    total = int(hist.sum())
    sum_all = int(np.dot(hist, np.arange(256, dtype=np.int64)))
    best_t, best_var = -1, -1.0
    wb = sumb = 0
    for t in range(256):
        wb += int(hist[t])
        sumb += t * int(hist[t])
        if wb == 0:
            continue
        wf = total - wb
        if wf == 0:
            break
        mb = sumb / wb
        mf = (sum_all - sumb) / wf
        var = wb * wf * (mb - mf) ** 2
        if var > best_var:
            best_var, best_t = var, t
    if best_t < 0:
        return int(img.flat[0])
    return best_t + 1
