"""Windowed mean / standard deviation engines on B200.

Drop-in for the reference's stats.py (/root/reference/pkg/src/docthresh/
stats.py:1-191).  All three engines return the same (mean f64, std f64,
count i64) the reference returns, bit for bit: exact integer window sums on
the device followed by the shared finishing step (stats.py:50-54) replayed in
fp64 round-to-nearest.  ``naive`` and ``integral`` share the O(1)-per-pixel
sliding-sum kernel; ``sampled`` runs the mask-restricted kernel (or the
sliding kernel for mask "full").
"""

from __future__ import annotations

import math
from typing import NamedTuple

import numpy as np

from . import engine
from .masks import SamplingMask, make_mask
from .validation import as_gray_image, check_coords, check_window


class WindowStats(NamedTuple):
    mean: float
    std: float
    count: int  # pixels actually used after border clipping


class IntegralPair(NamedTuple):
    """Zero-padded (H+1)x(W+1) int64 prefix-sum tables of x and x^2 (stats.py:37-41)."""

    sum_table: np.ndarray
    sqsum_table: np.ndarray


def _finish_scalar(total: int, total_sq: int, count: int) -> WindowStats:
    # stats.py:44-47 (scalar twin of the device finish; used on 1-pixel lookups only)
    mean = total / count
    var = total_sq / count - mean * mean
    return WindowStats(mean, math.sqrt(max(var, 0.0)), count)


def _validated(img):
    if engine.is_device_tensor(img):
        return img, False
    return as_gray_image(img), True


def _out(d, host):
    mean, std, cnt = d["mean"], d["std"], d["count"]
    if host:
        return mean.cpu().numpy(), std.cpu().numpy(), cnt.cpu().numpy().astype(np.int64)
    return mean, std, cnt.to(dtype=engine.torch_mod().int64)


def mean_std_integral(img, w: int):
    """stats.py:171-191: full clipped window, (mean, std, count)."""
    img, host = _validated(img)
    w = check_window(w)
    dev = engine.to_device(img)
    return _out(engine.window_stats(dev, w, want=("mean", "std", "count")), host)


def mean_std_naive(img, w: int):
    """stats.py:166-168: identical output to mean_std_integral (bitwise)."""
    img, host = _validated(img)
    w = check_window(w)
    dev = engine.to_device(img)
    return _out(engine.window_stats(dev, w, want=("mean", "std", "count")), host)


def mean_std_sampled(img, mask: SamplingMask):
    """stats.py:150-163: statistics over the in-bounds mask offsets."""
    img, host = _validated(img)
    dev = engine.to_device(img)
    if mask.structure == "full":
        return _out(engine.window_stats(dev, mask.window, want=("mean", "std", "count")), host)
    if mask.structure in engine.GS_CODES:
        return _out(engine.gs(dev, mask.structure, mask.window), host)
    return _out(engine.sampled(dev, mask.offsets), host)


def window_sums(img, w: int):
    """Exact (S, Q, count) of the clipped window per pixel (the integers stats.py
    builds with build_integral + the 4-corner gather, stats.py:82-91, 185-189)."""
    img, host = _validated(img)
    w = check_window(w)
    dev = engine.to_device(img)
    d = engine.window_stats(dev, w, want=("S", "Q", "count"))
    if host:
        return tuple(d[k].cpu().numpy() for k in ("S", "Q", "count"))
    return d["S"], d["Q"], d["count"]


def build_integral(img) -> IntegralPair:
    """stats.py:82-91: zero-padded int64 summed-area tables of f and f^2 (device-built)."""
    img = as_gray_image(img)
    s, sq = engine.integral_tables(engine.to_device(img))
    return IntegralPair(s.cpu().numpy(), sq.cpu().numpy())


def window_stats_naive(img, x: int, y: int, w: int) -> WindowStats:
    """stats.py:59-79: one pixel's clipped-window statistics."""
    img = as_gray_image(img)
    w = check_window(w)
    check_coords(img, x, y)
    S, Q, n = window_sums(img, w)
    return _finish_scalar(int(S[y, x]), int(Q[y, x]), int(n[y, x]))


def _rect_sum(table, y0, y1, x0, x1) -> int:
    return int(table[y1, x1] - table[y0, x1] - table[y1, x0] + table[y0, x0])


def window_stats_integral(ip: IntegralPair, x: int, y: int, w: int) -> WindowStats:
    """stats.py:98-109: same contract, answered from the integral tables."""
    w = check_window(w)
    h, iw = ip.sum_table.shape[0] - 1, ip.sum_table.shape[1] - 1
    if not (0 <= x < iw and 0 <= y < h):
        raise ValueError(f"coordinates ({x}, {y}) outside {iw}x{h} image")
    r = w // 2
    y0, y1 = max(y - r, 0), min(y + r, h - 1) + 1
    x0, x1 = max(x - r, 0), min(x + r, iw - 1) + 1
    return _finish_scalar(_rect_sum(ip.sum_table, y0, y1, x0, x1),
                          _rect_sum(ip.sqsum_table, y0, y1, x0, x1), (y1 - y0) * (x1 - x0))


def window_stats_sampled(img, mask: SamplingMask, x: int, y: int) -> WindowStats:
    """stats.py:112-128: one pixel's statistics over the in-bounds mask offsets."""
    img = as_gray_image(img)
    check_coords(img, x, y)
    d = engine.sampled(engine.to_device(img), mask.offsets)
    m, s, c = (float(d["mean"][y, x].item()), float(d["std"][y, x].item()),
               int(d["count"][y, x].item()))
    return WindowStats(m, s, c)


__all__ = ["WindowStats", "IntegralPair", "build_integral", "mean_std_integral",
           "mean_std_naive", "mean_std_sampled", "window_stats_integral", "window_stats_naive",
           "window_stats_sampled", "window_sums", "make_mask"]
