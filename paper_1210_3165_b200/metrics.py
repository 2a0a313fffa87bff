"""Foreground scoring (recall / precision / F-measure) and (W, k) sweeps on B200.

Drop-in for the reference's metrics.py (/root/reference/pkg/src/docthresh/
metrics.py:1-146): same names, defaults, tie rule, validation messages and
float results.  The pixel work runs in libdocthresh_b200:

* ``evaluate`` -- one ``dtb_confusion`` pass counts TP and the two foreground
  totals and checks both images are bi-level (validation.py:31-40) on the
  device.
* ``sweep`` -- per W, one statistics pass (full window or GS mask), then ONE
  ``dtb_sweep_counts`` pass that scores every k of the grid per pixel with the
  reference's fp64 threshold sequence and keeps two integers per k.  No
  prediction image is materialised, and the whole grid costs one device->host
  read of the counts.

Only the ratios R, P and FM are formed on the host, with the reference's own
expressions (metrics.py:56-60), so the floats are identical.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple, Sequence

import numpy as np

from . import _lib, engine
from .masks import make_mask
from .threshold import BinarizationParams, _validated
from .threshold import apply_global as _apply_global
from .threshold import otsu_threshold

DEFAULT_W_GRID = (11, 15, 21, 31, 41)
DEFAULT_K_GRID = (0.1, 0.2, 0.3, 0.34, 0.4, 0.5)
MAX_K = 64  # DTB_SWEEP_MAX_K; longer k grids are scored in chunks


@dataclass(frozen=True)
class EvalReport:
    """metrics.py:23-39."""

    tp: int
    tn: int
    fp: int
    fn: int
    recall: float
    precision: float
    f_measure: float

    def summary(self) -> str:
        return (
            f"TP = {self.tp}  TN = {self.tn}  FP = {self.fp}  FN = {self.fn}\n"
            f"R = {self.recall * 100:.2f}%\n"
            f"P = {self.precision * 100:.2f}%\n"
            f"FM = {self.f_measure * 100:.2f}%"
        )


def _report(tp: int, pred_fg: int, gt_fg: int, n: int) -> EvalReport:
    """metrics.py:52-61 from the device counts."""
    fp = pred_fg - tp
    fn = gt_fg - tp
    tn = n - tp - fp - fn
    recall = tp / (tp + fn) if tp + fn else 0.0
    precision = tp / (tp + fp) if tp + fp else 0.0
    fm = 2 * recall * precision / (recall + precision) if recall + precision else 0.0
    return EvalReport(tp, tn, fp, fn, recall, precision, fm)


def _device_binary(img):
    """as_gray_image's contract (host side for host inputs), then a device uint8 tensor."""
    img, _ = _validated(img)
    return engine.to_device(img)


def _confusion(pred, gt):
    """-> host list [tp, pred_fg, gt_fg, bad_pred_index, bad_gt_index] (bad = -1 if none)."""
    torch = engine.torch_mod()
    ref = pred if pred is not None else gt
    out = torch.empty(5, dtype=torch.int64, device=ref.device)
    rows, cols = ref.shape
    rc = _lib.lib().dtb_confusion(
        pred.data_ptr() if pred is not None else None, pred.stride(0) if pred is not None else 0,
        gt.data_ptr() if gt is not None else None, gt.stride(0) if gt is not None else 0,
        rows, cols, out.data_ptr(), engine._stream())
    _lib.check(rc, "dtb_confusion")
    return [int(v) for v in out.cpu().tolist()]


def _raise_not_binary(img, index: int) -> None:
    """validation.py:36-40 message for the first (row-major) offending pixel."""
    cols = img.shape[1]
    y, x = divmod(index, cols)
    v = int(img[y, x].item())
    raise ValueError(f"not a bi-level image: pixel ({x}, {y}) has value {v}, expected 0 or 255")


def _check_binary(img) -> int:
    """Validate a device image as bi-level; return its foreground count."""
    c = _confusion(None, img)
    if c[4] != -1:
        _raise_not_binary(img, c[4])
    return c[2]


def evaluate(pred, gt) -> EvalReport:
    """metrics.py:42-61: foreground (0) is the positive class; zero denominators give 0.0."""
    p = _device_binary(pred)
    g = _device_binary(gt)
    if tuple(p.shape) != tuple(g.shape):
        _check_binary(p)
        _check_binary(g)
        raise ValueError(f"shape mismatch: pred {tuple(p.shape)} vs gt {tuple(g.shape)}")
    tp, pf, gf, bad_p, bad_g = _confusion(p, g)
    if bad_p != -1:
        _raise_not_binary(p, bad_p)
    if bad_g != -1:
        _raise_not_binary(g, bad_g)
    return _report(tp, pf, gf, p.numel())


class SweepCell(NamedTuple):
    w: int
    k: float
    f_measure: float


@dataclass(frozen=True)
class SweepResult:
    """Full (W, k) grid of F-measures plus the winning cell (metrics.py:70-80)."""

    cells: tuple
    best: SweepCell

    def to_csv(self) -> str:
        lines = ["w,k,f_measure"]
        lines += [f"{c.w},{c.k:g},{c.f_measure:.6f}" for c in self.cells]
        return "\n".join(lines) + "\n"


def _cell_params(method, engine_name, mask, w, k) -> BinarizationParams:
    """metrics.py:139-146: validate one cell, naming it in the error."""
    kwargs = {"k_sauvola": k} if method == "sauvola" else {"k_niblack": k}
    try:
        return BinarizationParams(
            method=method, engine=engine_name, mask=mask, window=w, **kwargs
        ).validate()
    except ValueError as e:
        raise ValueError(f"sweep cell (W={w}, k={k}): {e}") from None


def _stats(dev, engine_name: str, mask: str, w: int):
    """Per-W (mean, std) device tensors, as metrics.py:119-124 selects them."""
    if engine_name in ("naive", "integral") or mask == "full":
        d = engine.window_stats(dev, w, want=("mean", "std"))
    else:
        m = make_mask(mask, w)
        d = engine.gs(dev, m.structure, m.window)
    return d["mean"], d["std"]


def sweep_counts(dev, gt, mean, std, ks: Sequence[float], method: str, r: float):
    """Device tensor (len(ks), 2) of [pred_fg, TP] for each k (dtb_sweep_counts)."""
    torch = engine.torch_mod()
    rows, cols = dev.shape
    out = torch.empty((len(ks), 2), dtype=torch.int64, device=dev.device)
    for j0 in range(0, len(ks), MAX_K):
        chunk = np.ascontiguousarray(ks[j0:j0 + MAX_K], dtype=np.float64)
        rc = _lib.lib().dtb_sweep_counts(
            dev.data_ptr(), dev.stride(0), gt.data_ptr(), gt.stride(0), rows, cols,
            mean.data_ptr(), std.data_ptr(), mean.stride(0),
            chunk.ctypes.data, len(chunk), engine.METHOD_CODES[method], float(r),
            out[j0:].data_ptr(), engine._stream())
        _lib.check(rc, "dtb_sweep_counts")
    return out


def sweep(
    img,
    gt,
    method: str = "sauvola",
    engine: str = "sampled",
    mask: str = "gs3",
    w_grid: Sequence[int] = DEFAULT_W_GRID,
    k_grid: Sequence[float] = DEFAULT_K_GRID,
    r: float = 128.0,
) -> SweepResult:
    """metrics.py:83-136: score every (W, k); best = max FM, ties to smaller W then k."""
    engine_name = engine
    dev = _device_binary(img)
    g = _device_binary(gt)
    gt_fg = _check_binary(g)
    if tuple(dev.shape) != tuple(g.shape):
        raise ValueError(f"shape mismatch: img {tuple(dev.shape)} vs gt {tuple(g.shape)}")
    if not w_grid or not k_grid:
        raise ValueError("w_grid and k_grid must be non-empty")

    ws = sorted(int(w) for w in w_grid)
    ks = sorted(float(k) for k in k_grid)

    if method == "otsu":
        fm = evaluate(_apply_global(dev, otsu_threshold(dev)), g).f_measure
        cells = tuple(SweepCell(w, k, fm) for w in ws for k in ks)
        return SweepResult(cells, cells[0])

    # metrics.py:116-118 validates each W's cells before computing it; validation has no
    # side effects, so checking the whole grid first raises the same first error.
    for w in ws:
        for k in ks:
            _cell_params(method, engine_name, mask, w, k)
    from . import engine as _eng  # the module (the `engine` argument shadows it)
    torch = _eng.torch_mod()
    counts = torch.empty((len(ws), len(ks), 2), dtype=torch.int64, device=dev.device)
    for i, w in enumerate(ws):
        mean, std = _stats(dev, engine_name, mask, w)
        counts[i] = sweep_counts(dev, g, mean, std, ks, method, r)
        del mean, std
    host = counts.cpu().tolist()
    n = dev.numel()
    cells = []
    best = None
    for i, w in enumerate(ws):
        for j, k in enumerate(ks):
            pf, tp = host[i][j]
            cell = SweepCell(w, k, _report(tp, pf, gt_fg, n).f_measure)
            cells.append(cell)
            if best is None or cell.f_measure > best.f_measure:
                best = cell
    return SweepResult(tuple(cells), best)
