"""Global (Otsu) and locally adaptive (Niblack, Sauvola) binarization on B200.

Drop-in for the reference's threshold.py (/root/reference/pkg/src/docthresh/
threshold.py:1-148): same names, defaults, validation messages and outputs
(0 = ink, 255 = background, strict ``<``, real-valued fp64 thresholds), with
the per-pixel work done by libdocthresh_b200 kernels on the current CUDA
device.  Engines "naive" and "integral" (and "sampled" with mask "full") are
the same exact full-window computation in the reference (stats.py:14-17), so
all three map to the O(1)-per-pixel sliding-sum kernel here; "sampled" with a
GS mask runs the mask-restricted kernel.

Inputs: a host array-like (validated like the reference, result returned as
numpy) or a CUDA uint8 tensor (result stays on the device as torch tensors).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine
from .masks import STRUCTURES, make_mask
from .validation import as_gray_image, check_window

METHODS = ("otsu", "niblack", "sauvola")
ENGINES = ("naive", "integral", "sampled")


@dataclass(frozen=True)
class BinarizationParams:
    """threshold.py:23-52: method/engine selection plus the knobs they read."""

    method: str = "sauvola"
    engine: str = "sampled"
    mask: str = "gs3"
    window: int = 21
    k_sauvola: float = 0.34
    k_niblack: float = -0.2
    r: float = 128.0

    def validate(self) -> "BinarizationParams":
        if self.method not in METHODS:
            raise ValueError(f"method: expected one of {METHODS}, got {self.method!r}")
        if self.engine not in ENGINES:
            raise ValueError(f"engine: expected one of {ENGINES}, got {self.engine!r}")
        check_window(self.window)
        if not self.k_sauvola > 0:
            raise ValueError(f"k_sauvola: must be > 0, got {self.k_sauvola}")
        if not self.r > 0:
            raise ValueError(f"r: must be > 0, got {self.r}")
        if self.engine == "sampled" and self.mask not in STRUCTURES:
            raise ValueError(f"mask: expected one of {STRUCTURES}, got {self.mask!r}")
        return self

    @property
    def k(self) -> float:
        return self.k_sauvola if self.method == "sauvola" else self.k_niblack

    @property
    def full_window(self) -> bool:
        return self.engine in ("naive", "integral") or self.mask == "full"


def _validated(img):
    """Host inputs validated like validation.py:8-28 (before any device work)."""
    if engine.is_host_tensor(img):
        if img.dtype != engine.torch_mod().uint8 or img.dim() != 2 or img.numel() == 0:
            raise ValueError(f"expected a non-empty 2-D uint8 image, got {tuple(img.shape)} "
                             f"{img.dtype}")
        return img, True
    if engine.is_device_tensor(img):
        if img.dim() != 2:
            raise ValueError(f"expected a 2-D grayscale image, got shape {tuple(img.shape)}")
        if img.numel() == 0:
            raise ValueError("image is empty")
        return img, False
    return as_gray_image(img), True


def _prepare(img):
    """-> (device tensor, host_out flag)."""
    img, host = _validated(img)
    return engine.to_device(img), host


def _host(t, like=None, out=None):
    """Device result -> host: numpy for array-like inputs, (pinned) torch for torch inputs."""
    if t is None:
        return None
    if engine.is_host_tensor(like):
        if out is None:
            out = engine.torch_mod().empty(tuple(t.shape), dtype=t.dtype,
                                           pin_memory=like.is_pinned())
        out.copy_(t, non_blocking=True)
        engine.torch_mod().cuda.current_stream().synchronize()
        return out
    return t.cpu().numpy()


def otsu_threshold(img) -> int:
    """threshold.py:55-88: histogram and the exact 256-step scan on the device (dtb_otsu)."""
    dev, _ = _prepare(img)
    return int(engine.otsu(dev).item())


def apply_global(img, t: int):
    """threshold.py:91-96: pixel < t -> 0, else 255."""
    img, host = _validated(img)
    if not isinstance(t, (int, np.integer)) or not 0 <= int(t) <= 255:
        raise ValueError(f"threshold: expected an integer in [0, 255], got {t!r}")
    dev = engine.to_device(img)
    out = engine.apply_global(dev, int(t))
    return _host(out) if host else out


def sauvola_threshold_at(stats, k: float, r: float) -> float:
    """threshold.py:99-106: t = m*(1 + k*(s/r - 1)) for one pixel's statistics."""
    if not k > 0:
        raise ValueError(f"k: must be > 0, got {k}")
    if not r > 0:
        raise ValueError(f"r: must be > 0, got {r}")
    return stats.mean * (1.0 + k * (stats.std / r - 1.0))


def niblack_threshold_at(stats, k: float) -> float:
    """threshold.py:109-110: t = m + k*s."""
    return stats.mean + k * stats.std


def binarize(img, params: BinarizationParams = BinarizationParams(), *, return_tmap: bool = True,
             out=None):
    """threshold.py:121-148.  Returns (binary uint8 {0,255}, tmap float64).

    ``return_tmap=False`` skips the 8 B/px fp64 threshold map (it is then None);
    the binary output is unchanged.  This is the fast path: 2 B/px of HBM traffic.
    Host torch tensors (ideally pinned) are accepted too: the copy in is
    asynchronous and ``out`` may name a preallocated (pinned) host tensor.
    """
    src = img
    img, host = _validated(img)
    params.validate()
    if (engine.is_host_tensor(src) and params.method != "otsu" and not return_tmap
            and src.is_contiguous()):
        # pinned host page: H2D / compute / D2H overlapped by row chunks (engine.host_streamed)
        if params.full_window:
            def band(dev_in, y0, y1, dev_out):
                engine.binarize_band(dev_in, 0, dev_in.shape[0], y0, y1, params.window,
                                     params.method, params.k, params.r, out=dev_out)
        else:
            structure = make_mask(params.mask, params.window).structure

            def band(dev_in, y0, y1, dev_out):
                engine.gs_band(dev_in, 0, dev_in.shape[0], y0, y1, structure, params.window,
                               params.method, params.k, params.r, out=dev_out)
        return engine.host_streamed(src, band, params.window // 2, out=out), None
    dev = engine.to_device(img)
    if params.method == "otsu":
        # histogram -> scan -> apply, stream-ordered with T kept on the device
        binary, tmap = engine.apply_global_dev(dev, engine.otsu(dev), want_tmap=return_tmap)
    elif params.full_window:
        binary, tmap = engine.binarize(dev, params.window, params.method, params.k, params.r,
                                       want_tmap=return_tmap)
    else:
        mask = make_mask(params.mask, params.window)
        binary, tmap = engine.gs(dev, mask.structure, mask.window, params.method, params.k,
                                 params.r, want_tmap=return_tmap)
    if host:
        return _host(binary, src, out), _host(tmap, src)
    return binary, tmap
