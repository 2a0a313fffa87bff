"""Device-side entry points: torch tensors as buffers, work done by libdocthresh_b200.

Every function here launches a kernel from libdocthresh_b200.so through the
C ABI (include/docthresh_b200.h) on the input tensor's device and that device's
current torch CUDA stream.  Inputs may be host numpy arrays (copied to the
device) or CUDA uint8 tensors (used in place).  Gray images are handed to the
kernels with a 16-byte aligned base and row pitch -- the row staging uses bulk
copies -- so host pages are uploaded into a pitched buffer and a device tensor
with an odd pitch is first copied into one.  There is no CPU path: without a
CUDA device these raise.
"""

from __future__ import annotations

import functools

import numpy as np

from . import _lib

METHOD_CODES = {"sauvola": _lib.DTB_METHOD_SAUVOLA, "niblack": _lib.DTB_METHOD_NIBLACK}

_torch = None
_cuda_ok = False  # set by the first successful availability check (it costs ~3 us a call)


def torch_mod():
    global _torch, _cuda_ok
    if _torch is None:
        import torch
        _torch = torch
    if not _cuda_ok:
        if not _torch.cuda.is_available():
            raise RuntimeError("paper_1210_3165_b200 needs a CUDA device (there is no CPU fallback)")
        _cuda_ok = True
    return _torch


def is_device_tensor(x) -> bool:
    if _torch is None and type(x).__module__.split(".")[0] != "torch":
        return False
    import torch
    return isinstance(x, torch.Tensor) and x.is_cuda


def is_host_tensor(x) -> bool:
    if _torch is None and type(x).__module__.split(".")[0] != "torch":
        return False
    import torch
    return isinstance(x, torch.Tensor) and not x.is_cuda


def _stream(stream=None) -> int:
    """The given stream, else the current stream of the current device (the wrapped entry
    points below make the input's device current)."""
    torch = torch_mod()
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _on_input_device(fn):
    """Run fn with the device of its first CUDA tensor argument current, so its launches (and
    the library's per-device launch state) use that device, not whichever device is current."""
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        for x in list(args) + list(kwargs.values()):
            if is_device_tensor(x):
                import torch
                with torch.cuda.device(x.device):
                    return fn(*args, **kwargs)
        return fn(*args, **kwargs)
    return wrapper


def _pitched(t):
    """A 2-D uint8 device image with a 16-byte aligned base and pitch (a view into a pitched
    copy when t's layout is not)."""
    if t.dim() == 2 and (t.data_ptr() % 16 or t.stride(0) % 16):
        torch = torch_mod()
        h, w = t.shape
        buf = torch.empty((h, -(-w // 16) * 16), dtype=torch.uint8, device=t.device)
        v = buf[:, :w]
        v.copy_(t)
        return v
    return t


def _check_device_image(t, ndim: int, what: str):
    torch = torch_mod()
    if t.dtype != torch.uint8:
        raise ValueError(f"{what}: expected a uint8 CUDA tensor, got {t.dtype}")
    if t.dim() != ndim:
        raise ValueError(f"expected a {ndim}-D image, got shape {tuple(t.shape)}")
    if t.numel() == 0:
        raise ValueError("image is empty")
    if t.stride(-1) != 1 or (ndim == 3 and t.stride(1) != 3):
        t = t.contiguous()
    return _pitched(t)


def to_device(arr, ndim: int = 2, what: str = "image"):
    """Host numpy (already validated) or CUDA tensor -> CUDA uint8 tensor with unit inner stride."""
    torch = torch_mod()
    if is_device_tensor(arr):
        return _check_device_image(arr, ndim, what)
    if not is_host_tensor(arr):
        arr = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.uint8))
    arr = arr.contiguous()
    if ndim == 2 and arr.shape[1] % 16:
        # upload into a pitched buffer (one 2-D copy): every width reaches the fast kernels
        h, w = arr.shape
        buf = torch.empty((h, -(-w // 16) * 16), dtype=torch.uint8, device="cuda")
        v = buf[:, :w]
        v.copy_(arr, non_blocking=arr.is_pinned())
        return v
    return arr.to("cuda", non_blocking=arr.is_pinned())


@_on_input_device
def binarize(gray, win: int, method: str, k: float, r: float, want_tmap: bool = True,
             stream=None, out=None, tmap_out=None):
    """Whole-image binarize -> (binary uint8 tensor, tmap float64 tensor or None).  ``out`` /
    ``tmap_out``: caller-owned result buffers (steady-state callers reuse them; ``tmap_out`` is
    an (h, w) float64 view, ideally of a buffer whose row pitch is a multiple of 16 bytes)."""
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    if out is None:
        out = torch.empty((h, w), dtype=torch.uint8, device=g.device)
    # a 16-byte row pitch lets the fast kernel's paired fp64 stores take the map
    tmap = None
    if want_tmap:
        tmap = tmap_out if tmap_out is not None else \
            torch.empty((h, w + (w & 1)), dtype=torch.float64, device=g.device)[:, :w]
    rc = _lib.lib().dtb_binarize(
        g.data_ptr(), g.stride(0), h, w, 0, h, 0, h, out.data_ptr(), out.stride(0),
        tmap.data_ptr() if tmap is not None else None, (tmap.stride(0) * 8) if tmap is not None else 0,
        int(win), METHOD_CODES[method], float(k), float(r), _stream(stream))
    _lib.check(rc, "dtb_binarize")
    return out, tmap


_side_streams = {}


def _streams_for(dev):
    """(copy-in, copy-out) side streams for a device, created once."""
    torch = torch_mod()
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _side_streams:
        with torch.cuda.device(key):
            _side_streams[key] = (torch.cuda.Stream(), torch.cuda.Stream())
    return _side_streams[key]


@_on_input_device
def host_streamed(host, band_fn, rad: int, out=None, chunk_rows: int | None = None):
    """Host page -> host binary with H2D, compute and D2H overlapped by row chunks.

    ``host`` is a (rows, cols) uint8 CPU tensor (pinned for real overlap).  Row chunk i is
    copied in on one side stream, computed on the current stream as soon as the input rows
    its windows reach (chunk end + rad) have landed, and copied out on another side stream
    while later chunks compute -- PCIe's two directions run concurrently instead of
    back to back.  ``band_fn(dev_in, y0, y1, dev_out_rows)`` computes output rows [y0, y1)
    from the full-page device buffer.  Returns the host result (synchronised).
    """
    torch = torch_mod()
    h, w = host.shape
    if out is None:
        out = torch.empty((h, w), dtype=torch.uint8, pin_memory=host.is_pinned())
    dev = torch.device("cuda", torch.cuda.current_device())
    cur = torch.cuda.current_stream()
    s_in, s_out = _streams_for(dev)
    pitch = -(-w // 16) * 16  # 16-byte pitch: the fast kernels stage rows with bulk copies
    dev_in = torch.empty((h, pitch), dtype=torch.uint8, device=dev)[:, :w]
    dev_out = torch.empty((h, pitch), dtype=torch.uint8, device=dev)[:, :w]
    if chunk_rows is None:
        import os
        n = int(os.environ.get("DTB_STREAM_CHUNKS", "16"))
        chunk_rows = max(256, -(-h // n))
    bounds = [(a, min(a + chunk_rows, h)) for a in range(0, h, chunk_rows)]
    s_in.wait_stream(cur)
    s_out.wait_stream(cur)
    ev_in = []
    with torch.cuda.stream(s_in):
        for a, b in bounds:
            dev_in[a:b].copy_(host[a:b], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s_in)
            ev_in.append(e)
    for a, b in bounds:
        need = min(b + rad, h)
        cur.wait_event(ev_in[(need - 1) // chunk_rows])
        band_fn(dev_in, a, b, dev_out[a:b])
        e = torch.cuda.Event()
        e.record(cur)
        s_out.wait_event(e)
        with torch.cuda.stream(s_out):
            out[a:b].copy_(dev_out[a:b], non_blocking=True)
    dev_in.record_stream(s_in)
    dev_out.record_stream(s_out)
    cur.wait_stream(s_out)
    cur.synchronize()
    return out


@_on_input_device
def binarize_band(buf, row0_global: int, rows_global: int, out_begin: int, out_end: int,
                  win: int, method: str, k: float, r: float, out=None, stream=None):
    """Binarize global rows [out_begin, out_end) from a buffer holding rows [row0, row0+len)."""
    torch = torch_mod()
    g = to_device(buf)
    in_rows, w = g.shape
    if out is None:
        out = torch.empty((out_end - out_begin, w), dtype=torch.uint8, device=g.device)
    rc = _lib.lib().dtb_binarize(
        g.data_ptr(), g.stride(0), in_rows, w, int(row0_global), int(rows_global), int(out_begin),
        int(out_end), out.data_ptr(), out.stride(0), None, 0, int(win), METHOD_CODES[method],
        float(k), float(r), _stream(stream))
    _lib.check(rc, "dtb_binarize")
    return out


def binarize_segments(segments, row0_global: int, rows_global: int, out_begin: int,
                      out_end: int, win: int, method: str, k: float, r: float, out=None,
                      stream=None):
    """Binarize global rows [out_begin, out_end) whose input rows are split over up to three
    buffers (dtb_binarize_segments).  ``segments`` = [(ptr, pitch, rows, cols), ...] with raw
    device pointers (e.g. a neighbour GPU's band mapped through CUDA IPC) stacked downward
    from global row ``row0_global``.  Returns the (out_end - out_begin, cols) binary tensor."""
    import ctypes
    torch = torch_mod()
    n = len(segments)
    cols = segments[0][3]
    ptrs = (ctypes.c_void_p * 3)(*[sg[0] for sg in segments] + [None] * (3 - n))
    pitches = (ctypes.c_int64 * 3)(*[sg[1] for sg in segments] + [0] * (3 - n))
    nrows = (ctypes.c_int32 * 3)(*[sg[2] for sg in segments] + [0] * (3 - n))
    if out is None:
        out = torch.empty((out_end - out_begin, cols), dtype=torch.uint8, device="cuda")
    rc = _lib.lib().dtb_binarize_segments(
        ptrs, pitches, nrows, n, int(row0_global), int(rows_global), int(cols), int(out_begin),
        int(out_end), out.data_ptr(), out.stride(0), int(win), METHOD_CODES[method], float(k),
        float(r), _stream(stream))
    _lib.check(rc, "dtb_binarize_segments")
    return out


def ipc_export(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t.data_ptr() in it)."""
    import ctypes
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_int64(0)
    _lib.check(_lib.lib().dtb_ipc_export(t.data_ptr(), h, ctypes.byref(off)), "dtb_ipc_export")
    return bytes(h), int(off.value)


def ipc_import(handle: bytes) -> int:
    """Map a peer process's allocation; returns its base device address (close with ipc_close)."""
    import ctypes
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    base = ctypes.c_void_p(0)
    _lib.check(_lib.lib().dtb_ipc_import(h, ctypes.byref(base)), "dtb_ipc_import")
    return int(base.value)


def ipc_close(base: int) -> None:
    _lib.check(_lib.lib().dtb_ipc_close(base), "dtb_ipc_close")


@_on_input_device
def binarize_batch(stack, win: int, method: str, k: float, r: float, out=None, stream=None):
    """(N, H, W) uint8 CUDA stack -> (N, H, W) binary, one launch."""
    torch = torch_mod()
    s = stack if is_device_tensor(stack) else torch.from_numpy(np.ascontiguousarray(stack)).to("cuda")
    s = s.contiguous()
    n, h, w = s.shape
    if out is None:
        out = torch.empty_like(s)
    rc = _lib.lib().dtb_binarize_batch(
        s.data_ptr(), s.stride(0), n, h, w, out.data_ptr(), out.stride(0), int(win),
        METHOD_CODES[method], float(k), float(r), _stream(stream))
    _lib.check(rc, "dtb_binarize_batch")
    return out


@_on_input_device
def window_stats(gray, win: int, want=("mean", "std", "count"), stream=None):
    """dict of requested (rows, cols) device tensors among S, Q, count, mean, std."""
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    dt = {"S": torch.int64, "Q": torch.int64, "count": torch.int32, "mean": torch.float64,
          "std": torch.float64}
    outs = {k: torch.empty((h, w), dtype=dt[k], device=g.device) for k in want}
    ptr = lambda k: outs[k].data_ptr() if k in outs else None  # noqa: E731
    rc = _lib.lib().dtb_window_stats(g.data_ptr(), g.stride(0), h, w, int(win), ptr("S"),
                                     ptr("Q"), ptr("count"), ptr("mean"), ptr("std"),
                                     _stream(stream))
    _lib.check(rc, "dtb_window_stats")
    return outs


@_on_input_device
def sampled(gray, offsets, method: str | None = None, k: float = 0.0, r: float = 128.0,
            want_tmap: bool = True, stream=None):
    """Mask-restricted statistics (stats.py:133-163) or binarization with them.

    method None -> dict(mean, std, count); else (binary, tmap or None).
    """
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32).reshape(-1, 2))
    dev_offs = torch.from_numpy(offs).to("cuda")
    L = _lib.lib()
    if method is None:
        mean = torch.empty((h, w), dtype=torch.float64, device=g.device)
        std = torch.empty_like(mean)
        cnt = torch.empty((h, w), dtype=torch.int32, device=g.device)
        rc = L.dtb_sampled_stats(g.data_ptr(), g.stride(0), h, w, dev_offs.data_ptr(),
                                 len(offs), mean.data_ptr(), std.data_ptr(), cnt.data_ptr(),
                                 None, 0, 0, 0.0, 1.0, _stream(stream))
        _lib.check(rc, "dtb_sampled_stats")
        return {"mean": mean, "std": std, "count": cnt}
    out = torch.empty((h, w), dtype=torch.uint8, device=g.device)
    tmap = torch.empty((h, w), dtype=torch.float64, device=g.device) if want_tmap else None
    rc = L.dtb_sampled_stats(g.data_ptr(), g.stride(0), h, w, dev_offs.data_ptr(), len(offs),
                             None, None, None, out.data_ptr(),
                             tmap.data_ptr() if tmap is not None else None,
                             METHOD_CODES[method], float(k), float(r), _stream(stream))
    _lib.check(rc, "dtb_sampled_stats")
    return out, tmap


GS_CODES = {"gs1": 1, "gs2": 2, "gs3": 3, "gs4": 4, "gs5": 5, "gs6": 6}


@_on_input_device
def gs(gray, structure: str, win: int, method: str | None = None, k: float = 0.0,
       r: float = 128.0, want_tmap: bool = True, stream=None):
    """GS-mask statistics / binarization in O(1) per pixel (dtb_gs_stats).

    Same results and return convention as ``sampled`` with make_mask(structure, win)'s
    offsets.  Windows whose tile does not fit in shared memory go to ``sampled``.
    """
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    L = _lib.lib()
    code = GS_CODES[structure]
    if method is None:
        mean = torch.empty((h, w), dtype=torch.float64, device=g.device)
        std = torch.empty_like(mean)
        cnt = torch.empty((h, w), dtype=torch.int32, device=g.device)
        rc = L.dtb_gs_stats(g.data_ptr(), g.stride(0), h, w, code, int(win), mean.data_ptr(),
                            std.data_ptr(), cnt.data_ptr(), None, 0, None, 0, 0.0, 1.0,
                            _stream(stream))
        res = {"mean": mean, "std": std, "count": cnt}
    else:
        out = torch.empty((h, w), dtype=torch.uint8, device=g.device)
        tmap = torch.empty((h, w), dtype=torch.float64, device=g.device) if want_tmap else None
        rc = L.dtb_gs_stats(g.data_ptr(), g.stride(0), h, w, code, int(win), None, None, None,
                            out.data_ptr(), out.stride(0),
                            tmap.data_ptr() if tmap is not None else None,
                            METHOD_CODES[method], float(k), float(r), _stream(stream))
        res = (out, tmap)
    if rc == _lib.DTB_E_UNSUPPORTED:
        from .masks import make_mask
        return sampled(g, make_mask(structure, win).offsets, method, k, r, want_tmap, stream)
    _lib.check(rc, "dtb_gs_stats")
    return res


@_on_input_device
def gs_band(buf, row0_global: int, rows_global: int, out_begin: int, out_end: int,
            structure: str, win: int, method: str, k: float, r: float, out=None, stream=None):
    """GS-mask binarization of global rows [out_begin, out_end) from a row-band buffer
    (dtb_gs_band); windows clip at the page's global borders."""
    torch = torch_mod()
    g = to_device(buf)
    in_rows, w = g.shape
    if out is None:
        out = torch.empty((out_end - out_begin, w), dtype=torch.uint8, device=g.device)
    rc = _lib.lib().dtb_gs_band(g.data_ptr(), g.stride(0), in_rows, w, int(row0_global),
                                int(rows_global), int(out_begin), int(out_end),
                                GS_CODES[structure], int(win), out.data_ptr(), out.stride(0),
                                METHOD_CODES[method], float(k), float(r), _stream(stream))
    if rc == _lib.DTB_E_UNSUPPORTED and (row0_global, in_rows) == (0, rows_global):
        # window too wide for the tiled kernel: the offset-gather kernel on the whole page
        from .masks import make_mask
        full, _ = sampled(g, make_mask(structure, win).offsets, method, k, r, want_tmap=False)
        out.copy_(full[out_begin:out_end])
        return out
    _lib.check(rc, "dtb_gs_band")
    return out


@_on_input_device
def to_gray(rgb, stream=None):
    torch = torch_mod()
    t = to_device(rgb, ndim=3, what="rgb")
    h, w, _ = t.shape
    out = torch.empty((h, w), dtype=torch.uint8, device=t.device)
    rc = _lib.lib().dtb_to_gray(t.data_ptr(), t.stride(0), out.data_ptr(), out.stride(0), h, w,
                                _stream(stream))
    _lib.check(rc, "dtb_to_gray")
    return out


@_on_input_device
def rgb_binarize(rgb, win: int, method: str, k: float, r: float, want_gray: bool = False,
                 stream=None):
    torch = torch_mod()
    t = to_device(rgb, ndim=3, what="rgb")
    h, w, _ = t.shape
    out = torch.empty((h, w), dtype=torch.uint8, device=t.device)
    gray = torch.empty((h, w), dtype=torch.uint8, device=t.device)
    rc = _lib.lib().dtb_rgb_binarize(t.data_ptr(), t.stride(0), h, w, out.data_ptr(),
                                     out.stride(0), gray.data_ptr(), gray.stride(0), int(win),
                                     METHOD_CODES[method], float(k), float(r), _stream(stream))
    _lib.check(rc, "dtb_rgb_binarize")
    return (out, gray) if want_gray else out


@_on_input_device
def histogram(gray, stream=None):
    """256-bin histogram (uint64) of a gray image, on the device."""
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    hist = torch.zeros(256, dtype=torch.int64, device=g.device)
    rc = _lib.lib().dtb_histogram(g.data_ptr(), g.stride(0), h, w, hist.data_ptr(),
                                  _stream(stream))
    _lib.check(rc, "dtb_histogram")
    return hist


@_on_input_device
def apply_global(gray, t: int, stream=None):
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    out = torch.empty((h, w), dtype=torch.uint8, device=g.device)
    rc = _lib.lib().dtb_apply_global(g.data_ptr(), g.stride(0), h, w, int(t), out.data_ptr(),
                                     out.stride(0), _stream(stream))
    _lib.check(rc, "dtb_apply_global")
    return out


@_on_input_device
def otsu(gray, stream=None):
    """Device int32 tensor [1] holding the Otsu T (dtb_otsu); no host synchronisation."""
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    hist = torch.empty(256, dtype=torch.int64, device=g.device)
    t = torch.empty(1, dtype=torch.int32, device=g.device)
    rc = _lib.lib().dtb_otsu(g.data_ptr(), g.stride(0), h, w, hist.data_ptr(), t.data_ptr(),
                             _stream(stream))
    _lib.check(rc, "dtb_otsu")
    return t


@_on_input_device
def apply_global_dev(gray, t_dev, want_tmap: bool = False, stream=None):
    """(binary, tmap or None) with T from a device int32 tensor (dtb_apply_global_dev)."""
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    out = torch.empty((h, w), dtype=torch.uint8, device=g.device)
    tmap = torch.empty((h, w), dtype=torch.float64, device=g.device) if want_tmap else None
    rc = _lib.lib().dtb_apply_global_dev(g.data_ptr(), g.stride(0), h, w, t_dev.data_ptr(),
                                         out.data_ptr(), out.stride(0),
                                         tmap.data_ptr() if tmap is not None else None,
                                         _stream(stream))
    _lib.check(rc, "dtb_apply_global_dev")
    return out, tmap


@_on_input_device
def integral_tables(gray, stream=None):
    """(H+1, W+1) int64 summed-area tables of f and f^2 (stats.py:82-91)."""
    torch = torch_mod()
    g = to_device(gray)
    h, w = g.shape
    s = torch.empty((h + 1, w + 1), dtype=torch.int64, device=g.device)
    sq = torch.empty_like(s)
    rc = _lib.lib().dtb_integral_tables(g.data_ptr(), g.stride(0), h, w, s.data_ptr(),
                                        sq.data_ptr(), _stream(stream))
    _lib.check(rc, "dtb_integral_tables")
    return s, sq
