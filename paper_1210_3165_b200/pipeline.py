"""PNM pages through the GPU, I/O overlapped with compute.

The reference's command line (cli.py:30-42, 85-93) reads a whole PNM file into
bytes, decodes it with read_pnm (pnm.py:78-133), converts P6 to gray, binarizes,
and writes a P5 file with write_pnm (pnm.py:136-150).  Here the same page-level
contract runs as a two-slot software pipeline:

* the header is parsed on the host (a few bytes; same checks and messages as
  read_pnm), then the binary payload is read by ``readinto`` straight into a
  pinned host slot -- no intermediate bytes object, no numpy copy;
* the slot is copied to the device on a copy stream; to_gray (P6) and the
  binarization run on a compute stream; the result comes back on a second
  copy stream into a pinned output slot;
* while page i is on the GPU the host reads page i+1 and writes page i-1.

ASCII pages (P2/P3) go through read_pnm's token parser first (the reference's
format semantics) and then take the same device path.

Outputs are byte-identical to ``write_pnm(binarize(read_gray(path), params)[0])``.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import engine
from .masks import make_mask
from .pnm import PnmError, parse_header, read_pnm
from .threshold import BinarizationParams

_HEAD_CHUNK = 1 << 16


@dataclass
class PipelineStats:
    pages: int = 0
    pixels: int = 0
    bytes_in: int = 0
    bytes_out: int = 0


class _Slot:
    """Pinned staging for one in-flight page plus the events that guard its reuse."""

    def __init__(self, torch):
        self.torch = torch
        self.inp = None   # pinned uint8 payload buffer
        self.out = None   # pinned uint8 result buffer
        self.done = None  # event: D2H of this slot's result finished
        self.pending = None  # (out_path, rows, cols) awaiting write-back

    def ensure(self, n_in: int, n_out: int):
        t = self.torch
        if self.inp is None or self.inp.numel() < n_in:
            self.inp = t.empty(n_in, dtype=t.uint8, pin_memory=True)
        if self.out is None or self.out.numel() < n_out:
            self.out = t.empty(n_out, dtype=t.uint8, pin_memory=True)


def _read_page(path: str, slot: _Slot, torch):
    """Header on the host, payload straight into the pinned slot.  -> (rows, cols, channels)."""
    with open(path, "rb") as fh:
        size = os.fstat(fh.fileno()).st_size
        head = fh.read(min(size, _HEAD_CHUNK))
        try:
            magic, width, height, ch, hd = parse_header(head)
            ok = magic in (b"P5", b"P6")
        except PnmError:
            if len(head) == size:
                raise
            ok = False
        if not ok:
            # ASCII formats, or a header longer than the first chunk: the reference codec
            fh.seek(0)
            img = read_pnm(fh.read())
            h, w = img.shape[:2]
            ch = 3 if img.ndim == 3 else 1
            slot.ensure(img.size, h * w)
            slot.inp[: img.size].numpy()[:] = img.reshape(-1)
            return h, w, ch
        start = hd.pos + 1
        count = width * height * ch
        slot.ensure(count, width * height)
        fh.seek(start)
        got = fh.readinto(memoryview(slot.inp.numpy())[:count])
        if got < count:
            raise PnmError(f"truncated payload at byte {start + got}: "
                           f"expected {count} bytes, got {got}")
        return height, width, ch


def _compute(params: BinarizationParams, dev_in, rows, cols, ch, torch):
    """Device page -> device binary (the engines threshold.binarize dispatches to)."""
    if ch == 3:
        gray = engine.to_gray(dev_in.view(rows, cols, 3))
    else:
        gray = dev_in.view(rows, cols)
    if params.method == "otsu":
        return engine.apply_global_dev(gray, engine.otsu(gray))[0]
    if params.full_window:
        return engine.binarize(gray, params.window, params.method, params.k, params.r,
                               want_tmap=False)[0]
    m = make_mask(params.mask, params.window)
    return engine.gs(gray, m.structure, m.window, params.method, params.k, params.r,
                     want_tmap=False)[0]


def binarize_files(pairs: Iterable[Sequence[str]],
                   params: BinarizationParams = BinarizationParams(),
                   slots: int = 2) -> PipelineStats:
    """Binarize (input PNM, output PGM) path pairs; returns byte/pixel counts.

    Equivalent, page for page, to the reference CLI's ``binarize IN OUT`` with these
    params (cli.py:85-93, without --threshold-map).
    """
    params.validate()
    torch = engine.torch_mod()
    dev = torch.device("cuda", torch.cuda.current_device())
    s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ring = [_Slot(torch) for _ in range(max(1, slots))]
    stats = PipelineStats()

    def drain(slot: _Slot):
        if slot.pending is None:
            return
        path, rows, cols = slot.pending
        slot.done.synchronize()
        n = rows * cols
        with open(path, "wb") as fh:
            fh.write(f"P5\n{cols} {rows}\n255\n".encode("ascii"))
            fh.write(memoryview(slot.out.numpy())[:n])
        stats.bytes_out += n
        slot.pending = None

    for i, (src, dst) in enumerate(pairs):
        slot = ring[i % len(ring)]
        drain(slot)  # this slot's previous page: written back before its buffers are reused
        rows, cols, ch = _read_page(src, slot, torch)
        n_in = rows * cols * ch
        with torch.cuda.stream(s_in):
            d_in = slot.inp[:n_in].to(dev, non_blocking=True)
            e_in = torch.cuda.Event()
            e_in.record(s_in)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(e_in)
            d_in.record_stream(s_cmp)
            binary = _compute(params, d_in, rows, cols, ch, torch)
            e_cmp = torch.cuda.Event()
            e_cmp.record(s_cmp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(e_cmp)
            binary.record_stream(s_out)
            slot.out[: rows * cols].view(rows, cols).copy_(binary, non_blocking=True)
            slot.done = torch.cuda.Event()
            slot.done.record(s_out)
        slot.pending = (dst, rows, cols)
        stats.pages += 1
        stats.pixels += rows * cols
        stats.bytes_in += n_in
    for slot in ring:
        drain(slot)
    return stats


def main(argv=None) -> int:
    """python -m paper_1210_3165_b200.pipeline IN OUT [IN OUT ...] (reference CLI defaults)."""
    import sys
    args = list(sys.argv[1:] if argv is None else argv)
    if not args or len(args) % 2:
        sys.stderr.write("usage: python -m paper_1210_3165_b200.pipeline IN OUT [IN OUT ...]\n")
        return 1
    try:
        st = binarize_files(list(zip(args[0::2], args[1::2])))
    except (OSError, PnmError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    print(f"{st.pages} pages, {st.pixels} px")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
