"""Sampling masks (geometric structures GS-1..GS-6 of the paper, plus FULL).

Same contract as the reference's masks.py:25-129 (offset sets, row-major order
with dy outer / dx inner, (0, 0) always present).  Pure host geometry: the
offsets parameterise the GPU sampled engine (dtb_sampled_stats); "full" is the
full window handled by the O(1)-per-pixel sliding kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .validation import check_window

STRUCTURES = ("gs1", "gs2", "gs3", "gs4", "gs5", "gs6", "full")


def _member(name: str, dx: int, dy: int, r: int) -> bool:
    on_row, on_col = dy == 0, dx == 0
    on_diag = abs(dx) == abs(dy)
    on_ring = max(abs(dx), abs(dy)) == r
    if name == "gs1":   # axis-aligned cross, 2W-1 px
        return on_row or on_col
    if name == "gs2":   # both diagonals, 2W-1 px
        return on_diag
    if name == "gs3":   # 8-ray star = cross + X, 4W-3 px
        return on_row or on_col or on_diag
    if name == "gs4":   # centre row + diagonals, 3W-2 px
        return on_row or on_diag
    if name == "gs5":   # perimeter ring + centre, 4W-3 px
        return on_ring or (on_row and on_col)
    if name == "gs6":   # cross + ring, 6W-9 px
        return on_row or on_col or on_ring
    return True         # full window, W^2 px


def _canonical(structure) -> str:
    name = str(structure).lower().replace("-", "").replace("_", "")
    if name not in STRUCTURES:
        raise ValueError(f"unknown mask structure {structure!r}; expected one of "
                         f"{', '.join(STRUCTURES)}")
    return name


@dataclass(frozen=True)
class SamplingMask:
    """Immutable window-relative offsets (dx, dy), row-major, (0, 0) included."""

    structure: str
    window: int
    offsets: tuple = field(repr=False)

    def __len__(self) -> int:
        return len(self.offsets)


def make_mask(structure: str, w: int) -> SamplingMask:
    name = _canonical(structure)
    w = check_window(w)
    r = w // 2
    offs = tuple((dx, dy) for dy in range(-r, r + 1) for dx in range(-r, r + 1)
                 if _member(name, dx, dy, r))
    return SamplingMask(structure=name, window=w, offsets=offs)


def mask_size(structure: str, w: int) -> int:
    return len(make_mask(structure, w))


def mask_to_ascii(mask: SamplingMask) -> str:
    r = mask.window // 2
    cells = set(mask.offsets)
    return "\n".join("".join("#" if (dx, dy) in cells else "." for dx in range(-r, r + 1))
                     for dy in range(-r, r + 1))
