"""Image conventions and pixel primitives — drop-in for pnprestore/image.py
(validate_image 32-41, constraint sets + project 48-90, pad_symmetric /
integral_image / box_sum 97-143, psnr 146-157).  Projection, PSNR, padding
and summed-area tables run on the GPU (the last two in float64, bitwise equal
to the reference); PGM / PFM file I/O (image.py:169-280) is in imageio.py."""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _arrays as A
from . import _lib as L


class Unconstrained:
    """No constraint; projection is the identity."""

    def __repr__(self) -> str:
        return "Unconstrained()"


class NonNegative:
    """The nonnegative orthant."""

    def __repr__(self) -> str:
        return "NonNegative()"


@dataclass(frozen=True)
class Box:
    """Per-pixel interval constraint [lo, hi]."""

    lo: float
    hi: float

    def __post_init__(self) -> None:
        if not self.lo < self.hi:
            raise ValueError(f"Box requires lo < hi, got [{self.lo}, {self.hi}]")


Constraint = Unconstrained | NonNegative | Box

UNCONSTRAINED = Unconstrained()
NON_NEGATIVE = NonNegative()
UNIT_BOX = Box(0.0, 1.0)


def bounds(constraint) -> tuple[float, float]:
    if isinstance(constraint, Unconstrained):
        return -math.inf, math.inf
    if isinstance(constraint, NonNegative):
        return 0.0, math.inf
    if isinstance(constraint, Box):
        return float(constraint.lo), float(constraint.hi)
    raise TypeError(f"unknown constraint {constraint!r}")


def validate_image(img, name: str = "image"):
    """2-D, non-empty, finite; numpy in -> float64 numpy out, tensors kept."""
    a, kind = A.validate(img, name)
    return a if kind == A.NUMPY else a


def project(img, constraint):
    """Euclidean projection onto the constraint set (per-pixel clamp, GPU)."""
    lo, hi = bounds(constraint)
    img, kind = A.validate(img, batch_ok=True)
    t = A.to_device(img)
    out = torch.empty_like(t)
    L.call("pnp_project", L.context(t.device.index), L.ptr(t), L.ptr(out), t.numel(), lo, hi)
    return A.from_device(out, kind)


def pad_symmetric(img, margin: int):
    """Half-sample mirror pad (i -> -i-1), margin <= min extent (image.py:97-113)."""
    img, kind = A.validate(img)
    if margin < 0:
        raise ValueError(f"margin must be >= 0, got {margin}")
    H, W = int(img.shape[0]), int(img.shape[1])
    if margin > min(H, W):
        raise ValueError(f"margin {margin} exceeds min image extent {min(H, W)}")
    g = A.to_device64(img)
    out = torch.empty((H + 2 * margin, W + 2 * margin), dtype=torch.float64, device=g.device)
    L.call("pnp_pad_symmetric_f64", L.context(g.device.index), L.ptr(g), H, W, int(margin),
           L.ptr(out))
    return A.from_device64(out, kind)


def integral_image(img):
    """Summed-area table with a zero leading row and column: entry (i, j) =
    sum of img over rows < i, columns < j (image.py:116-126)."""
    img, kind = A.validate(img)
    g = A.to_device64(img)
    H, W = int(g.shape[0]), int(g.shape[1])
    out = torch.empty((H + 1, W + 1), dtype=torch.float64, device=g.device)
    L.call("pnp_integral_image_f64", L.context(g.device.index), L.ptr(g), H, W, L.ptr(out))
    return A.from_device64(out, kind)


def box_sum(ii, top: int, left: int, size: int) -> float:
    """Sum of the size x size box at (top, left) from an integral image: four
    lookups (image.py:129-140)."""
    if size < 1:
        raise ValueError(f"box size must be >= 1, got {size}")
    height, width = int(ii.shape[0]) - 1, int(ii.shape[1]) - 1
    if top < 0 or left < 0 or top + size > height or left + size > width:
        raise ValueError(f"box ({top},{left}) of size {size} outside {height}x{width} extent")
    b, r = top + size, left + size
    if isinstance(ii, torch.Tensor):
        v = ii[[b, top, b, top], [r, r, left, left]].double().cpu().tolist()
    else:
        v = [float(ii[b, r]), float(ii[top, r]), float(ii[b, left]), float(ii[top, left])]
    return float(v[0] - v[1] - v[2] + v[3])


def psnr(reference, test, peak: float = 1.0) -> float:
    """Peak signal-to-noise ratio in dB; +inf when the images are identical."""
    r = A.to_device64(A.validate(reference, "reference")[0])
    t = A.to_device64(A.validate(test, "test")[0])
    if r.shape != t.shape:
        raise ValueError(f"dimension mismatch: {tuple(r.shape)} vs {tuple(t.shape)}")
    if peak <= 0:
        raise ValueError(f"peak must be > 0, got {peak}")
    mse = float(((r - t) ** 2).mean())
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)


# the reference keeps its PGM / PFM file I/O in image.py (169-280)
from .imageio import (  # noqa: E402,F401
    ImageFormatError,
    MalformedHeaderError,
    TruncatedPayloadError,
    UnsupportedFormatError,
    read_image,
    write_image,
)
