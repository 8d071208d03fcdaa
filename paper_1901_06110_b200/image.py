"""Image conventions and pixel primitives — drop-in for pnprestore/image.py
(validate_image 32-41, constraint sets + project 48-90, psnr 146-157).
Projection and PSNR run on the GPU; PGM / PFM file I/O (image.py:169-280)
is in imageio.py."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
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


def psnr(reference, test, peak: float = 1.0) -> float:
    """Peak signal-to-noise ratio in dB; +inf when the images are identical."""
    r = A.to_device(A.validate(reference, "reference")[0]).double()
    t = A.to_device(A.validate(test, "test")[0]).double()
    if r.shape != t.shape:
        raise ValueError(f"dimension mismatch: {tuple(r.shape)} vs {tuple(t.shape)}")
    if peak <= 0:
        raise ValueError(f"peak must be > 0, got {peak}")
    mse = float(((r - t) ** 2).mean())
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)
