"""Seeded synthetic inputs for the BASELINE.json configs (host-side, one-off).

The reference ships no dataset for this path and the paper's images are not
available, so every config is built from seeds.  The random stream is the
reference's splitmix64 (/root/reference/pkg/src/pnprestore/forward.py:37-79)
so draws are platform independent; simulators reuse the reference's
semantics (``sr_simulate`` forward.py:206-214, ``qis_simulate``
forward.py:263-298 — the latter runs in the native library, see
``forward.qis_simulate``).

``scene(H, W, seed)``:
  * uniforms u = SplitMix64(seed).uniforms(1 + 6*40)
  * linear ramp in [0.15, 0.85] along direction theta = 2*pi*u[0], over pixel
    centres ((x+0.5)/W, (y+0.5)/H), min-max normalised;
  * 40 shapes painted in order, shape i uses u[1+6i : 7+6i] =
    (kind, cy, cx, e1, e2, intensity): rect if kind < 0.5 else disc, centre
    (cy*H, cx*W), extents (0.02 + 0.13 e)*min(H, W) (half-height/half-width,
    or radius = first extent), pixel centres inside are set to intensity;
  * clip to [0, 1].
``noisy(clean, sigma, seed)`` adds SplitMix64(seed).normals(H*W)*sigma (not
clipped).
"""

from __future__ import annotations

import math

import numpy as np

_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1


class SplitMix64:
    """Counter-based splitmix64: output n uses state seed + n*GOLDEN."""

    def __init__(self, seed: int):
        self._state = seed & _MASK

    def next_uint64(self) -> int:
        self._state = (self._state + _GOLDEN) & _MASK
        z = self._state
        z = ((z ^ (z >> 30)) * _MIX1) & _MASK
        z = ((z ^ (z >> 27)) * _MIX2) & _MASK
        return (z ^ (z >> 31)) & _MASK

    def uniform(self) -> float:
        return (self.next_uint64() >> 11) * 2.0 ** -53

    def uniforms(self, n: int) -> np.ndarray:
        if n < 0:
            raise ValueError(f"n must be >= 0, got {n}")
        out = np.empty(n, dtype=np.float64)
        base = self._state
        step = 1 << 22
        with np.errstate(over="ignore"):
            for s in range(0, n, step):
                k = np.arange(s + 1, min(n, s + step) + 1, dtype=np.uint64)
                z = np.uint64(base) + np.uint64(_GOLDEN) * k
                z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
                z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
                z ^= z >> np.uint64(31)
                out[s:s + k.size] = (z >> np.uint64(11)) * 2.0 ** -53
        self._state = (self._state + n * _GOLDEN) & _MASK
        return out

    def normals(self, n: int) -> np.ndarray:
        pairs = (n + 1) // 2
        u = self.uniforms(2 * pairs)
        r = np.sqrt(-2.0 * np.log1p(-u[0::2]))
        th = 2.0 * math.pi * u[1::2]
        out = np.empty(2 * pairs)
        out[0::2] = r * np.cos(th)
        out[1::2] = r * np.sin(th)
        return out[:n]


def scene(h: int, w: int, seed: int, n_shapes: int = 40, rows: tuple | None = None) -> np.ndarray:
    """Clean float64 scene in [0, 1] (see module docstring).  ``rows=(r0, r1)``
    returns just those rows of the h x w scene (same values)."""
    r0, r1 = (0, h) if rows is None else rows
    u = SplitMix64(seed).uniforms(1 + 6 * n_shapes)
    th = 2.0 * math.pi * u[0]
    ys = (np.arange(h) + 0.5) / h
    xs = (np.arange(w) + 0.5) / w
    c, s_ = math.cos(th), math.sin(th)
    # the projection is linear, so its extrema sit at the image corners
    corners = [c * xs[i] + s_ * ys[j] for i in (0, -1) for j in (0, -1)]
    lo, hi = min(corners), max(corners)
    proj = c * xs[None, :] + s_ * ys[r0:r1, None]
    ramp = (proj - lo) / (hi - lo) if hi > lo else np.full_like(proj, 0.5)
    img = 0.15 + 0.7 * ramp
    side = min(h, w)
    for i in range(n_shapes):
        kind, cy, cx, e1, e2, val = u[1 + 6 * i:7 + 6 * i]
        cy, cx = cy * h, cx * w
        a = (0.02 + 0.13 * e1) * side
        b = (0.02 + 0.13 * e2) * side
        ext_y, ext_x = (a, b) if kind < 0.5 else (a, a)
        a0 = max(r0, int(math.floor(cy - ext_y - 1)))
        a1 = min(r1, int(math.ceil(cy + ext_y + 1)))
        c0 = max(0, int(math.floor(cx - ext_x - 1)))
        c1 = min(w, int(math.ceil(cx + ext_x + 1)))
        if a0 >= a1 or c0 >= c1:
            continue
        yy = (np.arange(a0, a1) + 0.5)[:, None] - cy
        xx = (np.arange(c0, c1) + 0.5)[None, :] - cx
        if kind < 0.5:
            m = (np.abs(yy) <= a) & (np.abs(xx) <= b)
        else:
            m = yy * yy + xx * xx <= a * a
        img[a0 - r0:a1 - r0, c0:c1][m] = val
    return np.clip(img, 0.0, 1.0)


def noisy(clean: np.ndarray, sigma: float, seed: int, first_index: int = 0) -> np.ndarray:
    """clean + sigma * splitmix normals (not clipped).  ``first_index`` (even)
    is the raster index of clean's first pixel in the full image, so rows of
    a large image can be generated independently (the stream is counter
    based: draw n uses state seed + n * GOLDEN)."""
    if first_index % 2:
        raise ValueError("first_index must be even (normals come in Box-Muller pairs)")
    rng = SplitMix64((seed + first_index * _GOLDEN) & _MASK)
    n = rng.normals(clean.size).reshape(clean.shape)
    return clean + sigma * n
