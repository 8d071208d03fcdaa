"""DSG-NLM (doubly stochastic Gaussian NLM) restated in float64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows
/root/reference/pkg/src/pnprestore/denoise.py; each function names the lines
it restates.  One extension beyond the reference: optional Gaussian patch
weights (``patch_sigma``), defined so that ``patch_sigma=None`` (uniform
taps 1/P) reproduces the reference's box patch distance exactly:

    map_t(s) = P^2 * sum_{a,b} w_a w_b (G(s+(a,b)) - G(s+t+(a,b)))^2,
    w = patch_taps(P, sigma)  (sum w = 1)

so ``k = exp(-map / (2 P^2 bw^2)) = exp(-sum w_a w_b D / (2 bw^2))``; with
``h = sqrt(2) * bw`` this is the north-star ``exp(-d / h^2)``.
"""

from __future__ import annotations

import math

import numpy as np

MASS_FLOOR = 1e-300                      # denoise.py:34
KERNEL_CACHE_BYTES = 1 << 30             # denoise.py:29
DENSE_MAX_PIXELS = 4096                  # denoise.py:36


def validate(img, name="image") -> np.ndarray:
    """image.py:32-41 — float64, 2-D, non-empty, finite."""
    a = np.asarray(img, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {a.shape}")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"{name} must be at least 1x1, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        raise ValueError(f"{name} contains non-finite values")
    return a


def check_params(P: int, R: int, bw: float) -> None:
    """PatchParams.__post_init__ (denoise.py:47-53)."""
    if P < 1 or P % 2 == 0:
        raise ValueError(f"patch_side must be odd and >= 1, got {P}")
    if R < 1:
        raise ValueError(f"window_radius must be >= 1, got {R}")
    if not bw > 0:
        raise ValueError(f"bandwidth must be > 0, got {bw}")


def pad_symmetric(img: np.ndarray, margin: int) -> np.ndarray:
    """Half-sample mirror pad, index -1 -> 0 (image.py:97-113)."""
    img = validate(img)
    if margin < 0:
        raise ValueError(f"margin must be >= 0, got {margin}")
    if margin > min(img.shape):
        raise ValueError(f"margin {margin} exceeds min image extent {min(img.shape)}")
    return np.pad(img, margin, mode="symmetric") if margin else img.copy()


def patch_taps(P: int, sigma: float | None = None) -> np.ndarray:
    """Normalized 1-D patch taps.  None -> box 1/P (the reference's only mode,
    denoise.py:186,194); otherwise a sampled Gaussian exp(-a^2/(2 sigma^2))."""
    if sigma is None:
        return np.full(P, 1.0 / P)
    if not sigma > 0:
        raise ValueError(f"patch_sigma must be > 0, got {sigma}")
    a = np.arange(P, dtype=np.float64) - (P - 1) // 2
    w = np.exp(-(a * a) / (2.0 * sigma * sigma))
    return w / w.sum()


def window_offsets(h: int, w: int, R: int):
    """Raster window offsets with clipped dst/src slices (denoise.py:91-103)."""
    for dy in range(-R, R + 1):
        rd = slice(max(0, -dy), h - max(0, dy))
        rs = slice(max(0, dy), h - max(0, -dy))
        for dx in range(-R, R + 1):
            cd = slice(max(0, -dx), w - max(0, dx))
            cs = slice(max(0, dx), w - max(0, -dx))
            yield dy, dx, (rd, cd), (rs, cs)


def hat(dy: int, dx: int, R: int) -> float:
    """Separable hat taper (denoise.py:61-67, 199-201)."""
    s = R + 1
    return (1.0 - abs(dy) / s) * (1.0 - abs(dx) / s)


class Engine:
    """Kernel maps for one guide (restates _DistanceEngine + _WeightEngine,
    denoise.py:106-204).  Distances use direct separable sums rather than the
    reference's summed-area table; the two agree to ~1e-15 (the reference
    itself pins SAT == direct at 1e-10, tests/test_denoise.py:134-140)."""

    def __init__(self, guide: np.ndarray, P: int, R: int, bw: float,
                 taps: np.ndarray | None = None):
        check_params(P, R, bw)
        self.h, self.w = guide.shape
        self.P, self.R = P, R
        self.half = (P - 1) // 2
        self.margin = R + self.half                               # denoise.py:55-58
        self.pad = pad_symmetric(guide, self.margin)
        self.taps = np.full(P, 1.0 / P) if taps is None else np.asarray(taps, np.float64)
        self.inv = 1.0 / (2.0 * P * P * bw * bw)                  # denoise.py:186
        n_off = (2 * R + 1) ** 2
        fits = n_off * self.h * self.w * 8 <= KERNEL_CACHE_BYTES  # denoise.py:187-189
        self.cache: dict | None = {} if fits else None

    def distance(self, dy: int, dx: int) -> np.ndarray:
        """P^2 * weighted patch SSD for every pixel s against s+(dy,dx)."""
        a0 = self.margin - self.half
        rh, rw = self.h + 2 * self.half, self.w + 2 * self.half
        base = self.pad[a0:a0 + rh, a0:a0 + rw]
        shifted = self.pad[a0 + dy:a0 + dy + rh, a0 + dx:a0 + dx + rw]
        d = base - shifted
        d *= d
        t = self.taps
        vert = np.zeros((self.h, rw))
        for a in range(self.P):
            vert += t[a] * d[a:a + self.h, :]
        out = np.zeros((self.h, self.w))
        for b in range(self.P):
            out += t[b] * vert[:, b:b + self.w]
        return out * float(self.P * self.P)

    def kernel(self, dy: int, dx: int) -> np.ndarray:
        if self.cache is not None and (dy, dx) in self.cache:
            return self.cache[(dy, dx)]
        k = np.exp(-self.inv * self.distance(dy, dx))            # denoise.py:194
        if self.cache is not None:
            self.cache[(dy, dx)] = k
        return k

    def offsets(self):
        return window_offsets(self.h, self.w, self.R)


def mass_sweep(e: Engine) -> np.ndarray:
    """Sweep 1: g = row mass of hat * K (denoise.py:207-212), floored (286)."""
    g = np.zeros((e.h, e.w))
    for dy, dx, dst, _ in e.offsets():
        g[dst] += hat(dy, dx, e.R) * e.kernel(dy, dx)[dst]
    return np.maximum(g, MASS_FLOOR)


def scale_sweep(e: Engine, g: np.ndarray) -> tuple[np.ndarray, float]:
    """Sweep 2: normalized row sums d and m = max d (denoise.py:215-224)."""
    d = np.zeros((e.h, e.w))
    rs = 1.0 / np.sqrt(g)
    for dy, dx, dst, src in e.offsets():
        d[dst] += hat(dy, dx, e.R) * e.kernel(dy, dx)[dst] * rs[dst] * rs[src]
    return d, float(d.max())


def filter_sweep(e: Engine, image: np.ndarray, g: np.ndarray, m: float) -> np.ndarray:
    """Sweep 3: rescaled filter + diagonal correction (denoise.py:227-241)."""
    out = np.zeros((e.h, e.w))
    mass = np.zeros((e.h, e.w))
    inv_m = 1.0 / m
    rs = 1.0 / np.sqrt(g)
    for dy, dx, dst, src in e.offsets():
        wgt = inv_m * hat(dy, dx, e.R) * e.kernel(dy, dx)[dst]
        wgt *= rs[dst]
        wgt *= rs[src]
        out[dst] += wgt * image[src]
        mass[dst] += wgt
    out += (1.0 - mass) * image
    return out


def _pair(image, guide):
    """_check_pair (denoise.py:244-251)."""
    image = validate(image, "image")
    if guide is None:
        return image, image
    guide = validate(guide, "guide")
    if guide.shape != image.shape:
        raise ValueError(f"dimension mismatch: image {image.shape} vs guide {guide.shape}")
    return image, guide


def dsg_sweeps(guide, P: int, R: int, bw: float, patch_sigma: float | None = None):
    """(g, d, m, engine) for a guide — the guide-only half of DSG-NLM."""
    guide = validate(guide, "guide")
    e = Engine(guide, P, R, bw, patch_taps(P, patch_sigma))
    g = mass_sweep(e)
    d, m = scale_sweep(e, g)
    return g, d, m, e


def dsg_nlm_denoise(image, P: int, R: int, bw: float, guide=None,
                    patch_sigma: float | None = None, return_aux: bool = False):
    """dsg_nlm_denoise (denoise.py:272-288).  ``return_aux`` also returns the
    normalized row sums d and their max m (north-star 'alpha')."""
    image, guide = _pair(image, guide)
    g, d, m, e = dsg_sweeps(guide, P, R, bw, patch_sigma)
    out = filter_sweep(e, image, g, m)
    return (out, d, m) if return_aux else out


class FrozenGuide:
    """FrozenGuide / freeze_guide (denoise.py:358-386)."""

    def __init__(self, guide, P: int, R: int, bw: float, patch_sigma=None):
        self.guide = validate(guide, "guide").copy()
        self.guide.setflags(write=False)
        self.g, self.d, self.m, self.e = dsg_sweeps(self.guide, P, R, bw, patch_sigma)

    def apply(self, image) -> np.ndarray:
        image = validate(image, "image")
        if image.shape != self.guide.shape:
            raise ValueError(f"dimension mismatch: image {image.shape} vs guide {self.guide.shape}")
        return filter_sweep(self.e, image, self.g, self.m)


def freeze_guide(guide, P, R, bw, patch_sigma=None) -> FrozenGuide:
    return FrozenGuide(guide, P, R, bw, patch_sigma)


def nlm_denoise(image, P: int, R: int, bw: float, guide=None, patch_sigma=None):
    """Plain row-stochastic NLM (denoise.py:254-269)."""
    image, guide = _pair(image, guide)
    e = Engine(guide, P, R, bw, patch_taps(P, patch_sigma))
    num = np.zeros(image.shape)
    den = np.zeros(image.shape)
    for dy, dx, dst, src in e.offsets():
        k = e.kernel(dy, dx)
        num[dst] += k[dst] * image[src]
        den[dst] += k[dst]
    return num / den


def dense_weights(guide, P: int, R: int, bw: float, patch_sigma=None) -> np.ndarray:
    """Explicit n x n W (build_dense_weights, denoise.py:389-418)."""
    guide = validate(guide, "guide")
    h, w = guide.shape
    n = h * w
    if n > DENSE_MAX_PIXELS:
        raise ValueError(f"{h}x{w} image too large for dense weights (n={n})")
    e = Engine(guide, P, R, bw, patch_taps(P, patch_sigma))
    e.cache = None
    idx = np.arange(n).reshape(h, w)
    W = np.zeros((n, n))
    for dy, dx, dst, src in e.offsets():
        k = np.exp(-e.inv * e.distance(dy, dx))
        W[idx[dst].ravel(), idx[src].ravel()] = hat(dy, dx, R) * k[dst].ravel()
    row = W.sum(axis=1)
    col = W.sum(axis=0)
    W *= 1.0 / np.sqrt(row)[:, None]
    W *= 1.0 / np.sqrt(col)[None, :]
    W /= W.sum(axis=1).max()
    diag = np.arange(n)
    W[diag, diag] += 1.0 - W.sum(axis=1)
    return W


def bandwidth_from_h(h: float) -> float:
    """North-star h -> reference bandwidth: bw = h / sqrt(2)."""
    return h / math.sqrt(2.0)
