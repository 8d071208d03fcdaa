"""Forward models restated in float64 numpy — TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/pnprestore/forward.py (line numbers cited per
function).  The super-resolution blur keeps the reference's 2-D shifted-add
order so that results agree with it to the last few ulps.
"""

from __future__ import annotations

import math

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
MASK = (1 << 64) - 1
QIS_FLOOR = 1e-6                                    # forward.py:223


class SplitMix64:
    """splitmix64 stream (forward.py:37-79)."""

    def __init__(self, seed: int):
        self.state = seed & MASK

    def next_uint64(self) -> int:
        self.state = (self.state + GOLDEN) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * MIX1) & MASK
        z = ((z ^ (z >> 27)) * MIX2) & MASK
        return (z ^ (z >> 31)) & MASK

    def uniforms(self, n: int) -> np.ndarray:
        k = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + np.uint64(GOLDEN) * k
            z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * GOLDEN) & MASK
        return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def normals(self, n: int) -> np.ndarray:
        """Box-Muller on consecutive pairs (forward.py:70-79)."""
        m = (n + 1) // 2
        u = self.uniforms(2 * m)
        r = np.sqrt(-2.0 * np.log1p(-u[0::2]))
        th = 2.0 * math.pi * u[1::2]
        out = np.empty(2 * m)
        out[0::2] = r * np.cos(th)
        out[1::2] = r * np.sin(th)
        return out[:n]


def gaussian_kernel(sigma: float, radius: int) -> np.ndarray:
    """Normalized separable Gaussian on (2r+1)^2 (forward.py:86-95)."""
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    p = np.exp(-(x * x) / (2.0 * sigma * sigma))
    k = p[:, None] * p[None, :]
    return k / k.sum()


def blur(img: np.ndarray, kernel: np.ndarray, boundary: str) -> np.ndarray:
    """Correlation with wrap/symmetric padding (_convolve, forward.py:134-148)."""
    r = kernel.shape[0] // 2
    h, w = img.shape
    if r > min(h, w):
        raise ValueError(f"kernel radius {r} exceeds image extent {min(h, w)}")
    pad = np.pad(img, r, mode="symmetric" if boundary == "symmetric" else "wrap")
    out = np.zeros_like(img, dtype=np.float64)
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            wt = kernel[dy + r, dx + r]
            if wt != 0.0:
                out += wt * pad[r + dy:r + dy + h, r + dx:r + dx + w]
    return out


def sr_apply(kernel, factor, boundary, x):
    """Blur then keep samples (k i, k j) (forward.py:151-156)."""
    x = np.asarray(x, np.float64)
    if x.shape[0] % factor or x.shape[1] % factor:
        raise ValueError(f"dimensions {x.shape} not divisible by factor {factor}")
    return blur(x, kernel, boundary)[::factor, ::factor]


def sr_adjoint(kernel, factor, boundary, y):
    """Zero-fill upsample then the same blur (forward.py:159-166)."""
    y = np.asarray(y, np.float64)
    up = np.zeros((y.shape[0] * factor, y.shape[1] * factor))
    up[::factor, ::factor] = y
    return blur(up, kernel, boundary)


def sr_data_term(kernel, factor, boundary, x, y) -> float:
    """0.5 ||A x - y||^2 (forward.py:177-180)."""
    r = sr_apply(kernel, factor, boundary, x) - y
    return 0.5 * float((r * r).sum())


def sr_gradient(kernel, factor, boundary, x, y):
    """A^T (A x - y) (forward.py:183-185)."""
    return sr_adjoint(kernel, factor, boundary, sr_apply(kernel, factor, boundary, x) - y)


def sr_simulate(x, kernel, factor, boundary, noise_sigma, seed):
    """A x + sigma * N(0,1) from SplitMix64(seed) (forward.py:206-214)."""
    y = sr_apply(kernel, factor, boundary, x)
    if noise_sigma > 0:
        y = y + noise_sigma * SplitMix64(seed).normals(y.size).reshape(y.shape)
    return y


def qis_simulate(x, K: int, gain: float, seed: int):
    """Knuth-product Poisson jots, raster-then-jot order (forward.py:263-298).
    Returns (ones, zeros)."""
    x = np.asarray(x, np.float64)
    stop = np.exp(-gain * np.clip(x, 0.0, 1.0) / K).ravel().tolist()
    rng = SplitMix64(seed)
    chunk = 1 << 16
    buf = rng.uniforms(chunk).tolist()
    pos = 0
    hits = np.zeros(x.size)
    for i, thr in enumerate(stop):
        fired = 0
        for _ in range(K):
            cnt = 0
            prod = 1.0
            while True:
                if pos == len(buf):
                    buf = rng.uniforms(chunk).tolist()
                    pos = 0
                prod *= buf[pos]
                pos += 1
                if prod <= thr:
                    break
                cnt += 1
            if cnt >= 1:
                fired += 1
        hits[i] = fired
    ones = hits.reshape(x.shape)
    return ones, K - ones


def qis_data_term(x, ones, zeros, K: int, gain: float, floor: float = QIS_FLOOR) -> float:
    """sum K0 z - K1 log(1 - e^-z), z = gain max(x,floor)/K (forward.py:312-319)."""
    z = gain * np.maximum(np.asarray(x, np.float64), floor) / K
    return float((zeros * z - ones * np.log(-np.expm1(-z))).sum())


def qis_gradient(x, ones, zeros, K: int, gain: float, floor: float = QIS_FLOOR):
    """(gain/K)(K0 - K1/expm1(z)) (forward.py:322-327)."""
    z = gain * np.maximum(np.asarray(x, np.float64), floor) / K
    return (gain / K) * (zeros - ones / np.expm1(z))


def qis_initial_estimate(ones, K: int, floor: float = QIS_FLOOR):
    """clip(K1/K, floor, 1) (forward.py:330-332)."""
    return np.clip(np.asarray(ones, np.float64) / K, floor, 1.0)
