"""Forward models on the B200 — drop-in for pnprestore/forward.py.

Names/semantics follow /root/reference/pkg/src/pnprestore/forward.py:
``gaussian_kernel`` (86-95), ``SuperResOp`` (98-131), ``sr_apply`` (151-156),
``sr_adjoint`` (159-166), ``sr_data_term`` (177-180), ``sr_gradient``
(183-185), ``power_iteration_lipschitz`` (188-203), ``sr_simulate``
(206-214), ``QisModel`` / ``QisCounts`` (226-260), ``qis_simulate``
(263-298), ``qis_data_term`` (312-319), ``qis_gradient`` (322-327),
``qis_initial_estimate`` (330-332).

Blur/decimation/adjoint and the QIS likelihood run in csrc/pnp_forward.cu.
The SR kernel must be separable (every kernel the reference builds is: its
``gaussian_kernel`` is an outer product); a non-separable kernel raises
ValueError.  ``qis_simulate``'s sequential Knuth sampler runs in the native
library on the host, bit-exact with the reference.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _arrays as A
from . import _lib as L
from .synth import SplitMix64  # noqa: F401  (reference forward.SplitMix64)

QIS_FLOOR = 1e-6


def gaussian_kernel(sigma: float, radius: int) -> np.ndarray:
    """Normalized Gaussian blur kernel on a (2r+1)^2 grid (host, tiny)."""
    if sigma <= 0:
        raise ValueError(f"sigma must be > 0, got {sigma}")
    if radius < 1:
        raise ValueError(f"radius must be >= 1, got {radius}")
    grid = np.arange(-radius, radius + 1, dtype=np.float64)
    prof = np.exp(-(grid ** 2) / (2.0 * sigma * sigma))
    k = prof[:, None] * prof[None, :]
    return k / k.sum()


@dataclass(frozen=True, eq=False)
class SuperResOp:
    """Blur kernel + integer downsampling factor + boundary handling."""

    kernel: np.ndarray
    factor: int
    boundary: str = "periodic"

    def __post_init__(self) -> None:
        k = np.asarray(self.kernel, dtype=np.float64)
        if k.ndim != 2 or k.shape[0] != k.shape[1] or k.shape[0] % 2 == 0:
            raise ValueError(f"kernel must be odd and square, got shape {k.shape}")
        if np.any(k < 0) or not np.all(np.isfinite(k)):
            raise ValueError("kernel entries must be finite and >= 0")
        if abs(float(k.sum()) - 1.0) > 1e-12:
            raise ValueError(f"kernel must sum to 1, got {float(k.sum())!r}")
        if self.factor < 1:
            raise ValueError(f"factor must be >= 1, got {self.factor}")
        if self.boundary not in ("periodic", "symmetric"):
            raise ValueError(f"boundary must be 'periodic' or 'symmetric', got {self.boundary!r}")
        k = k.copy()
        k.setflags(write=False)
        object.__setattr__(self, "kernel", k)
        # separable factorization k = u v^T (u = row sums, v = column sums)
        u, v = k.sum(axis=1), k.sum(axis=0)
        if np.abs(np.outer(u, v) - k).max() > 1e-12:
            raise ValueError("SuperResOp on the GPU needs a separable (rank-1) blur kernel")
        taps = [float(t) for t in u] + [float(t) for t in v]
        object.__setattr__(self, "_taps", (C.c_float * len(taps))(*taps))

    @property
    def radius(self) -> int:
        return self.kernel.shape[0] // 2

    @property
    def kernel_symmetric(self) -> bool:
        return np.array_equal(self.kernel, self.kernel[::-1, :]) and np.array_equal(
            self.kernel, self.kernel[:, ::-1])

    @property
    def _bnd(self) -> int:
        return 1 if self.boundary == "symmetric" else 0

    def _check_hr(self, H: int, W: int) -> None:
        if H % self.factor or W % self.factor:
            raise ValueError(f"dimensions {(H, W)} not divisible by factor {self.factor}")
        if self.radius > min(H, W):
            raise ValueError(f"kernel radius {self.radius} exceeds image extent {min(H, W)}")

    # ---- device entry points (float32 CUDA tensors, no validation) -------
    def apply_device(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        B, H, W = A.dims(x)
        k = self.factor
        if out is None:
            out = torch.empty(x.shape[:-2] + (H // k, W // k), dtype=torch.float32, device=x.device)
        L.call("pnp_sr_apply", L.context(x.device.index), L.ptr(x), L.ptr(out), B, H, W,
               self._taps, self.radius, k, self._bnd)
        return out

    def adjoint_device(self, y: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        B, h, w = A.dims(y)
        k = self.factor
        if out is None:
            out = torch.empty(y.shape[:-2] + (h * k, w * k), dtype=torch.float32, device=y.device)
        L.call("pnp_sr_adjoint", L.context(y.device.index), L.ptr(y), L.ptr(out), B, h * k, w * k,
               self._taps, self.radius, k, self._bnd)
        return out

    def gradient_device(self, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor,
                        data_out: torch.Tensor | None = None) -> torch.Tensor:
        B, H, W = A.dims(x)
        L.call("pnp_sr_grad", L.context(x.device.index), L.ptr(x), L.ptr(y), L.ptr(out), B, H, W,
               self._taps, self.radius, self.factor, self._bnd, L.ptr(data_out))
        return out

    def gram_device(self, x: torch.Tensor, out: torch.Tensor, shift: float = 0.0) -> torch.Tensor:
        """out = A^T A x + shift x (the standard PnP-ADMM x-update operator)."""
        B, H, W = A.dims(x)
        L.call("pnp_sr_gram", L.context(x.device.index), L.ptr(x), L.ptr(out), B, H, W,
               self._taps, self.radius, self.factor, self._bnd, float(shift))
        return out

    def cg_device(self, rhs: torch.Tensor, x: torch.Tensor, shift: float, tol: float,
                  max_iters: int, warm: bool):
        """Solve (A^T A + shift I) x = rhs per image by conjugate gradients on
        the device (x: in = start if warm, out = solution).  Returns per-image
        (iterations, relative residual, status) lists."""
        B, H, W = A.dims(x)
        it = (C.c_int * B)()
        res = (C.c_double * B)()
        stat = (C.c_int * B)()
        L.call("pnp_sr_cg", L.context(x.device.index), L.ptr(rhs), L.ptr(x), B, H, W, self._taps,
               self.radius, self.factor, self._bnd, float(shift), float(tol), int(max_iters),
               1 if warm else 0, it, res, stat)
        return list(it), list(res), list(stat)

    def gradient_xupdate_device(self, x, y, v, u, z, mu, alpha, rho, lo, hi, flags,
                                data_out=None) -> None:
        """grad f(x) with the linearized-ADMM x-update fused into the adjoint
        kernel: x <- proj(mu (alpha x + rho (v - u) - grad)), z = x + u."""
        B, H, W = A.dims(x)
        L.call("pnp_sr_grad_xupdate", L.context(x.device.index), L.ptr(x), L.ptr(y), B, H, W,
               self._taps, self.radius, self.factor, self._bnd, L.ptr(data_out), L.ptr(v),
               L.ptr(u), L.ptr(z), mu, alpha, rho, lo, hi, L.ptr(flags))


def _hr_input(op: SuperResOp, x, name="image"):
    x, kind = A.validate(x, name, batch_ok=True)
    t = A.to_device(x)
    _, H, W = A.dims(t)
    op._check_hr(H, W)
    return t, kind


def _lr_obs(op: SuperResOp, y, hr_shape):
    y, _ = A.validate(y, "observation", batch_ok=True)
    t = A.to_device(y)
    want = tuple(hr_shape[:-2]) + (hr_shape[-2] // op.factor, hr_shape[-1] // op.factor)
    if tuple(t.shape) != want:
        raise ValueError(f"dimension mismatch: A x is {want}, observation {tuple(t.shape)}")
    return t


def sr_apply(op: SuperResOp, x):
    """Blur then keep every factor-th sample (positions k*i, k*j)."""
    t, kind = _hr_input(op, x)
    return A.from_device(op.apply_device(t), kind)


def sr_adjoint(op: SuperResOp, y):
    """Zero-fill upsample then blur; exact adjoint of sr_apply."""
    y, kind = A.validate(y, "image", batch_ok=True)
    if not op.kernel_symmetric:
        raise ValueError("adjoint requires a per-axis symmetric kernel")
    t = A.to_device(y)
    _, h, w = A.dims(t)
    op._check_hr(h * op.factor, w * op.factor)
    return A.from_device(op.adjoint_device(t), kind)


def sr_data_term(op: SuperResOp, x, y) -> float:
    """Quadratic misfit 0.5 * ||y - A x||^2."""
    t, _ = _hr_input(op, x)
    yt = _lr_obs(op, y, tuple(t.shape))
    B = A.dims(t)[0]
    data = torch.empty(B, dtype=torch.float64, device=t.device)
    scratch = torch.empty_like(t)
    op.gradient_device(t, yt, scratch, data)
    return float(data[0]) if t.dim() == 2 else data.cpu().numpy()


def sr_gradient(op: SuperResOp, x, y):
    """Descent gradient A^T (A x - y) of the quadratic misfit."""
    if not op.kernel_symmetric:
        raise ValueError("adjoint requires a per-axis symmetric kernel")
    t, kind = _hr_input(op, x)
    yt = _lr_obs(op, y, tuple(t.shape))
    return A.from_device(op.gradient_device(t, yt, torch.empty_like(t)), kind)


def power_iteration_lipschitz(op: SuperResOp, hr_shape: tuple[int, int],
                              iters: int = 200, seed: int = 0) -> float:
    """Largest eigenvalue of A^T A by power iteration (forward.py:188-203).
    The start vector is SplitMix64(seed) uniforms + 0.5 drawn on the device
    (bit-identical to the host stream); the loop never synchronizes -- a zero
    norm (the reference's early ``return 0.0``) is detected once at the end."""
    if iters < 1:
        raise ValueError(f"iters must be >= 1, got {iters}")
    op._check_hr(*hr_shape)
    n = hr_shape[0] * hr_shape[1]
    dev = torch.device("cuda", torch.cuda.current_device())
    u = torch.empty(n, dtype=torch.float64, device=dev)
    L.call("pnp_splitmix_uniforms", L.context(dev.index), seed & ((1 << 64) - 1), n, L.ptr(u))
    x = (u + 0.5).reshape(hr_shape)
    x = (x / torch.sqrt((x * x).sum())).float()
    zero = torch.zeros((), dtype=torch.bool, device=dev)
    for _ in range(iters):
        z = op.adjoint_device(op.apply_device(x)).double()
        norm = torch.sqrt((z * z).sum())
        zero |= norm == 0.0
        x = (z / norm).float()
    z = op.adjoint_device(op.apply_device(x)).double()
    xd = x.double()
    ray = (xd * z).sum() / (xd * xd).sum()
    return 0.0 if bool(zero) else float(ray)


def sr_simulate(x, op: SuperResOp, noise_sigma: float, seed: int):
    """Observation A x plus iid Gaussian noise, bit-reproducible per seed
    (forward.py:206-214).  Blur/decimate and the SplitMix64 Box-Muller noise
    both run on the device; y + sigma * n is formed in float64 (numpy in ->
    float64 out, tensor in -> float32 out)."""
    if noise_sigma < 0:
        raise ValueError(f"noise_sigma must be >= 0, got {noise_sigma}")
    t, kind = _hr_input(op, x)
    y = op.apply_device(t)
    if noise_sigma > 0:
        ctx = L.context(y.device.index)
        s64 = seed & ((1 << 64) - 1)
        if kind == A.NUMPY:
            out = torch.empty(y.shape, dtype=torch.float64, device=y.device)
            L.call("pnp_sr_add_noise", ctx, L.ptr(y), y.numel(), s64, float(noise_sigma),
                   None, L.ptr(out))
            return out.cpu().numpy()
        out = torch.empty_like(y)
        L.call("pnp_sr_add_noise", ctx, L.ptr(y), y.numel(), s64, float(noise_sigma),
               L.ptr(out), None)
        y = out
    return A.from_device(y, kind)


# ---------------------------------------------------------------------------
# Single-photon (QIS) model
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class QisModel:
    """Oversampling factor K (jots per pixel) and sensor gain."""

    oversampling: int
    gain: float

    def __post_init__(self) -> None:
        if self.oversampling < 1:
            raise ValueError(f"oversampling must be >= 1, got {self.oversampling}")
        if not self.gain > 0:
            raise ValueError(f"gain must be > 0, got {self.gain}")


class QisCounts:
    """Per-pixel counts of jots that fired (ones) and stayed dark (zeros)."""

    def __init__(self, ones, zeros):
        ones, _ = A.validate(ones, "ones", batch_ok=True)
        zeros, _ = A.validate(zeros, "zeros", batch_ok=True)
        o = np.asarray(ones.cpu() if isinstance(ones, torch.Tensor) else ones, dtype=np.float64)
        z = np.asarray(zeros.cpu() if isinstance(zeros, torch.Tensor) else zeros, dtype=np.float64)
        if o.shape != z.shape:
            raise ValueError(f"dimension mismatch: {o.shape} vs {z.shape}")
        for name, arr in (("ones", o), ("zeros", z)):
            if np.any(arr < 0) or np.any(arr != np.round(arr)):
                raise ValueError(f"{name} must be nonnegative integers")
        total = o + z
        if total.min() != total.max():
            raise ValueError("ones + zeros must equal the same K at every pixel")
        self.ones = o
        self.zeros = z
        self.oversampling = int(total.flat[0])
        self._dev = None

    @property
    def shape(self):
        return self.ones.shape

    def device(self):
        """(ones, zeros) as float32 CUDA tensors (integers < 2^24: exact)."""
        if self._dev is None:
            self._dev = (A.to_device(self.ones), A.to_device(self.zeros))
        return self._dev


def qis_simulate(x, model: QisModel, seed: int) -> QisCounts:
    """Binary jots from the Poisson single-photon model (Knuth product method,
    raster-then-jot uniform consumption; native host loop, bit-exact)."""
    x, _ = A.validate(x)
    x = np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x, dtype=np.float64)
    stop = np.ascontiguousarray(np.exp(-model.gain * np.clip(x, 0.0, 1.0) / model.oversampling).ravel())
    hits = np.zeros(x.size)
    L.call("pnp_qis_simulate_host", stop.ctypes.data_as(C.c_void_p), x.size, model.oversampling,
           seed & ((1 << 64) - 1), hits.ctypes.data_as(C.c_void_p))
    ones = hits.reshape(x.shape)
    return QisCounts(ones, model.oversampling - ones)


def _qis_args(x, counts: QisCounts, model: QisModel):
    x, kind = A.validate(x, batch_ok=True)
    t = A.to_device(x)
    if tuple(t.shape) != tuple(counts.shape):
        raise ValueError(f"dimension mismatch: {tuple(t.shape)} vs {counts.shape}")
    if counts.oversampling != model.oversampling:
        raise ValueError(f"counts are for K={counts.oversampling}, model has K={model.oversampling}")
    return t, kind


def qis_grad_device(x, ones, zeros, model: QisModel, floor: float, grad=None, data_out=None):
    B, H, W = A.dims(x)
    L.call("pnp_qis_grad", L.context(x.device.index), L.ptr(x), L.ptr(ones), L.ptr(zeros),
           L.ptr(grad), B, H * W, model.gain / model.oversampling, float(floor), L.ptr(data_out))
    return grad


def qis_grad_xupdate_device(x, ones, zeros, model: QisModel, floor: float, v, u, z, mu, alpha,
                            rho, lo, hi, flags, data_out=None) -> None:
    """QIS gradient with the linearized-ADMM x-update fused (one pass)."""
    B, H, W = A.dims(x)
    L.call("pnp_qis_grad_xupdate", L.context(x.device.index), L.ptr(x), L.ptr(ones), L.ptr(zeros),
           B, H * W, model.gain / model.oversampling, float(floor), L.ptr(data_out), L.ptr(v),
           L.ptr(u), L.ptr(z), mu, alpha, rho, lo, hi, L.ptr(flags))


def qis_data_term(x, counts: QisCounts, model: QisModel, floor: float = QIS_FLOOR) -> float:
    """sum_i K0_i z_i - K1_i log(1 - exp(-z_i)), z = gain max(x, floor) / K."""
    t, _ = _qis_args(x, counts, model)
    ones, zeros = counts.device()
    data = torch.empty(A.dims(t)[0], dtype=torch.float64, device=t.device)
    qis_grad_device(t, ones, zeros, model, floor, None, data)
    return float(data[0]) if t.dim() == 2 else data.cpu().numpy()


def qis_gradient(x, counts: QisCounts, model: QisModel, floor: float = QIS_FLOOR):
    """Per-pixel derivative (gain/K) (K0_i - K1_i / (exp(z_i) - 1))."""
    t, kind = _qis_args(x, counts, model)
    ones, zeros = counts.device()
    return A.from_device(qis_grad_device(t, ones, zeros, model, floor, torch.empty_like(t)), kind)


def qis_initial_estimate(counts: QisCounts, floor: float = QIS_FLOOR) -> np.ndarray:
    """Fraction of fired jots, clamped to [floor, 1]."""
    return np.clip(counts.ones / counts.oversampling, floor, 1.0)
