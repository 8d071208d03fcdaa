"""Linearized PnP-ADMM restated in float64 — TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/pnprestore/solver.py:147-235 (Algorithm 1 of
arXiv 1901.06110) and image.py:81-90,146-157 (projection, PSNR).
"""

from __future__ import annotations

import math
from typing import Callable

import numpy as np

from . import dsg


class DivergenceError(RuntimeError):
    """solver.py:46-47."""


def project(img, lo: float | None, hi: float | None) -> np.ndarray:
    """Clamp projection (image.py:81-90); (None, None) = unconstrained copy."""
    img = np.asarray(img, np.float64)
    if lo is None and hi is None:
        return img.copy()
    if hi is None:
        return np.maximum(img, lo)
    return np.clip(img, lo, hi)


def psnr(ref, test, peak: float = 1.0) -> float:
    """image.py:146-157."""
    mse = float(np.mean((np.asarray(ref, np.float64) - np.asarray(test, np.float64)) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)


def residuals(x, v, v_prev, rho):
    """Mean-square primal gap and dual change (solver.py:147-153)."""
    return float(np.mean((x - v) ** 2)), float(np.mean((rho * (v - v_prev)) ** 2))


def make_denoiser(kind: str, P: int, R: int, bw: float, lam: float = 1.0,
                  freeze_at: int | None = 15, patch_sigma=None):
    """Schedule closure (solver.py:156-177)."""
    if kind == "identity" or lam == 0.0:
        return lambda img, k: img.copy()
    if kind == "nlm":
        return lambda img, k: dsg.nlm_denoise(img, P, R, bw, patch_sigma=patch_sigma)
    if kind == "dsg-adaptive":
        return lambda img, k: dsg.dsg_nlm_denoise(img, P, R, bw, patch_sigma=patch_sigma)
    frozen = None

    def fixed(img, k):
        nonlocal frozen
        if freeze_at is None or k < freeze_at:
            return dsg.dsg_nlm_denoise(img, P, R, bw, patch_sigma=patch_sigma)
        if frozen is None:
            frozen = dsg.freeze_guide(img, P, R, bw, patch_sigma)
        return frozen.apply(img)

    return fixed


def _finite(k, *arrays):
    for a in arrays:
        if not np.all(np.isfinite(a)):
            raise DivergenceError(f"non-finite iterate at iteration {k}")


def linearized_pnp_admm(x0, gradient: Callable, denoiser: Callable, *, rho: float,
                        alpha: float, max_iters: int, lo=None, hi=None,
                        objective: Callable | None = None, ground_truth=None,
                        callback=None, stop_tol=None):
    """solver.py:199-235.  Returns (v, records) with records as tuples
    (k, primal, dual, psnr, objective)."""
    x = project(x0, lo, hi)
    v = x.copy()
    u = np.zeros(x.shape)
    mu = 1.0 / (alpha + rho)
    recs = []
    for k in range(1, max_iters + 1):
        grad = gradient(x)
        x = mu * (alpha * x + rho * (v - u) - grad)
        _finite(k, x)
        x = project(x, lo, hi)
        v_prev = v
        dn_in = x + u
        _finite(k, dn_in)
        v = denoiser(dn_in, k)
        u = u + (x - v)
        _finite(k, v, u)
        primal, dual = residuals(x, v, v_prev, rho)
        q = psnr(ground_truth, v) if ground_truth is not None else math.nan
        obj = float(objective(x)) if objective is not None else math.nan
        recs.append((k, primal, dual, q, obj))
        if callback is not None:
            callback(k, x, v, u)
        if stop_tol is not None and primal < stop_tol and dual < stop_tol:
            break
    return v, recs


class CgBreakdownError(RuntimeError):
    """solver.py:50-51."""


def cg_solve(apply: Callable, rhs, tol: float, max_iters: int, x0=None):
    """Conjugate gradients for an SPD operator on images (solver.py:244-282).
    Returns (x, iterations, relative residual, converged)."""
    rhs = np.asarray(rhs, np.float64)
    bnorm = math.sqrt(float(np.sum(rhs * rhs)))
    if bnorm == 0.0:
        return np.zeros_like(rhs), 0, 0.0, True
    x = np.zeros_like(rhs) if x0 is None else np.array(x0, np.float64)
    r = rhs - apply(x)
    p = r.copy()
    rs = float(np.sum(r * r))
    it = 0
    for _ in range(max_iters):
        if math.sqrt(rs) / bnorm <= tol:
            break
        ap = apply(p)
        pap = float(np.sum(p * ap))
        if not math.isfinite(pap):
            raise DivergenceError("non-finite value inside conjugate gradients")
        if pap <= 0.0:
            raise CgBreakdownError(f"nonpositive curvature {pap!r}")
        a = rs / pap
        x = x + a * p
        r = r - a * ap
        rs_new = float(np.sum(r * r))
        p = r + (rs_new / rs) * p
        rs = rs_new
        it += 1
    res = math.sqrt(rs) / bnorm
    return x, it, res, res <= tol


def standard_pnp_admm_cg(x0, gram: Callable, atb, denoiser: Callable, *, rho: float,
                         max_iters: int, cg_tol: float, cg_max_iters: int,
                         cg_warm_start: bool = False, lo=None, hi=None,
                         objective: Callable | None = None, ground_truth=None):
    """Standard PnP-ADMM with the exact x-update by CG (solver.py:285-328):
    (A^T A + rho I) x = A^T y + rho (v - u); the constraint is applied once,
    to the returned v.  Returns (v, records) like linearized_pnp_admm."""
    x = np.array(x0, np.float64)
    v = x.copy()
    u = np.zeros(x.shape)
    recs = []
    for k in range(1, max_iters + 1):
        rhs = atb + rho * (v - u)
        x = cg_solve(lambda z: gram(z) + rho * z, rhs, cg_tol, cg_max_iters,
                     x0=x if cg_warm_start else None)[0]
        _finite(k, x)
        v_prev = v
        dn_in = x + u
        _finite(k, dn_in)
        v = denoiser(dn_in, k)
        u = u + (x - v)
        _finite(k, v, u)
        primal, dual = residuals(x, v, v_prev, rho)
        q = psnr(ground_truth, v) if ground_truth is not None else math.nan
        obj = float(objective(x)) if objective is not None else math.nan
        recs.append((k, primal, dual, q, obj))
    return project(v, lo, hi), recs
