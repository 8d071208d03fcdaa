"""Linearized plug-and-play ADMM on the B200 — drop-in for pnprestore/solver.py.

Names/semantics follow /root/reference/pkg/src/pnprestore/solver.py:
``SolverConfig`` (54-101), ``Problem`` (104-114), ``IterationRecord`` /
``write_log_csv`` (117-144), ``residuals`` (147-153), ``_make_denoiser``
(156-177), ``linearized_pnp_admm`` (199-235), ``make_sr_problem`` (335-349),
``make_qis_problem`` (352-362), ``default_sr_alpha`` / ``default_qis_alpha``
(365-374), ``DivergenceError`` (46-47).

The iterates x, v, u stay on the GPU for the whole run.  One iteration is
  grad (SR: fused residual+adjoint kernels, QIS: one elementwise kernel, the
        data term of the previous iterate rides along),
  x-update + projection + x+u + finite flags (one kernel),
  denoiser (DSG sweep + fixup, or the frozen apply),
  u-update + primal/dual/PSNR partial sums + finite flags (one kernel);
log scalars accumulate in device arrays and come back once at the end (or
per iteration when ``stop_tol`` / a host callback needs them).  A non-finite
iterate raises DivergenceError with the same iteration index as the
reference.

Plug-in callables (``Problem.gradient``, ``denoiser``, ``callback``) keep the
reference contract: plain callables receive float64 numpy arrays.  Callables
marked with :func:`device_callable` (and everything built by this package)
receive float32 CUDA tensors and stay on device.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _arrays as A
from . import _lib as L
from .denoise import PatchParams, freeze_guide, kcache_scope
from .forward import (QIS_FLOOR, QisCounts, QisModel, SuperResOp, power_iteration_lipschitz,
                      qis_grad_device, qis_grad_xupdate_device, qis_initial_estimate, sr_adjoint)
from .image import UNCONSTRAINED, Constraint, bounds

DENOISERS = ("identity", "nlm", "dsg-adaptive", "dsg-fixed")


class DivergenceError(RuntimeError):
    """An iterate picked up non-finite values; the run was aborted."""


class CgBreakdownError(RuntimeError):
    """Conjugate gradients met nonpositive curvature (operator not SPD)."""


@dataclass
class CgResult:
    """Result of cg_solve (reference solver.py:236-241)."""

    x: object
    iterations: int
    residual: float
    converged: bool


def cg_solve(apply: Callable, rhs, tol: float, max_iters: int, x0=None) -> CgResult:
    """Conjugate gradients for an SPD operator on images (solver.py:244-282).

    Stops when ||rhs - Op(x)|| / ||rhs|| <= tol (recursive residual) or after
    max_iters.  ``apply`` is any operator on images; numpy in -> numpy out
    (host operators, as in the reference), CUDA tensors in -> the iteration
    runs on the device with torch vector updates around the user operator.
    The SR x-update of standard_pnp_admm_cg does not come here: it runs the
    native batched solver (pnp_sr_cg).
    """
    if not tol > 0:
        raise ValueError(f"tol must be > 0, got {tol}")
    if max_iters < 1:
        raise ValueError(f"max_iters must be >= 1, got {max_iters}")
    if not isinstance(rhs, torch.Tensor):
        rhs, _ = A.validate(rhs, "rhs")
    xp = torch if isinstance(rhs, torch.Tensor) else np
    dot = (lambda a, b: float(torch.sum(a.double() * b.double()))) if xp is torch else \
        (lambda a, b: float(np.sum(a * b)))
    bnorm = math.sqrt(dot(rhs, rhs))
    if bnorm == 0.0:
        return CgResult(xp.zeros_like(rhs), 0, 0.0, True)
    x = xp.zeros_like(rhs) if x0 is None else (x0.clone() if xp is torch else np.array(x0, np.float64))
    r = rhs - apply(x)
    p = r.clone() if xp is torch else r.copy()
    rs = dot(r, r)
    it = 0
    for _ in range(max_iters):
        if math.sqrt(rs) / bnorm <= tol:
            break
        ap = apply(p)
        pap = dot(p, ap)
        if not math.isfinite(pap):
            raise DivergenceError("non-finite value inside conjugate gradients")
        if pap <= 0.0:
            raise CgBreakdownError(f"nonpositive curvature {pap!r}")
        step = rs / pap
        x = x + step * p
        r = r - step * ap
        rs_new = dot(r, r)
        p = r + (rs_new / rs) * p
        rs = rs_new
        it += 1
    res = math.sqrt(rs) / bnorm
    return CgResult(x, it, res, res <= tol)


def device_callable(fn, graph_from: int | None = None):
    """Mark a plug-in as device-native: it receives/returns CUDA tensors.

    ``graph_from=k`` additionally declares that calls for iterations >= k
    only launch stream-ordered device work (no host sync, no cudaMalloc
    outside torch's allocator), so the solver may capture those iterations
    into one CUDA graph."""
    fn._pnp_device = True
    fn._pnp_graph_from = graph_from
    return fn


def _is_device(fn) -> bool:
    return bool(getattr(fn, "_pnp_device", False))


def _graph_from(fn) -> int | None:
    return getattr(fn, "_pnp_graph_from", None) if _is_device(fn) else None


@dataclass
class SolverConfig:
    """Hyperparameters (reference solver.py:54-101) + ``patch_sigma``
    (Gaussian patch weights for the built-in DSG/NLM denoisers)."""

    rho: float = 1.0
    lam: float = 0.02
    alpha: float = 1.1
    max_iters: int = 250
    freeze_at: int | None = 15
    constraint: Constraint = UNCONSTRAINED
    denoiser: str = "dsg-fixed"
    patch_side: int = 7
    window_radius: int = 10
    bandwidth: float | None = None
    stop_tol: float | None = None
    cg_tol: float = 1e-6
    cg_max_iters: int = 200
    cg_warm_start: bool = False
    patch_sigma: float | None = None

    def __post_init__(self) -> None:
        if not self.rho > 0:
            raise ValueError(f"rho must be > 0, got {self.rho}")
        if self.lam < 0:
            raise ValueError(f"lam must be >= 0, got {self.lam}")
        if not self.alpha > 0:
            raise ValueError(f"alpha must be > 0, got {self.alpha}")
        if self.max_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        if self.freeze_at is not None and self.freeze_at < 1:
            raise ValueError(f"freeze_at must be >= 1, got {self.freeze_at}")
        if self.denoiser not in DENOISERS:
            raise ValueError(f"denoiser must be one of {DENOISERS}, got {self.denoiser!r}")
        if self.bandwidth is not None and not self.bandwidth > 0:
            raise ValueError(f"bandwidth must be > 0, got {self.bandwidth}")
        if not self.cg_tol > 0:
            raise ValueError(f"cg_tol must be > 0, got {self.cg_tol}")
        if self.cg_max_iters < 1:
            raise ValueError(f"cg_max_iters must be >= 1, got {self.cg_max_iters}")

    def effective_bandwidth(self) -> float:
        if self.bandwidth is not None:
            return self.bandwidth
        return math.sqrt(self.lam / self.rho)

    def patch_params(self) -> PatchParams:
        return PatchParams(self.patch_side, self.window_radius, self.effective_bandwidth(),
                           self.patch_sigma)


@dataclass
class Problem:
    """Data-term oracles plus optional extras (reference solver.py:104-114).

    ``device_gradient(x, grad_out, data_out)`` — set by make_sr_problem /
    make_qis_problem — is the device path: it writes grad f(x) into
    ``grad_out`` and, when ``data_out`` is given, f(x) (float64 per image)."""

    shape: tuple
    gradient: Callable
    x0: object
    objective: Callable | None = None
    ground_truth: object | None = None
    gram: Callable | None = None
    atb: object | None = None
    device_gradient: Callable | None = field(default=None, repr=False)
    # fused gradient + x-update (set by make_sr_problem / make_qis_problem):
    # (x, v, u, z, mu, alpha, rho, lo, hi, flags, data_out) -> None
    device_grad_xupdate: Callable | None = field(default=None, repr=False)
    # native CG on (A^T A + shift I) x = rhs (set by make_sr_problem):
    # (rhs, x, shift, tol, max_iters, warm) -> (iterations, residuals, status)
    device_cg: Callable | None = field(default=None, repr=False)
    device_atb: object | None = field(default=None, repr=False)
    # the gradient's native description for the C++ iteration loop
    # (pnp_admm_run): (kind, obs, obs2, taps, radius, factor, boundary,
    # gain_over_K, floor) with kind 0 = SR, 1 = QIS
    native_grad: tuple | None = field(default=None, repr=False)


@dataclass
class IterationRecord:
    index: int
    primal: float
    dual: float
    psnr: float
    time_ms: float
    objective: float


CSV_HEADER = "iter,primal,dual,psnr,time_ms,objective"


def write_log_csv(records, path, include_time: bool = True) -> None:
    """One row per iteration, LF endings, shortest float repr (solver.py:130-144)."""
    lines = [CSV_HEADER]
    for r in records:
        t = r.time_ms if include_time else 0.0
        lines.append(f"{r.index},{float(r.primal)!r},{float(r.dual)!r},"
                     f"{float(r.psnr)!r},{float(t)!r},{float(r.objective)!r}")
    with open(path, "w", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


def residuals(x, v, v_prev, rho: float) -> tuple[float, float]:
    """Mean-square primal gap ||x-v||^2/n and dual change ||rho (v-v_prev)||^2/n."""
    ts = [A.to_device(a) for a in (x, v, v_prev)]
    if not (ts[0].shape == ts[1].shape == ts[2].shape):
        raise ValueError(f"dimension mismatch: {tuple(ts[0].shape)}, {tuple(ts[1].shape)}, "
                         f"{tuple(ts[2].shape)}")
    x_, v_, vp = (t.double() for t in ts)
    return float(((x_ - v_) ** 2).mean()), float(((rho * (v_ - vp)) ** 2).mean())


# ---------------------------------------------------------------------------
# Denoiser schedules (solver.py:156-177), device resident
# ---------------------------------------------------------------------------

def _make_denoiser(config: SolverConfig):
    # graph_from: the first call sizes the native scratch; dsg-fixed freezes
    # (cudaMalloc) at freeze_at, so its capturable iterations start after it
    if config.denoiser == "identity" or config.lam == 0.0:
        return device_callable(lambda img, k: img.clone(), graph_from=2)
    params = config.patch_params()
    if config.denoiser == "nlm":
        return device_callable(lambda img, k: _nlm_device(img, params), graph_from=2)
    if config.denoiser == "dsg-adaptive":
        return device_callable(lambda img, k: _dsg_device(img, params), graph_from=2)
    state = {"frozen": None}

    def fixed(img, k):
        if config.freeze_at is None or k < config.freeze_at:
            return _dsg_device(img, params)
        if state["frozen"] is None:
            state["frozen"] = freeze_guide(img, params)
        return state["frozen"].apply_device(img)

    fn = device_callable(fixed, graph_from=(config.freeze_at or 1) + 1)
    if config.freeze_at is not None:  # after the freeze the solver may fuse the u-update
        fn._pnp_frozen_for = lambda k: state["frozen"] if k > config.freeze_at else None
    return fn


def _nlm_device(img: torch.Tensor, params: PatchParams) -> torch.Tensor:
    """Unchecked device plain NLM (inputs already validated by the solver)."""
    B, H, W = A.dims(img)
    out = torch.empty_like(img)
    L.call("pnp_nlm_denoise", L.context(img.device.index), L.ptr(img), L.ptr(img), L.ptr(out),
           B, H, W, params.window_radius, params.patch_side, params._ctaps(),
           float(params.bandwidth))
    return out


def _dsg_device(img: torch.Tensor, params: PatchParams) -> torch.Tensor:
    """Unchecked device DSG-NLM (inputs already validated by the solver)."""
    B, H, W = A.dims(img)
    out = torch.empty_like(img)
    dev = img.device.index
    with kcache_scope(dev, B, H, W, params):
        L.call("pnp_dsg_denoise", L.context(dev), L.ptr(img), L.ptr(img), L.ptr(out),
               B, H, W, params.window_radius, params.patch_side, params._ctaps(),
               float(params.bandwidth), None, None)
    return out


# ---------------------------------------------------------------------------
# Linearized PnP-ADMM (Algorithm 1)
# ---------------------------------------------------------------------------

def _host_wrap_array_fn(fn, kind_shape):
    """Host plug-in: numpy float64 in, result uploaded back to the device."""
    def run(t: torch.Tensor, *extra):
        res = fn(t.detach().cpu().numpy().astype(np.float64), *extra)
        return A.to_device(res, t.device.index).reshape(t.shape)
    return run


def linearized_pnp_admm(problem: Problem, config: SolverConfig, denoiser=None, callback=None,
                        graph: bool = False, native: bool = True):
    """Gradient-step PnP-ADMM; returns (final v, per-iteration records).

    Per iteration: x <- proj(mu (alpha x + rho (v - u) - grad f(x))) with
    mu = 1/(alpha + rho), then v <- D(x + u), then u <- u + (x - v).
    The result is a float64 numpy array when ``problem.x0`` is numpy, else a
    CUDA tensor.

    ``graph``: when nothing needs the host between iterations (no callback,
    no stop_tol) and both the gradient and the denoiser are this package's
    device paths, the iterations from the denoiser's ``graph_from`` on are
    captured into one CUDA graph and replayed (no per-launch host cost).
    Off by default: measured on the B200 (config 2, 30 and 250 iterations),
    one-shot capture + instantiation costs more than the eager launches it
    saves, because the eager host loop already keeps pace with the device.
    Results are bitwise identical to the eager loop; the captured
    iterations' ``time_ms`` are interpolated over the replay.

    ``native``: with a frozen-guide denoiser, a device forward model and no
    callback / stop_tol / graph, the iterations from the first frozen one on
    run in the library's C++ loop (``pnp_admm_run``; same calls, bitwise
    identical iterates); ``native=False`` keeps the Python loop.
    """
    dev = A.device_index()
    x0, kind = A.validate(problem.x0, "x0", batch_ok=True)
    x = A.to_device(x0, dev).clone()
    B, H, W = A.dims(x)
    n = H * W
    lo, hi = bounds(config.constraint)
    ctx = L.context(dev)
    if denoiser is None:
        denoiser = _make_denoiser(config)
    den = denoiser if _is_device(denoiser) else _host_wrap_array_fn(denoiser, None)

    if problem.device_gradient is not None:
        grad_fn = problem.device_gradient
    else:
        host_grad = _host_wrap_array_fn(problem.gradient, None)

        def grad_fn(xt, out, data_out):
            out.copy_(host_grad(xt))
            if data_out is not None and problem.objective is not None:
                data_out.fill_(float(problem.objective(xt.cpu().numpy().astype(np.float64))))
            return out

    track_obj = problem.device_gradient is not None or problem.objective is not None
    gt = None
    if problem.ground_truth is not None:
        gt = A.to_device(problem.ground_truth, dev)
        if tuple(gt.shape) != tuple(x.shape):
            raise ValueError("ground_truth shape differs from x0")

    iters = config.max_iters
    stats = torch.zeros((iters, B, 4), dtype=torch.float64, device=x.device)
    objv = torch.full((iters + 1, B), math.nan, dtype=torch.float64, device=x.device)
    flags = torch.zeros(iters, dtype=torch.int32, device=x.device)
    grad = torch.empty_like(x)
    z = torch.empty_like(x)
    mu = 1.0 / (config.alpha + config.rho)
    events = [None] * (iters + 1)  # created on demand (the C++ loop keeps its own)

    def _event(k):
        if events[k] is None:
            events[k] = torch.cuda.Event(enable_timing=True)
        return events[k]

    L.call("pnp_project", ctx, L.ptr(x), L.ptr(x), x.numel(), lo, hi)
    v = x.clone()
    u = torch.zeros_like(x)
    sync_each = callback is not None or config.stop_tol is not None
    gfrom = _graph_from(den)
    k_cap = iters + 1  # first captured iteration (none by default)
    if (graph and not sync_each and gfrom is not None
            and problem.device_gradient is not None):
        if graph and iters - max(gfrom, 2) + 1 >= 3:
            k_cap = max(gfrom, 2)
    t0 = time.perf_counter()
    _event(0).record()
    done = iters
    state = {"x": x, "v": v, "u": u}

    fused_grad = problem.device_grad_xupdate
    frozen_for = getattr(den, "_pnp_frozen_for", None)

    def step(k, record):
        x, v, u = state["x"], state["v"], state["u"]
        fk = flags[k - 1:k]
        # objective of the previous (projected) iterate rides on this gradient
        obj = objv[k - 2] if (k >= 2 and track_obj) else None
        if fused_grad is not None:  # grad + x-update in one kernel epilogue
            fused_grad(x, v, u, z, mu, float(config.alpha), float(config.rho), lo, hi, fk, obj)
        else:
            grad_fn(x, grad, obj)
            L.call("pnp_admm_xupdate", ctx, L.ptr(x), L.ptr(v), L.ptr(u), L.ptr(grad), L.ptr(z),
                   x.numel(), mu, float(config.alpha), float(config.rho), lo, hi, L.ptr(fk))
        v_prev = v
        fz = frozen_for(k) if frozen_for is not None else None
        if fz is not None:  # frozen apply + u-update in one fixup epilogue
            v = torch.empty_like(x)
            fz.apply_admm(z, v, u, x, v_prev, gt, float(config.rho), stats[k - 1], fk)
        else:
            v = den(z, k)
            if not isinstance(v, torch.Tensor) or v.dtype != torch.float32 or not v.is_contiguous():
                v = A.to_device(v, dev).reshape(x.shape)
            if v.data_ptr() in (z.data_ptr(), x.data_ptr(), u.data_ptr(), v_prev.data_ptr()):
                v = v.clone()  # a plug-in may hand back its input; iterates must not alias
            L.call("pnp_admm_uupdate", ctx, L.ptr(u), L.ptr(x), L.ptr(v), L.ptr(v_prev),
                   L.ptr(gt), B, n, float(config.rho), L.ptr(stats[k - 1]), L.ptr(fk))
        state["v"] = v
        if record:
            _event(k).record()

    # Native loop: once the denoiser is a frozen guide (from its first frozen
    # iteration on) and nothing needs the host between iterations, the
    # remaining iterations run in C++ (pnp_admm_run): the same two fused calls
    # per iteration with the same arguments -> bitwise-identical iterates, no
    # interpreter cost per iteration.
    native_spec = problem.native_grad if native else None
    if sync_each or k_cap <= iters or frozen_for is None or fused_grad is None:
        native_spec = None
    native_times = None

    def run_native(k, fzk):
        nk = native_spec
        v_cur = state["v"]
        v_other = torch.empty_like(x)
        ms = (C.c_float * (iters - k + 1))()
        vlast = C.c_int(0)
        L.call("pnp_admm_run", ctx, nk[0], L.ptr(nk[1]), L.ptr(nk[2]), B, H, W, nk[3], nk[4],
               nk[5], nk[6], float(nk[7]), float(nk[8]), fzk._h, k, iters, L.ptr(state["x"]),
               L.ptr(v_cur), L.ptr(v_other), L.ptr(state["u"]), L.ptr(z), L.ptr(gt), mu,
               float(config.alpha), float(config.rho), lo, hi, L.ptr(stats),
               L.ptr(objv) if track_obj else None, L.ptr(flags), ms, C.byref(vlast))
        state["v"] = v_other if vlast.value else v_cur
        return list(ms)

    for k in range(1, iters + 1):
        if native_spec is not None:
            fzk = frozen_for(k)
            if fzk is not None and getattr(fzk, "_dev", dev) == dev:
                native_times = (k, run_native(k, fzk))
                for kk in range(k, iters + 1):
                    events[kk] = None
                break
        if k == k_cap:  # capture the remaining iterations once, replay once
            # raw capture on a side stream (torch.cuda.graph would also run
            # gc.collect + empty_cache on every call)
            g = torch.cuda.CUDAGraph()
            cur = torch.cuda.current_stream(dev)
            side = torch.cuda.Stream(dev)
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                g.capture_begin()
                try:
                    for kk in range(k, iters + 1):
                        step(kk, False)
                finally:
                    g.capture_end()
            cur.wait_stream(side)
            g.replay()
            _event(iters).record()
            for kk in range(k, iters):
                events[kk] = None
            break
        step(k, True)
        x, v, u = state["x"], state["v"], state["u"]
        if sync_each:
            if int(flags[k - 1]):
                raise DivergenceError(f"non-finite iterate at iteration {k}")
            if callback is not None:
                if _is_device(callback):
                    callback(k, x, v, u)
                else:
                    callback(k, *(A.from_device(t.clone(), A.NUMPY) for t in (x, v, u)))
            if config.stop_tol is not None:
                s = stats[k - 1, 0].cpu()
                primal, dual = float(s[0]) / n, float(s[1]) / n
                if primal < config.stop_tol and dual < config.stop_tol:
                    done = k
                    break
    x, v, u = state["x"], state["v"], state["u"]
    if track_obj:  # objective at the final iterate
        grad_fn(x, grad, objv[done - 1])
    # one device->host read for flags, stats and objectives (it also waits
    # for the loop, so the timing events below are complete)
    packed = torch.cat([flags[:done].to(torch.float64), stats[:done].reshape(-1),
                        objv[:done].reshape(-1)]).cpu().numpy()
    fl = packed[:done]
    bad = np.nonzero(fl)[0]
    if bad.size:
        raise DivergenceError(f"non-finite iterate at iteration {int(bad[0]) + 1}")
    st = packed[done:done + done * B * 4].reshape(done, B, 4)
    ob = packed[done + done * B * 4:].reshape(done, B)
    wall = (time.perf_counter() - t0) * 1e3
    times = [events[0].elapsed_time(events[k]) if events[k] is not None else math.nan
             for k in range(1, done + 1)]
    if native_times is not None:  # C++ loop: its own per-iteration events
        k_n, ms = native_times
        base = events[0].elapsed_time(events[k_n - 1]) if k_n > 1 else 0.0
        for i, t in enumerate(ms):
            times[k_n - 1 + i] = base + float(t)
    if k_cap <= done:  # captured iterations: spread the replay time evenly
        t_a = times[k_cap - 2] if k_cap >= 2 else 0.0
        t_b = times[done - 1]
        for i in range(k_cap - 1, done):
            times[i] = t_a + (t_b - t_a) * (i - k_cap + 2) / (done - k_cap + 1)
    # per-iteration log, vectorized over the iterations (host cost ~ constant)
    prim = st[:done, :, 0] / n
    dual = st[:done, :, 1] / n
    if gt is not None:
        mse = st[:done, :, 2] / n
        q = np.where(mse == 0.0, math.inf, 10.0 * np.log10(1.0 / np.where(mse == 0, 1, mse)))
    else:
        q = np.full((done, B), math.nan)
    objs = ob[:done] if track_obj else np.full((done, B), math.nan)
    if B == 1 and x.dim() == 2:
        records = [IterationRecord(i + 1, p_, d_, q_, float(t_), o_) for i, (p_, d_, q_, t_, o_)
                   in enumerate(zip(prim[:, 0].tolist(), dual[:, 0].tolist(), q[:, 0].tolist(),
                                    times, objs[:, 0].tolist()))]
    else:
        records = [IterationRecord(i + 1, prim[i], dual[i], q[i], float(times[i]), objs[i])
                   for i in range(done)]
    del wall
    return A.from_device(v, kind), records


# ---------------------------------------------------------------------------
# Standard PnP-ADMM + CG baseline (solver.py:285-328)
# ---------------------------------------------------------------------------

def standard_pnp_admm_cg(problem: Problem, config: SolverConfig, denoiser=None, callback=None):
    """Standard PnP-ADMM: the exact quadratic x-update
    (A^T A + rho I) x = A^T y + rho (v - u) by conjugate gradients each
    iteration (from scratch unless config.cg_warm_start); the constraint is
    applied once, to the returned v.  Returns (v, records).

    SR problems built by make_sr_problem solve the x-update with the native
    batched CG (device scalars, no per-iteration host round trip); other
    problems use cg_solve on their ``gram`` operator.
    """
    if problem.gram is None or problem.atb is None:
        raise ValueError("standard ADMM baseline needs problem.gram and problem.atb")
    dev = A.device_index()
    x0, kind = A.validate(problem.x0, "x0", batch_ok=True)
    x = A.to_device(x0, dev).clone()
    B, H, W = A.dims(x)
    n = H * W
    lo, hi = bounds(config.constraint)
    ctx = L.context(dev)
    rho = float(config.rho)
    if denoiser is None:
        denoiser = _make_denoiser(config)
    den = denoiser if _is_device(denoiser) else _host_wrap_array_fn(denoiser, None)
    atb = problem.device_atb if problem.device_atb is not None else A.to_device(problem.atb, dev)
    native = problem.device_cg
    if native is None:
        host_gram = _host_wrap_array_fn(problem.gram, None)
        op = lambda z: host_gram(z) + rho * z  # noqa: E731
    gt = A.to_device(problem.ground_truth, dev) if problem.ground_truth is not None else None
    track_obj = problem.device_gradient is not None or problem.objective is not None
    iters = config.max_iters
    stats = torch.zeros((iters, B, 4), dtype=torch.float64, device=x.device)
    objv = torch.full((iters, B), math.nan, dtype=torch.float64, device=x.device)
    flags = torch.zeros(iters, dtype=torch.int32, device=x.device)
    rhs, z, scratch = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    v = x.clone()
    u = torch.zeros_like(x)
    t0 = time.perf_counter()
    times = []
    done = iters
    for k in range(1, iters + 1):
        fk = flags[k - 1:k]
        L.call("pnp_admm_std_rhs", ctx, L.ptr(rhs), L.ptr(atb), L.ptr(v), L.ptr(u), x.numel(), rho)
        if native is not None:
            _, _, status = native(rhs, x, rho, config.cg_tol, config.cg_max_iters,
                                  config.cg_warm_start)
            if any(st_ == 3 for st_ in status):
                raise DivergenceError("non-finite value inside conjugate gradients")
            if any(st_ == 2 for st_ in status):
                raise CgBreakdownError("nonpositive curvature inside conjugate gradients")
        else:
            x = cg_solve(op, rhs, config.cg_tol, config.cg_max_iters,
                         x0=x if config.cg_warm_start else None).x.contiguous()
        L.call("pnp_admm_std_z", ctx, L.ptr(z), L.ptr(x), L.ptr(u), x.numel(), L.ptr(fk))
        v_prev = v
        v = den(z, k)
        if not isinstance(v, torch.Tensor) or v.dtype != torch.float32 or not v.is_contiguous():
            v = A.to_device(v, dev).reshape(x.shape)
        if v.data_ptr() in (z.data_ptr(), x.data_ptr(), u.data_ptr(), v_prev.data_ptr()):
            v = v.clone()
        L.call("pnp_admm_uupdate", ctx, L.ptr(u), L.ptr(x), L.ptr(v), L.ptr(v_prev), L.ptr(gt),
               B, n, rho, L.ptr(stats[k - 1]), L.ptr(fk))
        if track_obj:
            if problem.device_gradient is not None:
                problem.device_gradient(x, scratch, objv[k - 1])
            else:
                objv[k - 1].fill_(float(problem.objective(x.cpu().numpy().astype(np.float64))))
        if int(flags[k - 1]):  # the reference checks after every step (solver.py:316-321)
            raise DivergenceError(f"non-finite iterate at iteration {k}")
        times.append((time.perf_counter() - t0) * 1e3)
        if callback is not None:
            if _is_device(callback):
                callback(k, x, v, u)
            else:
                callback(k, *(A.from_device(t.clone(), A.NUMPY) for t in (x, v, u)))
        if config.stop_tol is not None:
            s_ = stats[k - 1, 0].cpu()
            if float(s_[0]) / n < config.stop_tol and float(s_[1]) / n < config.stop_tol:
                done = k
                break
    st = stats[:done].cpu().numpy()
    ob = objv[:done].cpu().numpy()
    records = []
    for i in range(done):
        primal, dual = st[i, :, 0] / n, st[i, :, 1] / n
        if gt is not None:
            mse = st[i, :, 2] / n
            q = np.where(mse == 0.0, math.inf, 10.0 * np.log10(1.0 / np.where(mse == 0, 1, mse)))
        else:
            q = np.full(B, math.nan)
        obj = ob[i] if track_obj else np.full(B, math.nan)
        if B == 1 and x.dim() == 2:
            records.append(IterationRecord(i + 1, float(primal[0]), float(dual[0]), float(q[0]),
                                           times[i], float(obj[0])))
        else:
            records.append(IterationRecord(i + 1, primal, dual, q, times[i], obj))
    out = torch.empty_like(v)
    L.call("pnp_project", ctx, L.ptr(v), L.ptr(out), v.numel(), lo, hi)
    return A.from_device(out, kind), records


# ---------------------------------------------------------------------------
# Problem builders
# ---------------------------------------------------------------------------

def make_sr_problem(op: SuperResOp, observed, ground_truth=None) -> Problem:
    """SR problem; x0 = k^2 A^T y (solver.py:335-349).  Device resident."""
    obs, kind = A.validate(observed, "observation", batch_ok=True)
    y = A.to_device(obs)
    x0d = float(op.factor ** 2) * op.adjoint_device(y)
    x0 = A.from_device(x0d, kind)

    def device_gradient(x, out, data_out=None):
        return op.gradient_device(x, y, out, data_out)

    def device_grad_xupdate(x, v, u, z, mu, alpha, rho, lo, hi, flags, data_out=None):
        op.gradient_xupdate_device(x, y, v, u, z, mu, alpha, rho, lo, hi, flags, data_out)

    def device_cg(rhs, x, shift, tol, max_iters, warm):
        return op.cg_device(rhs, x, shift, tol, max_iters, warm)

    def gradient(x):
        from .forward import sr_gradient
        return sr_gradient(op, x, A.from_device(y, A.kind_of(x)))

    def objective(x):
        from .forward import sr_data_term
        return sr_data_term(op, x, A.from_device(y, A.kind_of(x)))

    def gram(x):
        from .forward import sr_apply
        return sr_adjoint(op, sr_apply(op, x))

    return Problem(shape=tuple(x0d.shape), gradient=gradient, x0=x0, objective=objective,
                   ground_truth=ground_truth, gram=gram,
                   atb=A.from_device(op.adjoint_device(y), kind),
                   device_gradient=device_gradient, device_grad_xupdate=device_grad_xupdate,
                   device_cg=device_cg, device_atb=op.adjoint_device(y),
                   native_grad=(0, y, None, op._taps, op.radius, op.factor, op._bnd, 0.0, 0.0))


def make_qis_problem(counts: QisCounts, model: QisModel, ground_truth=None,
                     floor: float = QIS_FLOOR) -> Problem:
    """QIS problem; x0 = clip(K1/K, floor, 1) (solver.py:352-362)."""
    ones, zeros = counts.device()
    if counts.oversampling != model.oversampling:
        raise ValueError(f"counts are for K={counts.oversampling}, model has K={model.oversampling}")

    def device_gradient(x, out, data_out=None):
        return qis_grad_device(x, ones, zeros, model, floor, out, data_out)

    def device_grad_xupdate(x, v, u, z, mu, alpha, rho, lo, hi, flags, data_out=None):
        qis_grad_xupdate_device(x, ones, zeros, model, floor, v, u, z, mu, alpha, rho, lo, hi,
                                flags, data_out)

    def gradient(x):
        from .forward import qis_gradient
        return qis_gradient(x, counts, model, floor)

    def objective(x):
        from .forward import qis_data_term
        return qis_data_term(x, counts, model, floor)

    return Problem(shape=counts.shape, gradient=gradient, x0=qis_initial_estimate(counts, floor),
                   objective=objective, ground_truth=ground_truth,
                   device_gradient=device_gradient, device_grad_xupdate=device_grad_xupdate,
                   native_grad=(1, ones, zeros, None, 0, 0, 0,
                                model.gain / model.oversampling, float(floor)))


def default_sr_alpha(op: SuperResOp, hr_shape, iters: int = 200, seed: int = 0) -> float:
    """1.05 x the power-iteration Lipschitz estimate (solver.py:365-368)."""
    return 1.05 * power_iteration_lipschitz(op, hr_shape, iters, seed)


def default_qis_alpha(counts: QisCounts, model: QisModel) -> float:
    """2 * gain * max(K0) / K (solver.py:371-374)."""
    return 2.0 * model.gain * float(counts.zeros.max()) / model.oversampling
