"""Host/device array plumbing for the drop-in API.

The reference (pnprestore) takes and returns float64 numpy images.  This
package accepts numpy arrays (drop-in: result comes back as float64 numpy)
or torch tensors (device-resident: result stays a float32 CUDA tensor).
Validation follows image.py:32-41 (2-D, non-empty, finite -> ValueError).
"""

from __future__ import annotations

import threading

import numpy as np
import torch

NUMPY, TORCH = "numpy", "torch"

# numpy arrays of at least this many elements move through pinned staging
# buffers with multi-threaded dtype casts (a pageable 256 MB copy plus
# single-threaded numpy casts cost ~0.4 s at 8192^2, 16x the denoise itself)
_BIG = 1 << 20


def _host_tensor(a: np.ndarray) -> torch.Tensor:
    """Zero-copy torch view of a host array (read-only arrays included)."""
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(np.ascontiguousarray(a))


def device_index() -> int:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1901_06110_b200 needs a CUDA device (B200); none is visible")
    return torch.cuda.current_device()


def kind_of(a) -> str:
    return TORCH if isinstance(a, torch.Tensor) else NUMPY


def validate(a, name: str = "image", batch_ok: bool = False):
    """Shape/finiteness checks; returns (array_or_tensor, kind)."""
    kind = kind_of(a)
    if kind == NUMPY:
        a = np.asarray(a, dtype=np.float64)
        shape = a.shape
        if a.size >= _BIG:  # one multi-threaded reduction (NaN / inf propagate)
            lo, hi = torch.aminmax(_host_tensor(a))
            finite = bool(torch.isfinite(lo)) and bool(torch.isfinite(hi))
        else:
            finite = bool(np.all(np.isfinite(a)))
    else:
        shape = tuple(a.shape)
        finite = _all_finite(a) if a.numel() else True
    nd_ok = len(shape) == 2 or (batch_ok and kind == TORCH and len(shape) == 3)
    if not nd_ok:
        raise ValueError(f"{name} must be 2-D, got shape {shape}")
    if shape[-2] < 1 or shape[-1] < 1 or (len(shape) == 3 and shape[0] < 1):
        raise ValueError(f"{name} must be at least 1x1, got shape {shape}")
    if not finite:
        raise ValueError(f"{name} contains non-finite values")
    return a, kind


def _all_finite(t: torch.Tensor) -> bool:
    """Native one-pass check for contiguous float32 CUDA tensors (no torch
    reduction kernels); torch for anything else."""
    if t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.data_ptr() % 16 == 0:
        import ctypes as C

        from . import _lib as L
        ok = C.c_int(0)
        L.call("pnp_check_finite", L.context(t.device.index), L.ptr(t), t.numel(), C.byref(ok))
        return bool(ok.value)
    return bool(torch.isfinite(t).all().item())


def to_device(a, dev: int | None = None) -> torch.Tensor:
    """float32, contiguous, on the current CUDA device (copy only if needed)."""
    if dev is None:
        dev = device_index()
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if t.dtype != torch.float32 or t.device != torch.device("cuda", dev):
            t = t.to(device=torch.device("cuda", dev), dtype=torch.float32)
        return t.contiguous()
    arr = np.asarray(a)
    if arr.size >= _BIG and arr.dtype.kind == "f":
        # multi-threaded cast into pinned staging, then a DMA copy (the caching
        # host allocator keeps the staging block until the copy completes)
        stage = torch.empty(arr.shape, dtype=torch.float32, pin_memory=True)
        cast_into(stage, _host_tensor(arr))
        return stage.to(torch.device("cuda", dev), non_blocking=True)
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    return torch.from_numpy(arr).to(torch.device("cuda", dev), non_blocking=False)


def to_device64(a, dev: int | None = None) -> torch.Tensor:
    """float64, contiguous, on the CUDA device (the float64 helper kernels)."""
    if dev is None:
        dev = device_index()
    if isinstance(a, torch.Tensor):
        return a.detach().to(device=torch.device("cuda", dev), dtype=torch.float64).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return torch.from_numpy(arr).to(torch.device("cuda", dev))


def from_device64(t: torch.Tensor, kind: str):
    """float64 device result -> float64 numpy (drop-in) or the tensor."""
    return t if kind == TORCH else t.cpu().numpy()


_stage_lock = threading.Lock()
_stage_buf: list = [None]


def _pinned_f32(n: int) -> torch.Tensor:
    """Grow-only pinned float32 staging buffer (allocated once: page-locking
    hundreds of MB per call would cost more than the copy)."""
    buf = _stage_buf[0]
    if buf is None or buf.numel() < n:
        buf = _stage_buf[0] = torch.empty(n, dtype=torch.float32, pin_memory=True)
    return buf[:n]


def cast_into(dst: torch.Tensor, src: torch.Tensor) -> None:
    """dst[...] = src between host tensors: the library's streaming AVX2
    casts for contiguous float32 <-> float64 (the numpy path's casts are host
    memory bound and on the call's critical path), torch's copy otherwise.
    Same bits either way (round to nearest even)."""
    from . import _lib as L

    pair = (src.dtype, dst.dtype)
    if (pair in ((torch.float32, torch.float64), (torch.float64, torch.float32))
            and src.is_contiguous() and dst.is_contiguous() and src.numel() == dst.numel()
            and not src.is_cuda and not dst.is_cuda):
        fn = "pnp_host_cast_f32_f64" if pair[0] == torch.float32 else "pnp_host_cast_f64_f32"
        L.call(fn, src.data_ptr(), dst.data_ptr(), src.numel(), 0)
    else:
        dst.copy_(src)


def from_device(t: torch.Tensor, kind: str):
    if kind == TORCH:
        return t
    if t.numel() >= _BIG:  # one DMA into pinned staging, multi-threaded cast
        out = np.empty(tuple(t.shape), dtype=np.float64)
        src = t.detach().float().contiguous().view(-1)
        with _stage_lock:
            stage = _pinned_f32(src.numel())
            stage.copy_(src)
            cast_into(torch.from_numpy(out).view(-1), stage)
        return out
    return t.detach().to("cpu").numpy().astype(np.float64)


class _Staging:
    """Named grow-only pinned float32 buffers, used under one lock."""

    def __init__(self):
        self.bufs: dict = {}

    def f32(self, name: str, n: int) -> torch.Tensor:
        buf = self.bufs.get(name)
        if buf is None or buf.numel() < n:
            buf = self.bufs[name] = torch.empty(n, dtype=torch.float32, pin_memory=True)
        return buf[:n]


_staging = _Staging()


class staging:
    """``with staging() as st``: exclusive use of the named pinned buffers
    (a call's copies out of / into them complete before the block ends)."""

    def __enter__(self):
        _stage_lock.acquire()
        return _staging

    def __exit__(self, *exc):
        _stage_lock.release()
        return False


_streams: dict = {}


def copy_stream(dev: int, name: str) -> torch.cuda.Stream:
    """A cached side stream per (device, role) for copy-engine transfers."""
    s = _streams.get((dev, name))
    if s is None:
        s = _streams[(dev, name)] = torch.cuda.Stream(torch.device("cuda", dev))
    return s


def download64_banded(t: torch.Tensor, st: _Staging, nbands: int, res=None) -> np.ndarray:
    """float32 device image -> float64 numpy array (``res``, else a new one):
    row bands go down on a copy stream into pinned staging while the host
    casts the bands that already arrived (ordered after the current stream's
    work on ``t``)."""
    H, W = int(t.shape[0]), int(t.shape[1])
    dev = t.device.index
    if res is None:
        res = np.empty((H, W), dtype=np.float64)
    dst = torch.from_numpy(res)
    stage = st.f32("out", H * W).view(H, W)
    d2h = copy_stream(dev, "d2h")
    d2h.wait_stream(torch.cuda.current_stream(t.device))
    rows = [(H * k // nbands, H * (k + 1) // nbands) for k in range(nbands)]
    evs = []
    with torch.cuda.stream(d2h):
        for r0, r1 in rows:
            stage[r0:r1].copy_(t[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(d2h)
            evs.append(ev)
    t.record_stream(d2h)
    for (r0, r1), ev in zip(rows, evs):
        ev.synchronize()
        cast_into(dst[r0:r1], stage[r0:r1])  # multi-threaded streaming cast
    return res


def dims(t: torch.Tensor):
    """(batch, H, W) of a 2-D or 3-D tensor."""
    if t.dim() == 2:
        return 1, int(t.shape[0]), int(t.shape[1])
    return int(t.shape[0]), int(t.shape[1]), int(t.shape[2])
