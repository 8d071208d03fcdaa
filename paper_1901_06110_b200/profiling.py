"""Live kernel timing (CUDA events on the library's stream) and measured
FP32/SFU peaks — the numbers bench.py's roofline object is built from."""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L

CATEGORIES = ("sweep", "fixup", "forward", "admm", "sweep_cached", "check")


def enable(flag: bool = True, device: int | None = None) -> None:
    dev = torch.cuda.current_device() if device is None else device
    L.call("pnp_ctx_profile", L.context(dev), 1 if flag else 0)


def read(device: int | None = None) -> dict:
    """{category: (device ms, launches)} since the last read (syncs the stream)."""
    dev = torch.cuda.current_device() if device is None else device
    ms = (C.c_double * len(CATEGORIES))()
    n = (C.c_int * len(CATEGORIES))()
    L.call("pnp_ctx_profile_read", L.context(dev), ms, n)
    return {c: (float(ms[i]), int(n[i])) for i, c in enumerate(CATEGORIES)}


def set_cache_limit(nbytes: int | None, device: int | None = None) -> None:
    """k-cache budget in bytes (None: unlimited, 0: disabled)."""
    dev = torch.cuda.current_device() if device is None else device
    L.cache_limits[dev] = None if nbytes is None else int(nbytes)
    L.call("pnp_ctx_set_cache_limit", L.context(dev), -1 if nbytes is None else int(nbytes))


def trim(device: int | None = None) -> None:
    """Return the idle memory of the device's stream-ordered pool (frozen
    guides' buffers after their handles died) to the device."""
    dev = torch.cuda.current_device() if device is None else device
    L.call("pnp_ctx_trim", L.context(dev))


def peak_rates(device: int | None = None) -> tuple[float, float]:
    """Measured (FFMA/s, MUFU.EX2/s) of the whole GPU."""
    dev = torch.cuda.current_device() if device is None else device
    f, x = C.c_double(), C.c_double()
    L.call("pnp_peak_rates", dev, C.byref(f), C.byref(x))
    return f.value, x.value

