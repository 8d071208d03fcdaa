"""Time the UNMODIFIED reference on the host cores — BENCH INFRASTRUCTURE ONLY.

Used by ``bench.py --impl reference`` (all host cores, one process per core)
and by the GPU arm's ``cpu_baseline`` leg (one core).  It imports
``pnprestore`` from ``oracle/_ref`` (installed from /root/reference/pkg by
oracle/build_ref.py) and calls its public ``dsg_nlm_denoise``
(denoise.py:272-288) as shipped: box patch weights, summed-area-table
distance engine, the three sweeps of denoise.py:207-241, kernel-map
memoization only under KERNEL_CACHE_BYTES (denoise.py:27-29).  Nothing of
this repo's package (and none of its .so files) is loaded here.

When oracle/_ref is missing the float64 port in oracle/dsg.py stands in and
the result says ``kind = "port"``.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = HERE / "_ref"


def available() -> bool:
    return (REF / "pnprestore" / "denoise.py").exists()


def _reference():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import pnprestore
    assert Path(pnprestore.__file__).resolve().is_relative_to(REF.resolve()), pnprestore.__file__
    return pnprestore


def kind() -> str:
    return "reference" if available() else "port"


def denoise_job(job):
    """(crop, P, R, bandwidth) -> (pixel-offsets, seconds) of one
    dsg_nlm_denoise call on a float64 copy of the crop (guide = image)."""
    crop, P, R, bw = job
    x = np.asarray(crop, dtype=np.float64)
    if available():
        ref = _reference()
        params = ref.PatchParams(P, R, bw)
        t = time.perf_counter()
        ref.dsg_nlm_denoise(x, params)
        dt = time.perf_counter() - t
    else:
        from . import dsg
        t = time.perf_counter()
        dsg.dsg_nlm_denoise(x, P, R, bw)
        dt = time.perf_counter() - t
    return x.size * (2 * R + 1) ** 2, dt


def uncached_side(R: int) -> int:
    """Smallest square crop whose kernel maps exceed KERNEL_CACHE_BYTES, so the
    reference recomputes them in every sweep, as it must at 8192^2."""
    n_off = (2 * R + 1) ** 2
    s = 16
    while n_off * s * s * 8 <= (1 << 30):
        s += 8
    return s
