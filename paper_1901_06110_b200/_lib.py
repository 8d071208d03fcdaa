"""ctypes binding of libpnpb200.so (C ABI in include/pnp_b200.h).

The native library is REQUIRED: there is no CPU fallback.  Importing the
package loads it (no GPU needed to load); calling a kernel without a CUDA
device raises RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# PNP_B200_LIB: development override to A/B a variant build of the same ABI
# (scripts/build_variant.py); the in-tree library is the product.
_VARIANT = os.environ.get("PNP_B200_LIB")
LIB_PATH = Path(_VARIANT) if _VARIANT else _PKG / "libpnpb200.so"

if not LIB_PATH.exists():  # fail loudly: the CUDA path is the product
    raise ImportError(
        f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        " or `python paper_1901_06110_b200/build.py`")

lib = C.CDLL(str(LIB_PATH))

vp = C.c_void_p
i32 = C.c_int
i64 = C.c_int64
f64 = C.c_double
fptr = C.POINTER(C.c_float)

_SIGS = {
    "pnp_version": (i32, []),
    "pnp_last_error": (C.c_char_p, []),
    "pnp_ctx_create": (i32, [i32, C.POINTER(vp)]),
    "pnp_ctx_destroy": (i32, [vp]),
    "pnp_ctx_set_stream": (i32, [vp, vp]),
    "pnp_ctx_synchronize": (i32, [vp]),
    "pnp_ctx_reserve": (i32, [vp, i32, i32, i32, i32, i32, i32]),
    "pnp_ctx_set_cache_limit": (i32, [vp, i64]),
    "pnp_ctx_bind_kcache": (i32, [vp, vp, i64]),
    "pnp_ctx_trim": (i32, [vp]),
    "pnp_frozen_cached": (i32, [vp]),
    "pnp_ctx_profile": (i32, [vp, i32]),
    "pnp_ctx_profile_read": (i32, [vp, C.POINTER(f64), C.POINTER(i32)]),
    "pnp_peak_rates": (i32, [i32, C.POINTER(f64), C.POINTER(f64)]),
    "pnp_dsg_denoise": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, fptr, f64, vp, vp]),
    "pnp_dsg_denoise_direct": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, fptr, f64]),
    "pnp_dsg_freeze": (i32, [vp, vp, i32, i32, i32, i32, i32, fptr, f64, C.POINTER(vp)]),
    "pnp_dsg_apply": (i32, [vp, vp, vp, vp]),
    "pnp_frozen_destroy": (i32, [vp]),
    "pnp_frozen_alpha": (i32, [vp, fptr]),
    "pnp_frozen_export": (i32, [vp, vp, vp, vp]),
    "pnp_frozen_shape": (i32, [vp] + [C.POINTER(i32)] * 5),
    "pnp_frozen_cache": (i32, [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(C.c_ulonglong)]),
    "pnp_nlm_denoise": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, fptr, f64]),
    "pnp_dsg_geometry": (i32, [i32, i32, i32, i32, i32, C.POINTER(i32)]),
    "pnp_dsg_groups": (i32, [i32, i32, i32, i32, i32]),
    "pnp_dsg_partial_floats": (i64, [i32, i32, i32, i32, i32, i32, i32]),
    "pnp_dsg_kcache_floats": (i64, [i32, i32, i32, i32, i32, i32]),
    "pnp_dsg_strip_sweep": (i32, [vp, i32, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32,
                                  fptr, f64, vp, i32, i32, vp]),
    "pnp_dsg_strip_fixup": (i32, [vp, i32, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                  i32, vp, vp, vp, vp, vp, vp, vp]),
    "pnp_dsg_strip_finalize": (i32, [vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32]),
    "pnp_sr_apply": (i32, [vp, vp, vp, i32, i32, i32, fptr, i32, i32, i32]),
    "pnp_sr_adjoint": (i32, [vp, vp, vp, i32, i32, i32, fptr, i32, i32, i32]),
    "pnp_sr_grad": (i32, [vp, vp, vp, vp, i32, i32, i32, fptr, i32, i32, i32, vp]),
    "pnp_qis_grad": (i32, [vp, vp, vp, vp, vp, i32, i32, f64, f64, vp]),
    "pnp_qis_data": (i32, [vp, vp, vp, vp, i32, i32, f64, f64, vp]),
    "pnp_qis_simulate_host": (i32, [vp, i64, i32, C.c_uint64, vp]),
    "pnp_admm_xupdate": (i32, [vp, vp, vp, vp, vp, vp, i64, f64, f64, f64, f64, f64, vp]),
    "pnp_admm_uupdate": (i32, [vp, vp, vp, vp, vp, vp, i32, i64, f64, vp, vp]),
    "pnp_project": (i32, [vp, vp, vp, i64, f64, f64]),
    "pnp_sr_grad_xupdate": (i32, [vp, vp, vp, i32, i32, i32, fptr, i32, i32, i32, vp,
                                  vp, vp, vp, f64, f64, f64, f64, f64, vp]),
    "pnp_qis_grad_xupdate": (i32, [vp, vp, vp, vp, i32, i32, f64, f64, vp,
                                   vp, vp, vp, f64, f64, f64, f64, f64, vp]),
    "pnp_dsg_apply_admm": (i32, [vp, vp, vp, vp, vp, vp, vp, vp, f64, vp, vp]),
    "pnp_sr_gram": (i32, [vp, vp, vp, i32, i32, i32, fptr, i32, i32, i32, f64]),
    "pnp_admm_std_rhs": (i32, [vp, vp, vp, vp, vp, i64, f64]),
    "pnp_sr_strip_residual": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, fptr, i32, i32,
                                    i32, vp]),
    "pnp_sr_strip_adjoint": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, i32, fptr, i32, i32,
                                   i32]),
    "pnp_admm_std_z": (i32, [vp, vp, vp, vp, i64, vp]),
    "pnp_sr_cg": (i32, [vp, vp, vp, i32, i32, i32, fptr, i32, i32, i32, f64, f64, i32, i32,
                        C.POINTER(i32), C.POINTER(f64), C.POINTER(i32)]),
    "pnp_check_finite": (i32, [vp, vp, i64, C.POINTER(i32)]),
    "pnp_host_cast_f32_f64": (i32, [vp, vp, i64, i32]),
    "pnp_host_cast_f64_f32": (i32, [vp, vp, i64, i32]),
    "pnp_host_zero_f64": (i32, [vp, i64, i32]),
    "pnp_flag_nonfinite": (i32, [vp, vp, i64, vp]),
    "pnp_splitmix_uniforms": (i32, [vp, C.c_uint64, i64, vp]),
    "pnp_pad_symmetric_f64": (i32, [vp, vp, i32, i32, i32, vp]),
    "pnp_integral_image_f64": (i32, [vp, vp, i32, i32, vp]),
    "pnp_patch_distance_map_f64": (i32, [vp, vp, i32, i32, i32, i32, i32, i32, vp]),
    "pnp_patch_ssd_pairs_f64": (i32, [vp, vp, i32, i32, i32, vp, i32, vp]),
    "pnp_dense_weights_f64": (i32, [vp, vp, i32, i32, i32, i32, f64, vp, vp]),
    "pnp_dsg_band_rows": (i32, [i32, i32, i32, i32, i32, i32, C.POINTER(i32), C.POINTER(i32)]),
    "pnp_dsg_denoise_banded": (i32, [vp, vp, vp, i32, i32, i32, i32, fptr, f64, i32,
                                     C.POINTER(vp)]),
    "pnp_dsg_band_sweep": (i32, [vp, vp, i32, i32, i32, i32, fptr, f64, i32, i32]),
    "pnp_dsg_band_finish": (i32, [vp, vp, vp, i32, i32, i32, i32, fptr, f64]),
    "pnp_admm_run": (i32, [vp, i32, vp, vp, i32, i32, i32, fptr, i32, i32, i32, f64, f64, vp,
                           i32, i32, vp, vp, vp, vp, vp, vp, f64, f64, f64, f64, f64, vp, vp, vp,
                           C.POINTER(C.c_float), C.POINTER(i32)]),
    "pnp_sr_add_noise": (i32, [vp, vp, i64, C.c_uint64, f64, vp, vp]),
}

EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    if _VARIANT and not hasattr(lib, _name):
        continue
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

PNP_OK, PNP_EINVAL, PNP_ECUDA, PNP_ENONFINITE, PNP_ENCCL = 0, 1, 2, 3, 4


class NativeError(RuntimeError):
    """Error reported by the native library (CUDA / NCCL failure)."""


def check(rc: int) -> None:
    if rc == PNP_OK:
        return
    msg = lib.pnp_last_error().decode(errors="replace")
    if rc in (PNP_EINVAL, PNP_ENONFINITE):
        raise ValueError(msg)
    raise NativeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args))


def ptr(t) -> vp:
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else vp(t.data_ptr())


_GEOM: dict = {}


def dsg_geometry(Hg: int, W: int, R: int, P: int, box: bool) -> tuple:
    """pnp_dsg_geometry: (TH, offset groups, block band Rb, sweep path, input
    halo above, input halo below, channel rows read below, 0)."""
    key = (Hg, W, R, P, bool(box))
    g = _GEOM.get(key)
    if g is None:
        out = (C.c_int * 8)()
        check(lib.pnp_dsg_geometry(Hg, W, R, P, int(bool(box)), out))
        g = _GEOM[key] = tuple(out)
    return g


def host_floats(values) -> C.Array:
    arr = (C.c_float * len(values))(*[float(v) for v in values])
    return arr


_tls = threading.local()
# k-cache budget per device as set through profiling.set_cache_limit
# (None: no limit, 0: disabled) -- the Python layer sizes the torch buffer
# it binds for each adaptive call from it
cache_limits: dict = {}


class _Ctx:
    """Owns one native context; destroyed when its thread's local storage
    goes away (thread exit) or at interpreter shutdown."""

    __slots__ = ("h",)

    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h and lib is not None:
                lib.pnp_ctx_destroy(self.h)
        except Exception:  # interpreter shutdown
            pass
        self.h = None


def _raw_stream(device: int) -> int:
    import torch

    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:  # no Stream object per call (this sits on every launch path)
        return int(get(device))
    return int(torch.cuda.current_stream(device).cuda_stream)


def context(device: int):
    """Per-(thread, device) native context, bound to torch's current stream
    (re-bound only when the current stream changed)."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ent = ctxs.get(device)
    if ent is None:
        h = vp()
        check(lib.pnp_ctx_create(device, C.byref(h)))
        ent = ctxs[device] = [_Ctx(h), None]
        lim = cache_limits.get(device, None)
        if lim is not None:
            check(lib.pnp_ctx_set_cache_limit(h, int(lim)))
    stream = _raw_stream(device)
    if stream != ent[1]:
        check(lib.pnp_ctx_set_stream(ent[0].h, vp(stream)))
        ent[1] = stream
    return ent[0].h
