"""DSG-NLM denoiser — drop-in for pnprestore/denoise.py on the B200.

Public names and semantics follow /root/reference/pkg/src/pnprestore/
denoise.py: ``PatchParams`` (39-58), ``hat_weight`` (61-67),
``dsg_nlm_denoise`` (272-288), ``nlm_denoise`` (254-269), ``FrozenGuide`` /
``freeze_guide`` (358-386).  All arithmetic runs in the sm_100a kernels of
libpnpb200.so (csrc/dsg_sweep.cuh); there is no CPU path.

Extension: ``PatchParams.patch_sigma`` selects Gaussian patch weights (the
BASELINE.json configs); ``None`` keeps the reference's box patch distance.
``PatchParams.from_h(P, R, h, patch_sigma)`` maps the north-star
``exp(-d/h^2)`` bandwidth to the reference's ``bandwidth = h / sqrt(2)``.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _arrays as A
from . import _lib as L


@dataclass(frozen=True)
class PatchParams:
    """Patch side (odd), search-window radius, kernel bandwidth (+ optional
    Gaussian patch-weight sigma)."""

    patch_side: int
    window_radius: int
    bandwidth: float
    patch_sigma: float | None = None

    def __post_init__(self) -> None:
        if self.patch_side < 1 or self.patch_side % 2 == 0:
            raise ValueError(f"patch_side must be odd and >= 1, got {self.patch_side}")
        if self.window_radius < 1:
            raise ValueError(f"window_radius must be >= 1, got {self.window_radius}")
        if not self.bandwidth > 0:
            raise ValueError(f"bandwidth must be > 0, got {self.bandwidth}")
        if self.patch_sigma is not None and not self.patch_sigma > 0:
            raise ValueError(f"patch_sigma must be > 0, got {self.patch_sigma}")

    @property
    def pad_margin(self) -> int:
        return self.window_radius + (self.patch_side - 1) // 2

    @classmethod
    def from_h(cls, patch_side: int, window_radius: int, h: float,
               patch_sigma: float | None = None) -> "PatchParams":
        """North-star bandwidth h (k = exp(-d/h^2)) -> reference bandwidth h/sqrt(2)."""
        return cls(patch_side, window_radius, h / math.sqrt(2.0), patch_sigma)

    def taps(self) -> np.ndarray:
        """Normalized 1-D patch taps (box 1/P, or sampled Gaussian)."""
        P = self.patch_side
        if self.patch_sigma is None:
            return np.full(P, 1.0 / P)
        a = np.arange(P, dtype=np.float64) - (P - 1) // 2
        w = np.exp(-(a * a) / (2.0 * self.patch_sigma ** 2))
        return w / w.sum()

    @property
    def is_box(self) -> bool:
        """The reference's box patch distance (equal taps): the library runs
        it with running-sum box filters, cost flat in P."""
        return self.patch_sigma is None or self.patch_side == 1

    def _ctaps(self):
        return (C.c_float * self.patch_side)(*[float(v) for v in self.taps()])


def hat_weight(s: tuple[int, int], r: tuple[int, int], window_radius: int) -> float:
    """Separable hat taper (reference denoise.py:61-67)."""
    dy, dx = s[0] - r[0], s[1] - r[1]
    if abs(dy) > window_radius or abs(dx) > window_radius:
        raise ValueError(f"offset ({dy},{dx}) outside window radius {window_radius}")
    scale = window_radius + 1
    return (1.0 - abs(dy) / scale) * (1.0 - abs(dx) / scale)


def nlm_kernel(guide, s: tuple[int, int], r: tuple[int, int], params: PatchParams) -> float:
    """exp(-||P_s - P_r||^2 / (2 P^2 bw^2)) for two pixels, patches from the
    mirror-padded guide (denoise.py:70-88); the SSD is a float64 device kernel."""
    guide, _ = A.validate(guide, "guide")
    h, w = int(guide.shape[0]), int(guide.shape[1])
    for name, (py, px) in (("s", s), ("r", r)):
        if not (0 <= py < h and 0 <= px < w):
            raise ValueError(f"pixel {name}={py, px} outside {h}x{w} image")
    half = (params.patch_side - 1) // 2
    if half > min(h, w):
        raise ValueError(f"margin {half} exceeds min image extent {min(h, w)}")
    g = A.to_device64(guide)
    pairs = torch.tensor([s[0], s[1], r[0], r[1]], dtype=torch.int32, device=g.device)
    out = torch.empty(1, dtype=torch.float64, device=g.device)
    L.call("pnp_patch_ssd_pairs_f64", L.context(g.device.index), L.ptr(g), h, w,
           params.patch_side, L.ptr(pairs), 1, L.ptr(out))
    ssd = float(out.item())
    side = params.patch_side
    return float(np.exp(-ssd / (2.0 * side * side * params.bandwidth ** 2)))


def patch_distance_map(guide, offset: tuple[int, int], params: PatchParams,
                       method: str = "integral"):
    """||P_s - P_{s+t}||^2 for every pixel s and one window offset t
    (denoise.py:161-174), float64 on the device.  Both methods are computed
    the reference's "direct" way (exact shifted-add order: bitwise equal to
    method="direct"; within the reference's own 1e-9 agreement of
    method="integral", whose summed-area table only reorders the sums)."""
    if method not in ("integral", "direct"):
        raise ValueError(f"unknown distance method {method!r}")
    guide, kind = A.validate(guide, "guide")
    dy, dx = offset
    if max(abs(dy), abs(dx)) > params.window_radius:
        raise ValueError(f"offset {offset} outside window radius {params.window_radius}")
    h, w = int(guide.shape[0]), int(guide.shape[1])
    _check_margin(params, h, w)
    g = A.to_device64(guide)
    out = torch.empty((h, w), dtype=torch.float64, device=g.device)
    L.call("pnp_patch_distance_map_f64", L.context(g.device.index), L.ptr(g), h, w,
           params.patch_side, params.window_radius, int(dy), int(dx), L.ptr(out))
    return A.from_device64(out, kind)


DENSE_WEIGHTS_MAX_PIXELS = 4096
# the reference memoizes kernel maps below this many bytes (denoise.py:27-29);
# here the analogue is the HBM k cache (profiling.set_cache_limit)
KERNEL_CACHE_BYTES = 1 << 30


def build_dense_weights(guide, params: PatchParams):
    """Explicit n x n doubly stochastic W (test-scale oracle, denoise.py:389-418),
    built on the device in float64 with the reference's literal matrix steps."""
    guide, kind = A.validate(guide, "guide")
    h, w = int(guide.shape[0]), int(guide.shape[1])
    n = h * w
    if n > DENSE_WEIGHTS_MAX_PIXELS:
        raise ValueError(f"{h}x{w} image too large for dense weights (n={n})")
    _check_margin(params, h, w)
    g = A.to_device64(guide)
    out = torch.empty((n, n), dtype=torch.float64, device=g.device)
    scratch = torch.empty(2 * n + 1, dtype=torch.float64, device=g.device)
    L.call("pnp_dense_weights_f64", L.context(g.device.index), L.ptr(g), h, w, params.patch_side,
           params.window_radius, float(params.bandwidth), L.ptr(out), L.ptr(scratch))
    return A.from_device64(out, kind)


_KC_HEADROOM = 4 << 30
# (device, B, H, W, R, P, box, limit) -> bytes granted last time (the
# free-memory query is paid only when a shape is new, the grant was partial,
# or torch could not hand the bytes out again)
_KC_GRANT: dict = {}


def _kcache_bytes(dev: int, B: int, H: int, W: int, params: PatchParams,
                  fresh: bool = False) -> tuple[int, int]:
    """(bytes to bind, bytes of the whole cache).  All tile rows when they fit
    in what torch can hand out (free HBM + its idle cache, less 4 GiB for the
    library's own scratch), else as many as fit (the rest recompute, same
    bits), 0 below 1/8 of them."""
    limit = L.cache_limits.get(dev, None)
    if limit == 0:
        return 0, 0
    key = (dev, B, H, W, params.window_radius, params.patch_side, params.is_box, limit)
    hit = _KC_GRANT.get(key)
    if hit is not None and not fresh and hit[0] == hit[1]:
        return hit
    R = params.window_radius
    geom = L.dsg_geometry(H, W, R, params.patch_side, params.is_box)
    general = geom[3] == 1  # the general half-window sweep: all tile rows or none
    if general:
        row = (2 * R * R + 2 * R) * geom[0] * (-(-W // 64) * 64) * 4 * B
    else:
        row = int(L.lib.pnp_dsg_kcache_floats(H, W, R, params.patch_side,
                                              int(params.is_box), 1)) * 4 * B
    if row <= 0:
        _KC_GRANT[key] = (0, 0)
        return 0, 0
    tiles = -(-H // geom[0])
    free, _ = torch.cuda.mem_get_info(dev)
    idle = torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    budget = free + idle - _KC_HEADROOM
    if limit is not None:
        budget = min(budget, limit)
    rows = min(tiles, max(0, budget) // row)
    n = rows * row if rows * 8 >= tiles and (rows == tiles or not general) else 0
    _KC_GRANT[key] = (n, tiles * row)
    return n, tiles * row


@contextlib.contextmanager
def kcache_scope(dev: int, B: int, H: int, W: int, params: PatchParams):
    """Bind a k cache from torch's caching allocator to this thread's native
    context for one adaptive call (or one DenoiseStream run): torch owns the
    memory, sees it, and recycles it when the scope ends (allocated on the
    current stream, which the context is bound to)."""
    buf = None
    if not torch.cuda.is_current_stream_capturing():
        n, _ = _kcache_bytes(dev, B, H, W, params)
        if n:
            try:
                buf = torch.empty(n, dtype=torch.uint8, device=torch.device("cuda", dev))
            except torch.cuda.OutOfMemoryError:
                n, _ = _kcache_bytes(dev, B, H, W, params, fresh=True)
                try:
                    buf = torch.empty(n, dtype=torch.uint8,
                                      device=torch.device("cuda", dev)) if n else None
                except torch.cuda.OutOfMemoryError:
                    buf = None
    ctx = L.context(dev)
    L.call("pnp_ctx_bind_kcache", ctx, L.ptr(buf), 0 if buf is None else buf.numel())
    try:
        yield buf
    finally:
        L.call("pnp_ctx_bind_kcache", ctx, None, 0)
        del buf


def _pair(image, guide):
    """_check_pair (denoise.py:244-251) -> device tensors + result kind."""
    image, kind = A.validate(image, "image", batch_ok=True)
    dev = A.device_index()
    x = A.to_device(image, dev)
    if guide is None:
        return x, x, kind, dev
    guide, _ = A.validate(guide, "guide", batch_ok=True)
    g = A.to_device(guide, dev)
    if tuple(g.shape) != tuple(x.shape):
        raise ValueError(f"dimension mismatch: image {tuple(x.shape)} vs guide {tuple(g.shape)}")
    return x, g, kind, dev


def _check_margin(p: PatchParams, H: int, W: int) -> None:
    if p.pad_margin > min(H, W):  # pad_symmetric (image.py:107-110)
        raise ValueError(f"margin {p.pad_margin} exceeds min image extent {min(H, W)}")


def dsg_nlm_denoise(image, params: PatchParams, guide=None, distances: str = "integral",
                    *, return_aux: bool = False):
    """Doubly stochastic NLM, W x = K x / m + (1 - d/m) x (denoise.py:272-288).

    ``distances="integral"`` (default) runs the fast sweeps; ``"direct"`` the
    brute-force per-pixel path, as in the reference (denoise.py:291-355: patch
    distances summed over every patch element, cost window area x patch area;
    the bench-denoiser baseline).  Both give the same result within fp32
    rounding (the reference pins them to 1e-9 in float64,
    tests/test_denoise.py:244-249).  ``return_aux=True`` also returns the
    normalized row sums d and the max row sum m (north-star "alpha") as
    device tensors (fast path).
    """
    if distances not in ("integral", "direct"):
        raise ValueError(f"unknown distance method {distances!r}")
    if distances == "direct" and not return_aux:
        x, g, kind, dev = _pair(image, guide)
        B, H, W = A.dims(x)
        _check_margin(params, H, W)
        out = torch.empty_like(x)
        L.call("pnp_dsg_denoise_direct", L.context(dev), L.ptr(x), L.ptr(g), L.ptr(out), B, H,
               W, params.window_radius, params.patch_side, params._ctaps(),
               float(params.bandwidth))
        return A.from_device(out, kind)
    if guide is None and not return_aux:
        bands = _numpy_bands(image, params)
        if bands:
            return _dsg_numpy_banded(image, params, bands)
    x, g, kind, dev = _pair(image, guide)
    B, H, W = A.dims(x)
    _check_margin(params, H, W)
    out = torch.empty_like(x)
    d = torch.empty_like(x) if return_aux else None
    alpha = torch.empty(B, dtype=torch.float32, device=x.device) if return_aux else None
    with kcache_scope(dev, B, H, W, params):
        L.call("pnp_dsg_denoise", L.context(dev), L.ptr(x), L.ptr(g), L.ptr(out), B, H, W,
               params.window_radius, params.patch_side, params._ctaps(), float(params.bandwidth),
               L.ptr(d), L.ptr(alpha))
    res = A.from_device(out, kind)
    if return_aux:
        return res, A.from_device(d, kind), (alpha if kind == A.TORCH else alpha.cpu().numpy().astype(np.float64))
    return res


# numpy drop-in path of one large image: host cast + upload of band j+1
# overlaps sweep A of band j (pnp_dsg_band_sweep), the download + float64 cast
# of the result goes band by band as well
_NP_BANDS = 8


def _numpy_bands(image, params: PatchParams):
    """Input rows [0, need[j]) of each band when the banded numpy path
    applies (a large 2-D numpy image of a native-endian float / integer type,
    guide = image, the P-templated sweep), else None: everything else takes
    the validated one-shot path."""
    if isinstance(image, torch.Tensor):
        return None
    a = np.asarray(image)
    if (a.ndim != 2 or a.size < A._BIG or a.dtype.kind not in "fiu" or a.dtype.itemsize > 8
            or not a.dtype.isnative):
        return None
    H, W = a.shape
    if params.pad_margin > min(H, W):
        return None
    geom = L.dsg_geometry(H, W, params.window_radius, params.patch_side, params.is_box)
    if geom[3] != 0 or -(-H // geom[0]) < 2 * _NP_BANDS:
        return None
    te, need = (C.c_int * _NP_BANDS)(), (C.c_int * _NP_BANDS)()
    L.call("pnp_dsg_band_rows", H, W, params.window_radius, params.patch_side,
           int(params.is_box), _NP_BANDS, te, need)
    return list(need)


def _dsg_numpy_banded(image, params: PatchParams, bands):
    """dsg_nlm_denoise(numpy) with the upload overlapping sweep A; same bits
    as the one-shot path.  Non-finite input is detected on the device (one
    flag pass over the uploaded float32 image) and confirmed in float64 on the
    host before raising, as image.py:35-40 does."""
    src = A._host_tensor(np.asarray(image))
    H, W = src.shape
    dev = A.device_index()
    d = torch.device("cuda", dev)
    x = torch.empty((H, W), dtype=torch.float32, device=d)
    out = torch.empty_like(x)
    flag = torch.zeros(1, dtype=torch.int32, device=d)
    cur = torch.cuda.current_stream(d)
    h2d = A.copy_stream(dev, "h2d")
    h2d.wait_stream(cur)
    ctx = L.context(dev)
    taps, R, P, bw = params._ctaps(), params.window_radius, params.patch_side, float(params.bandwidth)
    with A.staging() as st, kcache_scope(dev, 1, H, W, params):
        stage = st.f32("in", H * W).view(H, W)
        r0 = 0
        for j, r1 in enumerate(bands):
            if r1 > r0:
                A.cast_into(stage[r0:r1], src[r0:r1])  # multi-threaded cast
                ev = torch.cuda.Event()
                with torch.cuda.stream(h2d):
                    x[r0:r1].copy_(stage[r0:r1], non_blocking=True)
                    ev.record(h2d)
                x.record_stream(h2d)  # x stays allocated until the uploads land
                cur.wait_event(ev)
                r0 = r1
            L.call("pnp_dsg_band_sweep", ctx, L.ptr(x), H, W, R, P, taps, bw, len(bands), j)
        L.call("pnp_flag_nonfinite", ctx, L.ptr(x), x.numel(), L.ptr(flag))
        L.call("pnp_dsg_band_finish", ctx, L.ptr(x), L.ptr(out), H, W, R, P, taps, bw)
        # fault the result's pages in (threaded) while the device denoises
        res = np.empty((H, W), dtype=np.float64)
        L.call("pnp_host_zero_f64", res.ctypes.data, res.size, 0)
        res = A.download64_banded(out, st, _NP_BANDS, res)
    if int(flag.item()):
        a = np.asarray(image, dtype=np.float64)
        if not np.all(np.isfinite(a)):
            raise ValueError("image contains non-finite values")
        raise ValueError("image values exceed the float32 range of the device path")
    return res


def nlm_denoise(image, params: PatchParams, guide=None):
    """Plain row-stochastic NLM over the clipped window (denoise.py:254-269)."""
    x, g, kind, dev = _pair(image, guide)
    B, H, W = A.dims(x)
    _check_margin(params, H, W)
    out = torch.empty_like(x)
    ctx = L.context(dev)
    L.call("pnp_nlm_denoise", ctx, L.ptr(x), L.ptr(g), L.ptr(out), B, H, W,
           params.window_radius, params.patch_side, params._ctaps(), float(params.bandwidth))
    return A.from_device(out, kind)


class FrozenGuide:
    """Snapshot of a guide; ``apply`` is a fixed linear operator
    (denoise.py:358-386).  The native handle owns a device copy of the guide
    and its rs = g^-1/2, row sums d and max row sum m; ``apply(x)`` is
    bit-identical to ``dsg_nlm_denoise(x, params, guide)``."""

    def __init__(self, guide, params: PatchParams):
        guide, kind = A.validate(guide, "guide", batch_ok=True)
        self.params = params
        self._kind = kind
        self._dev = A.device_index()
        g = A.to_device(guide, self._dev)
        self._shape = tuple(g.shape)
        B, H, W = A.dims(g)
        _check_margin(params, H, W)
        if kind == A.NUMPY:
            self.guide = np.array(guide, dtype=np.float64, copy=True)
            self.guide.setflags(write=False)
        else:
            self.guide = g.clone()
        self._h = C.c_void_p()
        # the pair-weight cache comes from torch's caching allocator (torch
        # sees it; re-freezing reuses the freed block instead of mapping new
        # pages) and lives as long as the handle
        with kcache_scope(self._dev, B, H, W, params) as kc:
            ctx = L.context(self._dev)
            L.call("pnp_dsg_freeze", ctx, L.ptr(g), B, H, W, params.window_radius,
                   params.patch_side, params._ctaps(), float(params.bandwidth), C.byref(self._h))
            self._kc = kc if self.cache_info()["rows_cached"] else None
        self._B = B

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                # orders the cache's allocation stream after the last apply;
                # torch recycles self._kc once this object is gone
                L.lib.pnp_frozen_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @property
    def alpha(self) -> np.ndarray:
        """Max normalized row sum m per image (reference's ``_m``)."""
        out = (C.c_float * self._B)()
        L.call("pnp_frozen_alpha", self._h, out)
        return np.array(out[:], dtype=np.float64)

    def cache_info(self) -> dict:
        """Pair-weight cache residency: tile rows per image cached (the rest
        recompute their weights on every apply), tile rows, bytes."""
        rows, total, nbytes = C.c_int(), C.c_int(), C.c_ulonglong()
        L.call("pnp_frozen_cache", self._h, C.byref(rows), C.byref(total), C.byref(nbytes))
        return {"rows_cached": rows.value, "tile_rows": total.value, "bytes": nbytes.value}

    def row_sums(self) -> torch.Tensor:
        d = torch.empty(self._shape, dtype=torch.float32, device=torch.device("cuda", self._dev))
        L.call("pnp_frozen_export", L.context(self._dev), self._h, None, L.ptr(d))
        return d

    def apply(self, image, out: torch.Tensor | None = None):
        image, kind = A.validate(image, "image", batch_ok=True)
        x = A.to_device(image, self._dev)
        if tuple(x.shape) != self._shape:
            raise ValueError(f"dimension mismatch: image {tuple(x.shape)} vs guide {self._shape}")
        return A.from_device(self.apply_device(x, out), kind)

    def apply_device(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Unchecked device apply (x: contiguous float32 CUDA, guide's shape)."""
        if out is None:
            out = torch.empty_like(x)
        L.call("pnp_dsg_apply", L.context(self._dev), self._h, L.ptr(x), L.ptr(out))
        return out

    def apply_admm(self, z: torch.Tensor, v: torch.Tensor, u: torch.Tensor, x: torch.Tensor,
                   v_prev, gt, rho: float, stats: torch.Tensor, flags: torch.Tensor) -> None:
        """v = W z with the linearized-ADMM u-update fused into the apply:
        u += x - v; stats (float64 [B, 4]) = sum (x-v)^2, sum (rho (v-v_prev))^2,
        sum (gt-v)^2; flags |= 4 on non-finite v / u (solver.py:222-228)."""
        L.call("pnp_dsg_apply_admm", L.context(self._dev), self._h, L.ptr(z), L.ptr(v), L.ptr(u),
               L.ptr(x), L.ptr(v_prev), L.ptr(gt), float(rho), L.ptr(stats), L.ptr(flags))

    def as_denoiser(self):
        """(img, k) -> W img plug-in for linearized_pnp_admm, device resident."""
        from .solver import device_callable

        fn = device_callable(lambda img, k: self.apply_device(img), graph_from=2)
        fn._pnp_frozen_for = lambda k: self  # lets the solver fuse the u-update
        return fn


def freeze_guide(guide, params: PatchParams) -> FrozenGuide:
    """Freeze the weight-defining guide (denoise.py:384-386)."""
    return FrozenGuide(guide, params)
