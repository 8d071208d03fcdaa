"""Pipelined host -> device -> host DSG-NLM over a sequence of images.

A serving-style front end for the same denoiser: each image's host-to-device
copy, denoise and device-to-host copy run on three CUDA streams (copy-engine
H2D, compute, copy-engine D2H) over ``depth`` device buffer sets, so image
i+1 uploads and image i-1 downloads while image i is being denoised.  Every
image still crosses PCIe both ways; only the waiting overlaps.  Results are
bitwise identical to ``dsg_nlm_denoise`` on each image.  Input validation
(non-finite -> ValueError, reference image.py:35-40) runs on the device, in
stream order, and is reported when the batch is collected.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _arrays as A
from . import _lib as L
from .denoise import PatchParams, _check_margin, kcache_scope


class DenoiseStream:
    """``run(host_images)`` denoises a sequence of same-shape float32 images
    (pinned CPU tensors for full overlap) and returns host outputs."""

    def __init__(self, params: PatchParams, shape, device: int | None = None, depth: int = 2):
        self.params = params
        self.shape = tuple(int(s) for s in shape)
        if len(self.shape) not in (2, 3):
            raise ValueError(f"images must be 2-D (or a 3-D batch), got shape {self.shape}")
        self.dev = A.device_index() if device is None else device
        d = torch.device("cuda", self.dev)
        B, H, W = (1,) + self.shape if len(self.shape) == 2 else self.shape
        _check_margin(params, H, W)
        self.B, self.H, self.W = B, H, W
        self.depth = max(2, int(depth))
        self.din = [torch.empty(self.shape, dtype=torch.float32, device=d) for _ in range(self.depth)]
        self.dout = [torch.empty_like(self.din[0]) for _ in range(self.depth)]
        self.s_h2d, self.s_comp, self.s_d2h = (torch.cuda.Stream(d) for _ in range(3))
        self._taps = params._ctaps()
        L.call("pnp_ctx_reserve", L.context(self.dev), B, H, W, params.window_radius,
               params.patch_side, int(params.is_box))
        # the first image of a run has no earlier image to hide its upload
        # behind: it goes up in row bands and its sweep A starts band by band
        # (pnp_dsg_denoise_banded); later images overlap the previous denoise
        self._bands = None
        nb = 4
        geom = L.dsg_geometry(H, W, params.window_radius, params.patch_side, params.is_box)
        if B == 1 and geom[3] == 0 and -(-H // geom[0]) >= 4 * nb:
            te, need = (C.c_int * nb)(), (C.c_int * nb)()
            L.call("pnp_dsg_band_rows", H, W, params.window_radius, params.patch_side,
                   int(params.is_box), nb, te, need)
            self._bands = list(need)

    def run(self, host_images, host_outs=None):
        n = len(host_images)
        for im in host_images:
            if tuple(im.shape) != self.shape:
                raise ValueError(f"dimension mismatch: {tuple(im.shape)} vs {self.shape}")
        if host_outs is None:
            host_outs = [torch.empty(self.shape, dtype=torch.float32, pin_memory=True)
                         for _ in range(n)]
        d = torch.device("cuda", self.dev)
        flags = torch.zeros(n, dtype=torch.int32, device=d)
        cur = torch.cuda.current_stream(d)
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            s.wait_stream(cur)
        with torch.cuda.stream(self.s_comp):  # the k cache lives on the compute stream
            scope = kcache_scope(self.dev, self.B, self.H, self.W, self.params)
            scope.__enter__()
        try:
            return self._run(host_images, host_outs, n, d, flags, cur)
        finally:
            with torch.cuda.stream(self.s_comp):
                scope.__exit__(None, None, None)

    def _run(self, host_images, host_outs, n, d, flags, cur):
        up = [torch.cuda.Event() for _ in range(n)]
        done = [torch.cuda.Event() for _ in range(n)]
        down = [torch.cuda.Event() for _ in range(n)]
        p = self.params
        for i in range(n):
            k = i % self.depth
            banded = i == 0 and self._bands is not None
            band_ev = []
            with torch.cuda.stream(self.s_h2d):
                if i >= self.depth:
                    self.s_h2d.wait_event(done[i - self.depth])   # din[k] consumed
                src = host_images[i]
                if not isinstance(src, torch.Tensor):
                    src = torch.from_numpy(np.ascontiguousarray(src, dtype=np.float32))
                if banded:
                    r0 = 0
                    for r1 in self._bands:
                        if r1 > r0:
                            self.din[k][r0:r1].copy_(src[r0:r1], non_blocking=True)
                            r0 = r1
                        ev = torch.cuda.Event()
                        ev.record(self.s_h2d)
                        band_ev.append(ev)
                else:
                    self.din[k].copy_(src, non_blocking=True)
                up[i].record(self.s_h2d)
            with torch.cuda.stream(self.s_comp):
                if not banded:
                    self.s_comp.wait_event(up[i])
                if i >= self.depth:
                    self.s_comp.wait_event(down[i - self.depth])  # dout[k] downloaded
                ctx = L.context(self.dev)
                x = self.din[k]
                if banded:  # sweep A band by band as the rows arrive
                    evs = (C.c_void_p * len(band_ev))(*[e.cuda_event for e in band_ev])
                    L.call("pnp_dsg_denoise_banded", ctx, L.ptr(x), L.ptr(self.dout[k]), self.H,
                           self.W, p.window_radius, p.patch_side, self._taps,
                           float(p.bandwidth), len(band_ev), evs)
                    self.s_comp.wait_event(up[i])
                    L.call("pnp_flag_nonfinite", ctx, L.ptr(x), x.numel(), L.ptr(flags[i:i + 1]))
                else:
                    L.call("pnp_flag_nonfinite", ctx, L.ptr(x), x.numel(), L.ptr(flags[i:i + 1]))
                    L.call("pnp_dsg_denoise", ctx, L.ptr(x), L.ptr(x), L.ptr(self.dout[k]),
                           self.B, self.H, self.W, p.window_radius, p.patch_side, self._taps,
                           float(p.bandwidth), None, None)
                done[i].record(self.s_comp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(done[i])
                host_outs[i].copy_(self.dout[k], non_blocking=True)
                down[i].record(self.s_d2h)
        for s in (self.s_h2d, self.s_comp, self.s_d2h):
            cur.wait_stream(s)
        bad = torch.nonzero(flags).flatten().tolist()  # syncs
        if bad:
            raise ValueError(f"image {bad[0]} contains non-finite values")
        return host_outs


def denoise_host_sequence(host_images, params: PatchParams, depth: int = 2):
    """Convenience wrapper: pipelined denoise of same-shape host images."""
    if not len(host_images):
        return []
    return DenoiseStream(params, tuple(host_images[0].shape), depth=depth).run(host_images)
