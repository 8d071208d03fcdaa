"""Host/device timeline of dsg_nlm_denoise(float64 numpy) at 8192^2 (diagnosis):
the banded path's steps with host timestamps and device events."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import _arrays as A, _lib as L, denoise as D  # noqa: E402

n = 8192
params = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
img = np.random.default_rng(0).random((n, n))
print("threads", torch.get_num_threads(), "THP", Path("/sys/kernel/mm/transparent_hugepage/enabled").read_text().strip())
for _ in range(2):
    pnp.dsg_nlm_denoise(img, params)
torch.cuda.synchronize()


def run(trace):
    image = img
    bands = D._numpy_bands(image, params)
    t0 = time.perf_counter()
    T = lambda name: trace.append((name, (time.perf_counter() - t0) * 1e3))
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
    e_start = torch.cuda.Event(enable_timing=True)
    e_start.record(cur)
    evs = []
    with A.staging() as st, D.kcache_scope(dev, 1, H, W, params):
        stage = st.f32("in", H * W).view(H, W)
        r0 = 0
        T("setup")
        for j, r1 in enumerate(bands):
            if r1 > r0:
                A.cast_into(stage[r0:r1], src[r0:r1])
                T(f"cast{j}")
                ev = torch.cuda.Event()
                with torch.cuda.stream(h2d):
                    x[r0:r1].copy_(stage[r0:r1], non_blocking=True)
                    ev.record(h2d)
                cur.wait_event(ev)
                r0 = r1
            L.call("pnp_dsg_band_sweep", ctx, L.ptr(x), H, W, R, P, taps, bw, len(bands), j)
            e = torch.cuda.Event(enable_timing=True)
            e.record(cur)
            evs.append((f"bandA{j}", e))
        L.call("pnp_flag_nonfinite", ctx, L.ptr(x), x.numel(), L.ptr(flag))
        L.call("pnp_dsg_band_finish", ctx, L.ptr(x), L.ptr(out), H, W, R, P, taps, bw)
        e = torch.cuda.Event(enable_timing=True)
        e.record(cur)
        evs.append(("finish", e))
        T("enqueued")
        res = np.empty((H, W), dtype=np.float64)
        L.call("pnp_host_zero_f64", res.ctypes.data, res.size, 0)
        T("zero_fill")
        res = A.download64_banded(out, st, D._NP_BANDS, res)
        T("download_cast")
    flag.item()
    T("done")
    torch.cuda.synchronize()
    dev_t = [(name, e_start.elapsed_time(e)) for name, e in evs]
    return dev_t


for rep in range(3):
    tr = []
    dt = run(tr)
    print("host:", " ".join(f"{k}={v:.1f}" for k, v in tr))
    print("dev: ", " ".join(f"{k}={v:.1f}" for k, v in dt))
walls = []
for _ in range(5):
    w0 = time.perf_counter()
    pnp.dsg_nlm_denoise(img, params)
    walls.append((time.perf_counter() - w0) * 1e3)
print("api wall", np.round(walls, 1))
# raw host bandwidths
a = np.random.default_rng(1).random((n, n))
s32 = torch.empty((n, n), dtype=torch.float32).pin_memory()
for _ in range(2):
    t = time.perf_counter(); s32.copy_(torch.from_numpy(a)); c = (time.perf_counter() - t) * 1e3
print("cast f64->pinned f32 ms", round(c, 1))
gx = torch.empty((n, n), dtype=torch.float32, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); gx.copy_(s32, non_blocking=True); torch.cuda.synchronize(); h = (time.perf_counter() - t) * 1e3
    t = time.perf_counter(); s32.copy_(gx, non_blocking=True); torch.cuda.synchronize(); dd = (time.perf_counter() - t) * 1e3
print("H2D ms", round(h, 2), "D2H ms", round(dd, 2))
r = np.empty((n, n)); t = time.perf_counter(); torch.from_numpy(r).zero_(); print("zero-fill fresh 512MB ms", round((time.perf_counter() - t) * 1e3, 1))
t = time.perf_counter(); torch.from_numpy(r).copy_(s32); print("cast pinned f32 -> f64 (touched) ms", round((time.perf_counter() - t) * 1e3, 1))
r2 = np.empty((n, n)); t = time.perf_counter(); torch.from_numpy(r2).copy_(s32); print("cast pinned f32 -> f64 (fresh) ms", round((time.perf_counter() - t) * 1e3, 1))
