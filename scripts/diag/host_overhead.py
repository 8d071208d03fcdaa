"""Host-side cost of one dsg_nlm_denoise call (device tensor): Python wrapper
vs the native call, for the P-templated and the general path (diagnosis)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import _lib as L, denoise as D  # noqa: E402

for (n, R, P, box) in ((256, 21, 11, True), (256, 5, 5, False), (512, 10, 7, False)):
    p = pnp.PatchParams(P, R, 0.15) if box else pnp.PatchParams.from_h(P, R, 10 / 255, 1.5)
    x = torch.rand(n, n, device="cuda")
    out = torch.empty_like(x)
    for _ in range(5):
        pnp.dsg_nlm_denoise(x, p)
    torch.cuda.synchronize()
    # whole Python call (includes the validation sync)
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pnp.dsg_nlm_denoise(x, p)
        ts.append(time.perf_counter() - t0)
    # the native call alone, issued back to back (host issue cost)
    ctx = L.context(0)
    taps = p._ctaps()
    tn = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.call("pnp_dsg_denoise", ctx, L.ptr(x), L.ptr(x), L.ptr(out), 1, n, n, R, P, taps,
               float(p.bandwidth), None, None)
        tn.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    for _ in range(20):
        D._pair(x, None)
    tv = (time.perf_counter() - t0) / 20
    t0 = time.perf_counter()
    for _ in range(20):
        with D.kcache_scope(0, 1, n, n, p):
            pass
    tk = (time.perf_counter() - t0) / 20
    torch.cuda.synchronize()
    print(f"{n}^2 R{R} P{P} {'box' if box else 'gauss'}: python call {1e3 * sorted(ts)[10]:.3f} ms "
          f"(wall incl. sync), native issue {1e3 * sorted(tn)[10]:.3f} ms, validate {1e3 * tv:.3f}, "
          f"kcache_scope {1e3 * tk:.3f}")
