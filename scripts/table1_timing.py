"""The paper's Table 1 / the reference's bench-denoiser shape on the GPU:
256^2 smoothed SplitMix64 noise (cli.py:448-453), R = 21, box patches
P in {11, 17, 23, 29}, bandwidth 0.15 -- device time per dsg_nlm_denoise
(CUDA events, median of 20) and the reference itself (oracle/_ref, 1 core)
on the same image; plus box vs Gaussian taps at the config shape (R = 10,
P = 7, 8192^2 and 512^2) to show what the box path costs.
usage: table1_timing.py [--no-ref]"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda", 0)


def dev_ms(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


raw = pnp.SplitMix64(0).uniforms(256 * 256).reshape(256, 256)
img = pnp.sr_apply(pnp.SuperResOp(pnp.gaussian_kernel(2.0, 5), 1, "symmetric"), raw)
x = torch.from_numpy(np.asarray(img, np.float32)).to(dev)
res = {"table1": {}}
for P in (11, 17, 23, 29):
    p = pnp.PatchParams(P, 21, 0.15)
    geom = L.dsg_geometry(256, 256, 21, P, True)
    ms = dev_ms(lambda: pnp.dsg_nlm_denoise(x, p))
    row = {"gpu_ms": ms, "gpixel_offsets_per_s": 256 * 256 * 43 * 43 / (ms * 1e-3) / 1e9,
           "path": ["P-templated", "general half-window", "general full-window"][geom[3]],
           "TH": geom[0], "groups": geom[1]}
    if "--no-ref" not in sys.argv:
        sys.path.insert(0, str(ROOT))
        from oracle import refcpu
        if refcpu.available():
            units, s = refcpu.denoise_job((np.asarray(img), P, 21, 0.15))
            row["reference_cpu_s"] = s
            row["speedup"] = s / (ms * 1e-3)
    res["table1"][P] = row
    print(P, json.dumps(row), flush=True)
t = [r["gpu_ms"] for r in res["table1"].values()]
res["max_over_min"] = max(t) / min(t)
for n in (512, 8192):
    xx = torch.rand(n, n, device=dev)
    for sig in (None, 2.0):
        p = pnp.PatchParams(7, 10, (12 / 255) / 2 ** 0.5, sig)
        ms = dev_ms(lambda: pnp.dsg_nlm_denoise(xx, p), reps=5 if n > 4096 else 20)
        key = f"{n}^2 R10 P7 {'box' if sig is None else 'gaussian'}"
        res[key] = {"gpu_ms": ms, "gpixel_offsets_per_s": n * n * 441 / (ms * 1e-3) / 1e9}
        print(key, json.dumps(res[key]), flush=True)
    del xx
    torch.cuda.empty_cache()
print(json.dumps(res))
