"""A/B of the L2 evict_last budget of k-cache applies (PNP_KEEP_MB).

Config 2 (512^2 SR, frozen bicubic guide, 30 linearized-ADMM iterations):
median solve time per setting, the device time of the solver's own
iteration clock, a bare frozen-apply time, and a bitwise check of the final
iterate against the first setting.  Usage: python scripts/keep_ab.py [MB ...]
"""
import os
import sys
import time

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import synth  # noqa: E402

# settings "KEEP_MB" or "KEEP_MB:APW_MB" (APW: persisting access-policy window)
budgets = sys.argv[1:] or ["0", "32", "48", "64", "80", "96"]
dev = torch.device("cuda", 0)
truth = synth.scene(512, 512, 2).astype(np.float32)
op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
y = pnp.sr_simulate(truth.astype(np.float64), op, 5 / 255, seed=102).astype(np.float32)
yd = torch.from_numpy(y).to(dev)
guide = F.interpolate(yd.double()[None, None], scale_factor=2, mode="bicubic",
                      align_corners=False)[0, 0].clamp(0, 1).float().contiguous()
p2 = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=30, constraint=pnp.UNIT_BOX)
gt = torch.from_numpy(truth).to(dev)
prob = pnp.make_sr_problem(op, yd, ground_truth=gt)
fz = pnp.freeze_guide(guide, p2)
ref = None
for rep in range(2):
    for mb in budgets:
        keep, _, apw = mb.partition(":")
        os.environ["PNP_KEEP_MB"] = keep
        os.environ["PNP_APW_MB"] = apw or "0"
        runs, dev_ms = [], []
        for i in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            v, recs = pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
            torch.cuda.synchronize()
            if i:
                runs.append(time.perf_counter() - t0)
                dev_ms.append(recs[-1].time_ms)
        xa = torch.rand(512, 512, device=dev)
        for _ in range(5):
            fz.apply(xa)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            fz.apply(xa)
        e1.record()
        torch.cuda.synchronize()
        if ref is None:
            ref = v.clone()
        s = float(np.median(runs))
        print(f"rep {rep} KEEP:APW={mb:>6s}  solve {s * 1e3:6.3f} ms  {30 / s:8.0f} it/s  "
              f"device {float(np.median(dev_ms)):6.3f} ms  apply {e0.elapsed_time(e1) * 10:6.1f} us  "
              f"bitwise_equal={bool(torch.equal(v, ref))}", flush=True)
