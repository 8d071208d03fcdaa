"""Fixed vs per-iteration host cost of linearized_pnp_admm on config 2
(wall time for several iteration counts; development aid)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch
import torch.nn.functional as F

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import synth

dev = torch.device("cuda", 0)
truth = synth.scene(512, 512, 2).astype(np.float32)
op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
y = pnp.sr_simulate(truth.astype(np.float64), op, 5 / 255, seed=102).astype(np.float32)
yd = torch.from_numpy(y).to(dev)
guide = F.interpolate(yd.double()[None, None], scale_factor=2, mode="bicubic",
                      align_corners=False)[0, 0].clamp(0, 1).float().contiguous()
p2 = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
gt = torch.from_numpy(truth).to(dev)
fz = pnp.freeze_guide(guide, p2)
prob = pnp.make_sr_problem(op, yd, ground_truth=gt)
for iters in (1, 2, 5, 30, 100):
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=iters, constraint=pnp.UNIT_BOX)
    for _ in range(3):
        pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
    torch.cuda.synchronize()
    reps = 10
    t = time.perf_counter()
    for _ in range(reps):
        v, recs = pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
    wall = (time.perf_counter() - t) / reps * 1e3
    print(f"iters {iters:4d}: wall {wall:7.3f} ms  device {recs[-1].time_ms:7.3f} ms  "
          f"wall-device {wall - recs[-1].time_ms:6.3f} ms", flush=True)
