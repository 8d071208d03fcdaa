"""Paper Fig. 2 style comparison on the GPU: linearized PnP-ADMM vs the
standard PnP-ADMM with a CG x-update, config-2 problem (512^2 SR, frozen
Gaussian-weight bicubic guide), same iterations (development aid)."""
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
fz = pnp.freeze_guide(guide, pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0))
prob = pnp.make_sr_problem(op, yd, ground_truth=torch.from_numpy(truth).to(dev))
for its in (30,):
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=its, constraint=pnp.UNIT_BOX,
                           cg_tol=1e-6, cg_max_iters=200)
    for name, fn in (("linearized", pnp.linearized_pnp_admm), ("standard-cg", pnp.standard_pnp_admm_cg)):
        fn(prob, cfg, denoiser=fz.as_denoiser())
        torch.cuda.synchronize()
        t = time.perf_counter()
        v, recs = fn(prob, cfg, denoiser=fz.as_denoiser())
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"{name:12s} {its} its: {dt*1e3:8.2f} ms  ({its/dt:8.1f} iters/s)  final PSNR "
              f"{recs[-1].psnr:.4f} dB", flush=True)
