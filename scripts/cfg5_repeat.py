"""Config-5 batched SR solve repeated: wall / device time and PSNR per run
(development aid; PNP_PDL in the environment selects the launch mode)."""
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
nb, side = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 1024
op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
p2 = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
truths = [synth.scene(side, side, 1000 + i).astype(np.float32) for i in range(nb)]
yb = torch.stack([pnp.sr_simulate(torch.from_numpy(t).to(dev), op, 0.0, seed=0) for t in truths])
yb = (yb + 0.02 * torch.randn(yb.shape, generator=torch.Generator().manual_seed(0)).to(dev)).contiguous()
gtb = torch.from_numpy(np.stack(truths)).to(dev)
guides = F.interpolate(yb.double()[:, None], scale_factor=2, mode="bicubic",
                       align_corners=False)[:, 0].clamp(0, 1).float().contiguous()
cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=20, constraint=pnp.UNIT_BOX)
prob = pnp.make_sr_problem(op, yb, ground_truth=gtb)
fz = pnp.freeze_guide(guides, p2)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, recs = pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"run {i}: wall {1e3*(t1-t0):.1f} ms device {recs[-1].time_ms:.1f} ms "
          f"psnr {float(np.mean(recs[-1].psnr)):.6f}", flush=True)
