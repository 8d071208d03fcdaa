"""Config-3 QIS solve repeated: wall / device time per run and around the
freeze iteration (development aid)."""
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import synth

dev = torch.device("cuda", 0)
truth3 = synth.scene(512, 512, 3).astype(np.float32)
model = pnp.QisModel(128, 64.0)
counts = pnp.qis_simulate(truth3.astype(np.float64), model, seed=103)
prob = pnp.make_qis_problem(counts, model, ground_truth=torch.from_numpy(truth3).to(dev))
prob.x0 = torch.from_numpy(prob.x0.astype(np.float32)).to(dev)
cfg3 = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=pnp.default_qis_alpha(counts, model),
                        max_iters=50, freeze_at=15, constraint=pnp.UNIT_BOX,
                        denoiser="dsg-fixed", patch_side=7, window_radius=10,
                        bandwidth=(10 / 255) / math.sqrt(2), patch_sigma=2.0)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, recs = pnp.linearized_pnp_admm(prob, cfg3)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ts = [r.time_ms for r in recs]
    print(f"run {i}: wall {1e3 * (t1 - t0):.2f} ms device {ts[-1]:.2f}: it1-14 {ts[13]:.2f} "
          f"it15 {ts[14] - ts[13]:.2f} it16-50 {ts[-1] - ts[14]:.2f} psnr {recs[-1].psnr:.4f}",
          flush=True)
