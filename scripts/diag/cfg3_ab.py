"""Config-3 solve wall time with the package at argv[1] (A/B across revisions)."""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, sys.argv[1])
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import synth  # noqa: E402

print(pnp.__file__)
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
runs = []
for i in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, recs = pnp.linearized_pnp_admm(prob, cfg3)
    torch.cuda.synchronize()
    runs.append((time.perf_counter() - t0) * 1e3)
print("walls", np.round(runs, 2), "median of last 9", np.median(runs[3:]))
x = torch.rand(512, 512, device=dev)
p = pnp.PatchParams.from_h(7, 10, 10 / 255, 2.0)
for _ in range(5):
    pnp.dsg_nlm_denoise(x, p)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    pnp.dsg_nlm_denoise(x, p)
torch.cuda.synchronize()
print("512^2 adaptive wall us", (time.perf_counter() - t0) * 1e4)
