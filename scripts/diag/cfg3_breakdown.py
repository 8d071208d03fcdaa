"""Config-3 solve: wall vs device time by kernel category (diagnosis)."""
import math
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import profiling, synth  # noqa: E402

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
for i in range(6):
    profiling.enable(True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, recs = pnp.linearized_pnp_admm(prob, cfg3)
    torch.cuda.synchronize()
    w = (time.perf_counter() - t0) * 1e3
    pr = profiling.read()
    profiling.enable(False)
    dev_ms = sum(a for a, _ in pr.values())
    print(f"wall {w:.2f} ms  device {dev_ms:.2f} ms  " +
          " ".join(f"{k}={a:.2f}/{n}" for k, (a, n) in pr.items() if n))
x = torch.rand(512, 512, device=dev)
p = pnp.PatchParams.from_h(7, 10, 10 / 255, 2.0)
for cache in (None, 0):
    profiling.set_cache_limit(cache)
    for _ in range(3):
        pnp.dsg_nlm_denoise(x, p)
    profiling.enable(True)
    for _ in range(10):
        pnp.dsg_nlm_denoise(x, p)
    pr = profiling.read()
    profiling.enable(False)
    print("512^2 adaptive, cache", cache, {k: (round(a / 10, 4), n // 10) for k, (a, n) in pr.items() if n})
profiling.set_cache_limit(None)
