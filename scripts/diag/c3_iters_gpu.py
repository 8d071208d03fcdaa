"""Config-3 ADMM on the GPU with v saved at selected iterations (diagnosis)."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import synth  # noqa: E402
from conftest import load_golden  # noqa: E402

KEEP = list(range(1, 17)) + [20, 30, 40, 50]
gd = load_golden("cfg3.npz")
truth = synth.scene(512, 512, 3).astype(np.float32)
dev = torch.device("cuda", 0)
model = pnp.QisModel(128, 64.0)
counts = pnp.QisCounts(gd["ones"].astype(np.float64), gd["zeros"].astype(np.float64))
prob = pnp.make_qis_problem(counts, model, ground_truth=torch.from_numpy(truth).to(dev))
prob.x0 = torch.from_numpy(np.asarray(prob.x0, dtype=np.float32)).to(dev)
alpha = pnp.default_qis_alpha(counts, model)
cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=alpha, max_iters=50, freeze_at=15,
                       constraint=pnp.UNIT_BOX, denoiser="dsg-fixed", patch_side=7,
                       window_radius=10, bandwidth=(10 / 255) / math.sqrt(2.0), patch_sigma=2.0)
saved = {}


def cb(k, x, v, u):
    if k in KEEP:
        saved[f"v{k}"] = v.float().cpu().numpy() if isinstance(v, torch.Tensor) else np.float32(v)
        saved[f"x{k}"] = x.float().cpu().numpy() if isinstance(x, torch.Tensor) else np.float32(x)


v, recs = pnp.linearized_pnp_admm(prob, cfg, callback=cb)
saved["rec"] = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
np.savez(ROOT / "gpurun_out" / "c3_iters_gpu.npz", **saved)
dv = np.abs(v.double().cpu().numpy() - gd["v"])
print("max dv", dv.max(), "n>1e-4", int((dv > 1e-4).sum()), "psnr diff",
      np.abs(saved["rec"][:, 3] - gd["rec"][:, 3]).max())
