"""Config-2 ADMM loop: wall vs device time per iteration + cProfile of the
host side (development aid)."""
import cProfile
import pstats
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
ITERS = int(sys.argv[1]) if len(sys.argv) > 1 else 30
GRAPH = {"on": True, "off": False}.get(sys.argv[2] if len(sys.argv) > 2 else "", None)
cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=ITERS, constraint=pnp.UNIT_BOX)
gt = torch.from_numpy(truth).to(dev)
fz = pnp.freeze_guide(guide, p2)
prob = pnp.make_sr_problem(op, yd, ground_truth=gt)


def run():
    return pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser(), graph=GRAPH)


for _ in range(3):
    run()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    v, recs = run()
torch.cuda.synchronize()
wall = (time.perf_counter() - t) / 5
print(f"[{ITERS} its, graph={GRAPH}] wall per run {wall*1e3:.2f} ms = {ITERS/wall:.0f} iters/s; "
      f"device time "
      f"{recs[-1].time_ms:.2f} ms; psnr {recs[-1].psnr:.4f}")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    run()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# per-category device time inside the loop (CUDA events around each launch)
from paper_1901_06110_b200 import profiling  # noqa: E402
profiling.enable(True)
run()
torch.cuda.synchronize()
pr = profiling.read()
profiling.enable(False)
print({k: (round(v[0] / ITERS * 1e3, 1), v[1] // ITERS) for k, v in pr.items() if v[1]},
      "(us per iteration, launches per iteration)")
