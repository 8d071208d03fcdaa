"""Small fixed workload for ncu: one adaptive DSG-NLM denoise (sweep A C=1,
sweep B C=2) + two frozen applies at n^2, R=10, P=7 Gaussian (config-4 params)."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import paper_1901_06110_b200 as pnp

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(n, n, device="cuda", generator=g)
out = pnp.dsg_nlm_denoise(x, p)
fz = pnp.freeze_guide(x, p)
y = fz.apply_device(x)
y = fz.apply_device(x)
torch.cuda.synchronize()
print("ok", float(out.mean()), float(y.mean()))
