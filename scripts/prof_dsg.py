"""Small fixed workload for ncu: one adaptive DSG-NLM denoise (sweep A C=1,
sweep B C=2) + two frozen applies at n^2, R=10, P=7 Gaussian (config-4 params).

usage: prof_dsg.py [n] [--nocache]"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import profiling

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if args else 2048
if "--nocache" in sys.argv:
    profiling.set_cache_limit(0)
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand(n, n, device="cuda", generator=g)
out = pnp.dsg_nlm_denoise(x, p)
fz = pnp.freeze_guide(x, p)
y = fz.apply_device(x)
y = fz.apply_device(x)
torch.cuda.synchronize()
print("ok", float(out.mean()), float(y.mean()))
