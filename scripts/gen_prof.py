"""One adaptive denoise through the general sweep (box taps), for ncu."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
P = int(sys.argv[2]) if len(sys.argv) > 2 else 7
R = int(sys.argv[3]) if len(sys.argv) > 3 else 10
x = torch.rand(n, n, device="cuda")
p = pnp.PatchParams(P, R, 0.15)
for _ in range(2):
    pnp.dsg_nlm_denoise(x, p)
torch.cuda.synchronize()
print("ok")
