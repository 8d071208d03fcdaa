"""One adaptive denoise (for ncu captures of the sweep kernels)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1901_06110_b200 as pnp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
x = torch.rand(n, n, device="cuda")
pnp.dsg_nlm_denoise(x, p)
torch.cuda.synchronize()
