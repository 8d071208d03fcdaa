"""512^2 adaptive denoise timing, box vs Gaussian P7 R10 (A/B helper)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1901_06110_b200 as pnp  # noqa: E402

x = torch.rand(512, 512, device="cuda")
for name, p in (("box", pnp.PatchParams(7, 10, 0.15)),
                ("gauss", pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0))):
    for _ in range(5):
        pnp.dsg_nlm_denoise(x, p)
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pnp.dsg_nlm_denoise(x, p)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"512^2 {name}: median {ts[15]:.3f} ms, min {ts[0]:.3f}")
