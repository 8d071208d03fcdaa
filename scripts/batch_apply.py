"""Frozen apply of a batch of images (config-5 shape) per image (development aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1901_06110_b200 as pnp

p = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
B, n = int(sys.argv[1]), int(sys.argv[2])
x = torch.rand(B, n, n, device="cuda")
fz = pnp.freeze_guide(x, p)
out = torch.empty_like(x)
for _ in range(2):
    fz.apply_device(x, out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    fz.apply_device(x, out)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"B={B} {n}^2 frozen apply {ms:.2f} ms = {ms / B * 1e3:.1f} us per image, "
      f"{B * n * n * 441 / ms / 1e9:.3f} T pixel*offset/s", flush=True)
