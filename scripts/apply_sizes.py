"""Frozen-apply + ADMM-step timing for a list of image sizes (development aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1901_06110_b200 as pnp

p = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
for n in [int(a) for a in sys.argv[1:]]:
    x = torch.rand(n, n, device="cuda")
    fz = pnp.freeze_guide(x, p)
    out = torch.empty_like(x)
    for _ in range(3):
        fz.apply_device(x, out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    s.record()
    for _ in range(reps):
        fz.apply_device(x, out)
    e.record()
    torch.cuda.synchronize()
    ta = s.elapsed_time(e) / reps * 1e3
    s.record()
    for _ in range(reps):
        pnp.dsg_nlm_denoise(x, p)
    e.record()
    torch.cuda.synchronize()
    print(f"{n}^2 frozen apply {ta:8.1f} us  adaptive {s.elapsed_time(e) / reps * 1e3:8.1f} us",
          flush=True)
    del fz
