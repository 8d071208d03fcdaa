"""Per-call timing distribution of the adaptive denoise on small images
(device events and host wall; development aid)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import profiling

p = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
for n in [int(a) for a in sys.argv[1:]] or [256, 512]:
    x = torch.rand(n, n, device="cuda")
    for _ in range(5):
        pnp.dsg_nlm_denoise(x, p)
    torch.cuda.synchronize()
    dev, wall = [], []
    for _ in range(100):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record()
        pnp.dsg_nlm_denoise(x, p)
        e.record()
        torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e6)
        dev.append(s.elapsed_time(e) * 1e3)
    dev, wall = np.array(dev), np.array(wall)
    profiling.enable(True)
    pnp.dsg_nlm_denoise(x, p)
    torch.cuda.synchronize()
    pr = profiling.read()
    profiling.enable(False)
    print(f"{n}^2 adaptive: device median {np.median(dev):.1f} p90 {np.percentile(dev, 90):.1f} "
          f"max {dev.max():.1f} us; wall median {np.median(wall):.1f} max {wall.max():.1f} us; "
          f"{ {k: round(v[0] * 1e3, 1) for k, v in pr.items() if v[1]} }", flush=True)
