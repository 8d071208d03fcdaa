"""Timing of the sync_call e2e step and torch allocator counters (diagnosis)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1901_06110_b200 as pnp  # noqa: E402

n = 8192
params = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
host_in = torch.from_numpy(bench.make_image_rows(n, 0, n)).pin_memory()
host_out = torch.empty_like(host_in).pin_memory()
dev = torch.device("cuda", 0)
for mode in ("sync", "dev"):
    x = host_in.to(dev)
    for i in range(6):
        torch.cuda.synchronize()
        s0 = torch.cuda.memory_stats()
        t0 = time.perf_counter()
        if mode == "sync":
            xd = host_in.to(dev, non_blocking=True)
            yd = pnp.dsg_nlm_denoise(xd, params)
            host_out.copy_(yd, non_blocking=True)
        else:
            pnp.dsg_nlm_denoise(x, params)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        s1 = torch.cuda.memory_stats()
        print(mode, i, f"{dt:.2f} ms", "device allocs", s1["num_device_alloc"] - s0["num_device_alloc"],
              "frees", s1["num_device_free"] - s0["num_device_free"],
              "reserved GB", round(torch.cuda.memory_reserved() / 2**30, 1), flush=True)
small = torch.rand(256, 256, device=dev)
p1 = pnp.PatchParams.from_h(5, 5, 10 / 255, 1.5)
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        pnp.dsg_nlm_denoise(small, p1, return_aux=True)
    torch.cuda.synchronize()
    print("config1 ms/call", (time.perf_counter() - t0) * 1e3 / 50)
