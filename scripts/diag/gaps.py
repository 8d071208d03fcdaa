"""Kernel timeline of one 8192^2 adaptive denoise (device tensor): where do
the ~2 ms between the sum of kernel times and the event-timed call go?
(torch.profiler / CUPTI kernel records; diagnosis)"""
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
if len(sys.argv) > 3:  # n R P: box patches (the reference's own), bandwidth 0.15
    p = pnp.PatchParams(int(sys.argv[3]), int(sys.argv[2]), 0.15)
else:
    p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
x = torch.rand(n, n, device="cuda")
for _ in range(3):
    pnp.dsg_nlm_denoise(x, p)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    pnp.dsg_nlm_denoise(x, p)
e1.record()
torch.cuda.synchronize()
print("event ms per call", e0.elapsed_time(e1) / 5)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        pnp.dsg_nlm_denoise(x, p)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev = None
for e in evs:
    s, t = e.time_range.start - t0, e.time_range.end - t0
    gap = (s - prev) if prev is not None else 0
    print(f"{s / 1e3:9.3f} ms  dur {(t - s) / 1e3:8.3f}  gap {gap / 1e3:7.3f}  {e.name[:80]}")
    prev = t
cpu = [e for e in prof.events() if e.device_type.name == "CPU" and "cuda" in e.name.lower()]
agg = {}
for e in cpu:
    agg.setdefault(e.name, [0, 0.0])
    agg[e.name][0] += 1
    agg[e.name][1] += (e.time_range.end - e.time_range.start) / 1e3
for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"host {k[:60]:60s} x{c:4d} {ms:8.3f} ms")
