"""Host cost of kcache_scope around a 512^2 adaptive denoise (diagnosis)."""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import denoise as D, solver as S  # noqa: E402

x = torch.rand(512, 512, device="cuda")
p = pnp.PatchParams.from_h(7, 10, 10 / 255, 2.0)
for _ in range(5):
    S._dsg_device(x, p)
torch.cuda.synchronize()


def t(fn, n=200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print("dsg_device us", t(lambda: S._dsg_device(x, p)))
print("scope only us", t(lambda: D.kcache_scope(0, 1, 512, 512, p).__enter__()))
print("capturing us", t(lambda: torch.cuda.is_current_stream_capturing(), 2000))
print("kcache_bytes us", t(lambda: D._kcache_bytes(0, 1, 512, 512, p), 2000))
print("empty 231MB us", t(lambda: torch.empty(231 << 20, dtype=torch.uint8, device="cuda"), 2000))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    S._dsg_device(x, p)
e1.record()
torch.cuda.synchronize()
print("device us per call", e0.elapsed_time(e1) * 10)
