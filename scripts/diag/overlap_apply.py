"""Do a k-cache (HBM-bound) frozen apply and a recompute (FP32-bound) frozen
apply overlap when issued on two streams?  (feasibility of a cached/recompute
offset split; diagnosis)"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import profiling  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
xa = torch.rand(n, n, device="cuda")
xb = torch.rand(n, n, device="cuda")
fa = pnp.freeze_guide(xa, p)                      # cached
profiling.set_cache_limit(0)
fb = pnp.freeze_guide(xb, p)                      # recompute
profiling.set_cache_limit(None)
print("cached:", fa.cache_info(), "recompute:", fb.cache_info())
oa, ob = torch.empty_like(xa), torch.empty_like(xb)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def ev_time(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ta = ev_time(lambda: fa.apply_device(xa, oa))
tb = ev_time(lambda: fb.apply_device(xb, ob))


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        fa.apply_device(xa, oa)
    with torch.cuda.stream(s2):
        fb.apply_device(xb, ob)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


tab = ev_time(both)
print(f"{n}^2: cached {ta:.3f} ms, recompute {tb:.3f} ms, sum {ta + tb:.3f}, "
      f"two streams {tab:.3f} ms (max {max(ta, tb):.3f})")
print("checksums", float(oa.double().sum()), float(ob.double().sum()))
