"""8192^2: ShardedDSG (one strip, LocalComm) vs dsg_nlm_denoise on the same
image, alternating, CUDA events; kernel lists of one call each (diagnosis)."""
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200.parallel import LocalComm, ShardedDSG  # noqa: E402

n = 8192
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
sh = ShardedDSG(p, n, n, 1, [0], LocalComm(), device=torch.device("cuda", 0), kcache=True)
st = sh.states[0]
x = torch.rand(n, n, device="cuda")
st.own(st.buf).copy_(x)


def t(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for _ in range(2):
    sh.denoise()
    pnp.dsg_nlm_denoise(x, p)
for r in range(3):
    print(f"sharded {t(sh.denoise):.3f} ms   single {t(lambda: pnp.dsg_nlm_denoise(x, p)):.3f} ms")
for name, fn in (("sharded", sh.denoise), ("single", lambda: pnp.dsg_nlm_denoise(x, p))):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"],
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    print(f"== {name}")
    for e in evs:
        print(f"  {(e.time_range.start - t0) / 1e3:8.3f} +{(e.time_range.end - e.time_range.start) / 1e3:7.3f}"
              f"  {e.name[:70]}")
