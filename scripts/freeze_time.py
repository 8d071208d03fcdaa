"""freeze_guide wall time at 512^2 (allocation + sweeps) and its kernel split
(development aid)."""
import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import profiling
p = pnp.PatchParams.from_h(7, 10, 10 / 255, 2.0)
x = torch.rand(512, 512, device="cuda")
for i in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    fz = pnp.freeze_guide(x, p)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"freeze {i}: {1e3*(t1-t0):.2f} ms", flush=True)
profiling.enable(True)
fz = pnp.freeze_guide(x, p)
torch.cuda.synchronize()
print({k: (round(v[0], 3), v[1]) for k, v in profiling.read().items() if v[1]})
