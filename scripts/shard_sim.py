"""Virtual-shard timing of the config-4 row-strip algorithm on one GPU: the
N strips run back to back (LocalComm), so total/N estimates the per-rank
device time of an N-GPU run without its NCCL exchanges (development aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200.parallel import LocalComm, ShardedDSG

n = 8192
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
x = torch.rand(n, n, device="cuda")


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


base = t(lambda: pnp.dsg_nlm_denoise(x, p))
print(f"single call: {base:.2f} ms")
ref = pnp.dsg_nlm_denoise(x, p)
for N in (1, 2, 4, 8):
    sh = ShardedDSG(p, n, n, N, range(N), LocalComm())
    sh.load(x)
    ms = t(sh.denoise)
    same = torch.equal(sh.gather(), ref)
    print(f"N={N}: all strips {ms:.2f} ms -> {ms / N:.2f} ms per rank, ideal {base / N:.2f}; "
          f"efficiency bound {base / ms:.3f}; bitwise == single: {same}", flush=True)
    del sh
    torch.cuda.empty_cache()
