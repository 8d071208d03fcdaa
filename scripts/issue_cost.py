"""Host issue cost of the native ADMM loop vs its device time (config 2):
pnp_admm_run without timing returns as soon as everything is queued
(development aid)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import _lib as L
from paper_1901_06110_b200 import synth

dev = torch.device("cuda", 0)
truth = torch.from_numpy(synth.scene(512, 512, 2).astype(np.float32)).to(dev)
op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
y = pnp.sr_simulate(truth, op, 5 / 255, seed=102)
fz = pnp.freeze_guide(truth, pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0))
x, v0, v1, u, z = (torch.rand(512, 512, device=dev) for _ in range(5))
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
stats = torch.zeros((N, 1, 4), dtype=torch.float64, device=dev)
flags = torch.zeros(N, dtype=torch.int32, device=dev)
ctx = L.context(0)


def run(k1, ms=None):
    L.call("pnp_admm_run", ctx, 0, L.ptr(y), None, 1, 512, 512, op._taps, op.radius, op.factor,
           op._bnd, 0.0, 0.0, fz._h, 1, k1, L.ptr(x), L.ptr(v0), L.ptr(v1), L.ptr(u), L.ptr(z),
           L.ptr(truth), 0.5, 1.0, 1.0, 0.0, 1.0, L.ptr(stats), None, L.ptr(flags), ms, None)


for _ in range(3):
    run(N)
torch.cuda.synchronize()
for n in (1, 10, N):
    t0 = time.perf_counter()
    run(n)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{n:4d} its: host issue {1e6 * (t1 - t0) / n:7.1f} us/it, "
          f"issue+drain {1e6 * (t2 - t0) / n:7.1f} us/it", flush=True)
# per-entry host cost
for name, fn in (("apply_admm", lambda: L.call("pnp_dsg_apply_admm", ctx, fz._h, L.ptr(z), L.ptr(v1), L.ptr(u), L.ptr(x), L.ptr(v0), L.ptr(truth), 1.0, L.ptr(stats), L.ptr(flags))),
                 ("sr_grad_xupdate", lambda: op.gradient_xupdate_device(x, y, v0, u, z, 0.5, 1.0, 1.0, 0.0, 1.0, flags))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: host {1e6 * (t1 - t0) / 20:7.1f} us/call", flush=True)
