"""Where does a small freeze_guide's wall time go?  (config 2: 1024^2 guide
of a 512^2 x2 SR problem, P7 R10; diagnosis)"""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import profiling  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
p = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
g = torch.rand(n, n, device="cuda")


def run(label, keep=False, reps=6):
    fzs, walls, evs = [], [], []
    for i in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fz = pnp.freeze_guide(g, p)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        walls.append((t1 - t0) * 1e3)
        evs.append(e0.elapsed_time(e1))
        if keep:
            fzs.append(fz)
        else:
            del fz
    print(f"{label:34s} issue ms {['%.2f' % w for w in walls]}  device ms "
          f"{['%.2f' % e for e in evs]}  wall+sync {(t2 - t0) * 1e3:.2f}")


run("freeze (handle dropped each time)")
run("freeze (handles kept)", keep=True)
profiling.set_cache_limit(0)
run("freeze, no k cache")
profiling.set_cache_limit(None)
fz = pnp.freeze_guide(g, p)
x = torch.rand(n, n, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    fz.apply_device(x)
e1.record()
torch.cuda.synchronize()
print("apply ms", e0.elapsed_time(e1) / 20, fz.cache_info())

# the bench's config-2 loop: freeze, solve, re-freeze with the old handle alive
import gc  # noqa: E402

import numpy as np  # noqa: E402

truth = torch.rand(512, 512, device="cuda")
op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
y = op.apply(truth) if hasattr(op, "apply") else None
gd = torch.rand(512, 512, device="cuda")
cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=30, constraint=pnp.UNIT_BOX)
prob = pnp.make_sr_problem(op, torch.rand(256, 256, device="cuda"), ground_truth=truth)
for mode in ("plain", "del", "gc"):
    fz = None
    ts = []
    for i in range(6):
        if mode == "del":
            fz = None
        if mode == "gc":
            gc.collect()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fz = pnp.freeze_guide(gd, p)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        v, recs = pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
        torch.cuda.synchronize()
        ts.append((t1 - t0) * 1e3)
    print(mode, "freeze ms", ["%.2f" % t for t in ts], "live handles",
          sum(1 for o in gc.get_objects() if type(o).__name__ == "FrozenGuide"))

# host-phase breakdown of FrozenGuide.__init__ inside the solve loop
import ctypes as C  # noqa: E402

from paper_1901_06110_b200 import _arrays as A  # noqa: E402
from paper_1901_06110_b200 import _lib as L  # noqa: E402

fz = None
for i in range(8):
    fz = None
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    gg, kind = A.validate(gd, "guide", batch_ok=True)
    t.append(time.perf_counter())
    g2 = A.to_device(gg, 0)
    gclone = g2.clone()
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    h = C.c_void_p()
    ctx = L.context(0)
    L.call("pnp_dsg_freeze", ctx, L.ptr(g2), 1, 512, 512, 10, 7, p._ctaps(), float(p.bandwidth),
           C.byref(h))
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    fz = pnp.freeze_guide(gd, p)
    v, recs = pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
    L.lib.pnp_frozen_destroy(h)
    torch.cuda.synchronize()
    print("validate %.2f to_device+clone %.2f sync %.2f native-issue %.2f native-sync %.2f" %
          tuple((t[j + 1] - t[j]) * 1e3 for j in range(5)))
