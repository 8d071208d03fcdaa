"""Do the FP32-bound sweep A (+k-cache store) and the HBM-bound cached sweep B
overlap when launched on two streams?  (experiment; development aid)"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import _lib as L

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
R, P = 10, 7
TH = 26
tiles_y = -(-n // TH)
taps = p._ctaps()
dev = torch.device("cuda", 0)


def mkctx(stream):
    h = C.c_void_p()
    L.check(L.lib.pnp_ctx_create(0, C.byref(h)))
    L.check(L.lib.pnp_ctx_set_stream(h, C.c_void_p(stream.cuda_stream)))
    return h


class Img:
    def __init__(self, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.x = torch.rand(n, n, device="cuda", generator=g)
        self.rs = torch.rand(n, n, device="cuda", generator=g) * 0.1 + 0.2
        pf = int(L.lib.pnp_dsg_partial_floats(n, n, R, P, 2, tiles_y))
        self.part = torch.empty(pf, device="cuda")
        kf = int(L.lib.pnp_dsg_kcache_floats(n, n, R, P, tiles_y))
        self.kc = torch.empty(kf, device="cuda")

    def sweep(self, ctx, pass_):
        L.check(L.lib.pnp_dsg_strip_sweep(ctx, pass_, L.ptr(self.x), L.ptr(self.x), L.ptr(self.rs),
                                          n, n, 0, n, 0, tiles_y, R, P, taps, float(p.bandwidth),
                                          L.ptr(self.part), 0, tiles_y, L.ptr(self.kc)))


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
c1, c2 = mkctx(s1), mkctx(s2)
a, b = Img(1), Img(2)
b.sweep(c2, 0)  # fill b's k cache
torch.cuda.synchronize()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    a.sweep(c1, 0)   # sweep A + store  (stream 1)
    b.sweep(c2, 1)   # sweep B cached   (stream 2)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def only_a():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    a.sweep(c1, 0)
    cur.wait_stream(s1)


def only_b():
    cur = torch.cuda.current_stream()
    s2.wait_stream(cur)
    b.sweep(c2, 1)
    cur.wait_stream(s2)


ta, tb, tab = timed(only_a), timed(only_b), timed(both)
print(f"{n}^2: A+store alone {ta:.2f} ms, B cached alone {tb:.2f} ms, sum {ta + tb:.2f}, "
      f"concurrent {tab:.2f} ms ({(ta + tb) / tab:.2f}x)")
