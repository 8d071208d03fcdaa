"""Host side of the numpy call's tail: result allocation (4 KB pages vs
transparent huge pages), zero-fill, f32 -> f64 cast from pinned staging, and
D2H + cast overlap (diagnosis)."""
import mmap
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_1901_06110_b200 import _arrays as A  # noqa: E402

n = 8192
print("threads", torch.get_num_threads(),
      Path("/sys/kernel/mm/transparent_hugepage/enabled").read_text().strip(),
      Path("/sys/kernel/mm/transparent_hugepage/defrag").read_text().strip())


def huge(shape):
    nb = int(np.prod(shape)) * 8
    mm = mmap.mmap(-1, nb, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    mm.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(mm, dtype=np.float64).reshape(shape)


def t(fn, reps=3):
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        out.append((time.perf_counter() - t0) * 1e3)
    return " ".join("%.1f" % v for v in out)


src = torch.rand(n, n, dtype=torch.float32).pin_memory()
print("alloc+zero 4K   ", t(lambda: torch.from_numpy(np.empty((n, n))).zero_()))
print("alloc+zero huge ", t(lambda: torch.from_numpy(huge((n, n))).zero_()))


def cast(mk, touch, native):
    r = mk((n, n))
    if touch:
        torch.from_numpy(r).zero_()
    t0 = time.perf_counter()
    if native:
        A.cast_into(torch.from_numpy(r), src)
    else:
        torch.from_numpy(r).copy_(src)
    return (time.perf_counter() - t0) * 1e3


for native in (False, True):
    for name, mk in (("4K", np.empty), ("huge", huge)):
        print(f"{'native' if native else 'torch '} cast fresh {name}",
              " ".join("%.1f" % cast(mk, False, native) for _ in range(3)),
              f"| touched {name}", " ".join("%.1f" % cast(mk, True, native) for _ in range(3)))
s64 = np.random.default_rng(0).random((n, n))
st32 = torch.empty(n * n, dtype=torch.float32, pin_memory=True).view(n, n)
for native in (False, True):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        if native:
            A.cast_into(st32, torch.from_numpy(s64))
        else:
            st32.copy_(torch.from_numpy(s64))
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{'native' if native else 'torch '} f64 -> pinned f32", " ".join("%.1f" % v for v in ts))
x = torch.rand(n, n, device="cuda")
for name, mk in (("4K", np.empty), ("huge", huge)):
    for nb in (8, 16, 32):
        ts = []
        for _ in range(3):
            r = mk((n, n))
            torch.from_numpy(r).zero_()
            torch.cuda.synchronize()
            with A.staging() as st:
                t0 = time.perf_counter()
                A.download64_banded(x, st, nb, r)
                ts.append((time.perf_counter() - t0) * 1e3)
        print(f"D2H+cast {name} bands {nb}:", " ".join("%.1f" % v for v in ts))
