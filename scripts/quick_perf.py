"""Quick CUDA-event timing of the DSG kernels (development aid, not the bench)."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

import paper_1901_06110_b200 as pnp


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [512, 2048, 8192]
    p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
    for n in sizes:
        x = torch.rand(n, n, device="cuda")
        units = n * n * 21 * 21
        t = timeit(lambda: pnp.dsg_nlm_denoise(x, p), reps=3 if n > 4096 else 10)
        fz = pnp.freeze_guide(x, p)
        out = torch.empty_like(x)
        ta = timeit(lambda: fz.apply_device(x, out), reps=3 if n > 4096 else 20)
        print(f"{n}^2 R10 P7: adaptive {t*1e3:.3f} ms = {units/t/1e12:.3f} Tpix.off/s ; "
              f"frozen apply {ta*1e3:.3f} ms = {units/ta/1e12:.3f} Tpix.off/s", flush=True)


if __name__ == "__main__":
    main()
