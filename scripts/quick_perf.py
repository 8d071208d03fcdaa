"""Quick CUDA-event timing of the DSG kernels (development aid, not the bench).

usage: quick_perf.py [sizes...] [--nocache]   (k cache on by default, as in the library)
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import paper_1901_06110_b200 as pnp
from paper_1901_06110_b200 import profiling


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
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    modes = ["cache", "nocache"] if "--both" in sys.argv else (
        ["nocache"] if "--nocache" in sys.argv else ["cache"])
    sizes = [int(a) for a in args] or [512, 2048, 8192]
    p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
    for mode in modes:
        profiling.set_cache_limit(0 if mode.startswith("nocache") else None)
        for n in sizes:
            x = torch.rand(n, n, device="cuda")
            units = n * n * 21 * 21
            t = timeit(lambda: pnp.dsg_nlm_denoise(x, p), reps=3 if n > 4096 else 10)
            profiling.enable(True)
            pnp.dsg_nlm_denoise(x, p)
            pr = profiling.read()
            profiling.enable(False)
            fz = pnp.freeze_guide(x, p)
            out = torch.empty_like(x)
            ta = timeit(lambda: fz.apply_device(x, out), reps=3 if n > 4096 else 20)
            del fz
            print(f"[{mode}] {n}^2 R10 P7: adaptive {t*1e3:.3f} ms = {units/t/1e12:.3f} "
                  f"Tpix.off/s ; frozen apply {ta*1e3:.3f} ms = {units/ta/1e12:.3f} Tpix.off/s ; "
                  f"kernels {{{', '.join(f'{k}: {v[0]:.2f}ms/{v[1]}' for k, v in pr.items() if v[1])}}}",
                  flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
