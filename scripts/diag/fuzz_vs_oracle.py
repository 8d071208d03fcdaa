"""Randomized parity sweep (diagnosis): random shapes, radii, patch sides,
box / Gaussian taps, batches, own guides -- adaptive, frozen (k cache on and
off) and sharded calls against the float64 oracle (max |err| <= 1e-4) and
against each other (bitwise)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import profiling  # noqa: E402
from paper_1901_06110_b200.parallel import sharded_dsg_nlm_denoise  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
worst = 0.0
fails = []
for case in range(n_cases):
    P = int(rng.choice([1, 3, 5, 7, 9, 11, 13, 15, 17, 21, 25, 31]))
    R = int(rng.choice([1, 2, 3, 5, 8, 10, 13, 21, 33]))
    box = bool(rng.random() < 0.5) or P > 15
    sigma = None if box else float(rng.uniform(0.8, 3.0))
    M = R + (P - 1) // 2
    H = int(rng.integers(max(M, 8), max(M, 8) + 90))
    W = int(rng.integers(max(M, 8), max(M, 8) + 150))
    bw = float(rng.uniform(0.08, 0.4))
    img = rng.random((H, W))
    guide = rng.random((H, W)) if rng.random() < 0.3 else None
    p = pnp.PatchParams(P, R, bw, sigma)
    tag = f"case {case}: {H}x{W} P{P} R{R} {'box' if box else f'gauss{sigma:.2f}'} bw{bw:.3f}" \
          f"{' guide' if guide is not None else ''}"
    try:
        out = pnp.dsg_nlm_denoise(img, p, guide=guide)
        ref = oracle.dsg_nlm_denoise(img, P, R, bw, guide=guide, patch_sigma=sigma)
        err = float(np.abs(out - ref).max())
        worst = max(worst, err)
        ok = err <= 1e-4
        g = guide if guide is not None else img
        x = torch.from_numpy(img.astype(np.float32)).cuda()
        gt_ = torch.from_numpy(g.astype(np.float32)).cuda()
        fz = pnp.freeze_guide(gt_, p)
        a = fz.apply(x)
        b = pnp.dsg_nlm_denoise(x, p, guide=gt_)
        ok &= bool(torch.equal(a, b))
        profiling.set_cache_limit(0)
        try:
            c = pnp.freeze_guide(gt_, p).apply(x)
        finally:
            profiling.set_cache_limit(None)
        ok &= bool(torch.equal(a, c))
        if guide is None and H >= 2 * 32:
            try:
                s = sharded_dsg_nlm_denoise(x, p, 2)
                ok &= bool(torch.equal(s, b))
            except ValueError as e:  # strips thinner than their halos
                tag += f" (no 2-strip run: {e})"
        print(f"{tag}: max|err| {err:.2e} {'ok' if ok else 'FAIL'}", flush=True)
        if not ok:
            fails.append(tag)
    except ValueError as e:
        print(f"{tag}: ValueError {e}")
print(f"worst {worst:.3e}; failures: {fails or 'none'}")
