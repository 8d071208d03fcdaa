"""Randomized parity sweep of the SR operator (diagnosis): random shapes,
factors, blur radii / sigmas, boundaries and batches -- sr_apply, sr_adjoint
and sr_gradient against the float64 oracle (max |err| <= 2e-6 on [0, 1]
inputs), and every batched result bitwise equal to its single-image call.
Covers the factor-2 / 9x9 fast tiles (interior and boundary) and the generic
kernels."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import forward as ofw  # noqa: E402
import paper_1901_06110_b200 as pnp  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
worst, fails = 0.0, []
for case in range(n_cases):
    k = int(rng.choice([1, 2, 2, 2, 3, 4]))
    rad = int(rng.choice([1, 2, 3, 4, 4, 4, 6, 8]))
    sigma = float(rng.uniform(0.6, 2.5))
    boundary = "symmetric" if rng.random() < 0.6 else "periodic"
    lo = max(2 * rad + 2, 8)
    H = k * int(rng.integers(-(-lo // k), 180 // k + 2))
    W = k * int(rng.integers(-(-lo // k), 260 // k + 2))
    B = int(rng.choice([1, 1, 2, 3]))
    ker = ofw.gaussian_kernel(sigma, rad)
    op = pnp.SuperResOp(pnp.gaussian_kernel(sigma, rad), k, boundary)
    x = rng.random((B, H, W)).astype(np.float32)
    y = rng.random((B, H // k, W // k)).astype(np.float32)
    tag = f"case {case}: B{B} {H}x{W} k{k} r{rad} s{sigma:.2f} {boundary}"
    try:
        xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        ap = pnp.sr_apply(op, xt).cpu().numpy()
        ad = pnp.sr_adjoint(op, yt).cpu().numpy()
        gr = pnp.sr_gradient(op, xt, yt).cpu().numpy()
        for i in range(B):
            errs = [np.abs(ap[i] - ofw.sr_apply(ker, k, boundary, x[i])).max(),
                    np.abs(ad[i] - ofw.sr_adjoint(ker, k, boundary, y[i])).max(),
                    np.abs(gr[i] - ofw.sr_gradient(ker, k, boundary, x[i], y[i])).max()]
            worst = max(worst, *errs)
            if max(errs) > 2e-6:
                fails.append(f"{tag} image {i}: errors {errs}")
            if B > 1:
                single = [pnp.sr_apply(op, xt[i].contiguous()).cpu().numpy(),
                          pnp.sr_adjoint(op, yt[i].contiguous()).cpu().numpy(),
                          pnp.sr_gradient(op, xt[i].contiguous(), yt[i].contiguous()).cpu().numpy()]
                for name, a_, s_ in zip(("apply", "adjoint", "gradient"), (ap, ad, gr), single):
                    if not np.array_equal(a_[i], s_):
                        fails.append(f"{tag} image {i}: batched {name} != single")
    except Exception as e:  # noqa: BLE001
        fails.append(f"{tag}: {type(e).__name__}: {e}")
print(f"{n_cases} cases, worst max|err| vs the float64 oracle {worst:.3g}")
print("failures:", fails or "none")
sys.exit(1 if fails else 0)
