"""Small invocations of every device path, for compute-sanitizer
(racecheck / synccheck / memcheck; profiles/sanitizer_*.log):
P-templated sweep in all modes (recompute, k-cache store, cached C=1 / C=2),
both fixup variants, the banded numpy path, the general sweep (half and full
window, box and Gaussian), plain NLM, the native ADMM loop (SR + QIS),
standard PnP-ADMM + CG."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import profiling  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device="cuda").manual_seed(0)


def rand(*s):
    return torch.rand(*s, device=dev, generator=g)


pg = pnp.PatchParams(7, 5, 0.2, 2.0)          # P-templated sweep
x = rand(96, 150)
profiling.set_cache_limit(0)                  # recompute sweeps
a = pnp.dsg_nlm_denoise(x, pg)
profiling.set_cache_limit(None)               # store + cached C=2 (px fixup: many groups)
b = pnp.dsg_nlm_denoise(x, pg)
assert torch.equal(a, b)
fz = pnp.freeze_guide(x, pg)                  # cached C=1 + apply fixup
assert torch.equal(fz.apply(x), a)
xt = rand(1, 40 * 26, 2 * 64 * 4)             # many tiles, NG <= 2: tile fixup
pnp.dsg_nlm_denoise(xt[0], pnp.PatchParams(7, 3, 0.2, 2.0))
big = np.random.default_rng(1).random((1056, 1000))   # banded numpy path
pnp.dsg_nlm_denoise(big, pnp.PatchParams(5, 3, 0.2, 1.5))
pnp.dsg_nlm_denoise(rand(70, 90), pnp.PatchParams(17, 6, 0.2))        # general, box
pnp.dsg_nlm_denoise(rand(60, 70), pnp.PatchParams(19, 4, 0.2, 3.0))   # general, Gaussian
pnp.dsg_nlm_denoise(rand(104, 104), pnp.PatchParams(1, 100, 0.3))     # general, full window
pnp.nlm_denoise(x, pg)
op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
truth = rand(64, 96)
y = (op.apply_device(truth) + 0.02 * rand(32, 48)).contiguous()
prob = pnp.make_sr_problem(op, y, ground_truth=truth)
cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=3, constraint=pnp.UNIT_BOX)
pnp.linearized_pnp_admm(prob, cfg, denoiser=pnp.freeze_guide(truth, pg).as_denoiser())
cfgq = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=128.0, max_iters=4, freeze_at=2,
                        constraint=pnp.UNIT_BOX, denoiser="dsg-fixed", patch_side=5,
                        window_radius=3, bandwidth=0.1, patch_sigma=1.5)
counts = pnp.qis_simulate(truth.double().cpu().numpy(), pnp.QisModel(16, 16.0), seed=3)
pnp.linearized_pnp_admm(pnp.make_qis_problem(counts, pnp.QisModel(16, 16.0)), cfgq)
cfgs = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=2, constraint=pnp.UNIT_BOX,
                        cg_tol=1e-6, cg_max_iters=20)
pnp.standard_pnp_admm_cg(prob, cfgs, denoiser=pnp.freeze_guide(truth, pg).as_denoiser())
# SR fast tiles (factor 2, 9x9: interior tiles of a 192 x 224 batch) and
# their boundary tiles, residual + adjoint + fused x-update
ys = rand(2, 96, 112)
xs = rand(2, 192, 224)
op.adjoint_device(ys)
op.apply_device(xs)
pnp.sr_gradient(op, xs, ys)
torch.cuda.synchronize()
print("sanitize cases ok")
