"""Outputs of every device path on small seeded inputs, saved to an .npz
(argv[1]); run against the product library and against the PNP_CHECKS +
PNP_JITTER debug build (tests/test_checks_gpu.py): the debug build asserts
every shared-memory index and global write, and reorders the warps at each
barrier, so equal bits across runs show the barrier / ordered-flush protocol
holds and no access leaves its buffer."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1901_06110_b200 as pnp  # noqa: E402
from paper_1901_06110_b200 import profiling  # noqa: E402
from paper_1901_06110_b200.parallel import sharded_dsg_nlm_denoise  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device="cuda").manual_seed(0)
out = {}


def rand(*s):
    return torch.rand(*s, device=dev, generator=g)


def keep(name, t):
    out[name] = t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


pg = pnp.PatchParams(7, 5, 0.2, 2.0)
x = rand(96, 150)
profiling.set_cache_limit(0)
keep("fast_recompute", pnp.dsg_nlm_denoise(x, pg))
profiling.set_cache_limit(None)
o, d, a = pnp.dsg_nlm_denoise(x, pg, return_aux=True)
keep("fast_cached", o), keep("fast_d", d), keep("fast_alpha", a)
keep("fast_frozen", pnp.freeze_guide(x, pg).apply(x))
xb = rand(3, 80, 140)
keep("fast_batch", pnp.dsg_nlm_denoise(xb, pnp.PatchParams(5, 10, 0.25, 1.5)))
xt = rand(40 * 26, 4 * 64)
keep("fast_tile_fixup", pnp.dsg_nlm_denoise(xt, pnp.PatchParams(7, 3, 0.2, 2.0)))
keep("fast_sharded", sharded_dsg_nlm_denoise(rand(300, 200), pnp.PatchParams(7, 10, 0.15, 2.0), 3))
keep("banded_numpy", pnp.dsg_nlm_denoise(np.random.default_rng(1).random((1056, 1000)),
                                         pnp.PatchParams(5, 3, 0.2, 1.5)))
keep("gen_box", pnp.dsg_nlm_denoise(rand(70, 90), pnp.PatchParams(17, 6, 0.2)))
keep("gen_box_r21", pnp.dsg_nlm_denoise(rand(96, 130), pnp.PatchParams(11, 21, 0.15)))
keep("gen_gauss", pnp.dsg_nlm_denoise(rand(60, 70), pnp.PatchParams(19, 4, 0.2, 3.0)))
keep("gen_near", pnp.dsg_nlm_denoise(rand(104, 104), pnp.PatchParams(1, 100, 0.3)))
keep("gen_sharded", sharded_dsg_nlm_denoise(rand(256, 200), pnp.PatchParams(17, 21, 0.15), 2))
xg = rand(2, 90, 140)
keep("gen_frozen", pnp.freeze_guide(xg, pnp.PatchParams(13, 9, 0.2)).apply(rand(2, 90, 140)))
profiling.set_cache_limit(0)
keep("gen_recompute", pnp.dsg_nlm_denoise(xg, pnp.PatchParams(13, 9, 0.2)))
profiling.set_cache_limit(None)
keep("gen_cached", pnp.dsg_nlm_denoise(xg, pnp.PatchParams(13, 9, 0.2)))
keep("nlm", pnp.nlm_denoise(x, pg))
op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
truth = rand(64, 96)
y = (op.apply_device(truth) + 0.02 * rand(32, 48)).contiguous()
prob = pnp.make_sr_problem(op, y, ground_truth=truth)
cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=4, constraint=pnp.UNIT_BOX)
v, recs = pnp.linearized_pnp_admm(prob, cfg, denoiser=pnp.freeze_guide(truth, pg).as_denoiser())
keep("admm_sr", v)
keep("admm_sr_rec", np.array([[r.primal, r.dual, r.psnr, r.objective] for r in recs]))
cfgs = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=2, constraint=pnp.UNIT_BOX,
                        cg_tol=1e-6, cg_max_iters=20)
v, _ = pnp.standard_pnp_admm_cg(prob, cfgs, denoiser=pnp.freeze_guide(truth, pg).as_denoiser())
keep("admm_cg", v)
# SR fast tiles (factor 2, 9x9: interior tiles of a 192 x 224 batch) + boundary
# tiles; a frozen-guide ADMM run at that size (pipelined loop, fused x-update)
ys, xs = rand(2, 96, 112), rand(2, 192, 224)
keep("sr_adjoint_batch", op.adjoint_device(ys))
keep("sr_apply_batch", op.apply_device(xs))
keep("sr_grad_batch", pnp.sr_gradient(op, xs, ys))
prob2 = pnp.make_sr_problem(op, ys, ground_truth=xs)
cfg2 = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=3, constraint=pnp.UNIT_BOX)
v, recs = pnp.linearized_pnp_admm(prob2, cfg2, denoiser=pnp.freeze_guide(xs, pg).as_denoiser())
keep("admm_sr_batch", v)
keep("admm_sr_batch_rec", np.array([[r.primal, r.dual, r.psnr, r.objective] for r in recs]))
torch.cuda.synchronize()
np.savez(sys.argv[1], **out)
print("checks run ok:", len(out), "outputs")
