"""Row-strip sharded DSG-NLM (virtual shards on one GPU, same algorithm and
exchanges as the multi-GPU run) is bit-identical to the single-GPU call."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("H,W,R,P,sigma,N", [
    (300, 200, 10, 7, 2.0, 2),
    (300, 200, 10, 7, 2.0, 3),
    (160, 70, 5, 5, 1.5, 4),
    (600, 130, 21, 3, None, 3),
    (1040, 256, 10, 7, 2.0, 8),
])
@pytest.mark.parametrize("kcache", [True, False])
def test_virtual_shards_bit_identical(H, W, R, P, sigma, N, kcache):
    import paper_1901_06110_b200 as pnp
    from paper_1901_06110_b200.parallel import sharded_dsg_nlm_denoise
    g = torch.Generator(device="cuda").manual_seed(H * W + N)
    x = torch.rand(H, W, device="cuda", generator=g)
    p = pnp.PatchParams(P, R, 0.15, sigma)
    ref, d, m = pnp.dsg_nlm_denoise(x, p, return_aux=True)
    out = sharded_dsg_nlm_denoise(x, p, N, kcache=kcache)
    assert torch.equal(out, ref)


@pytest.mark.parametrize("H,W,N,P,R", [(312, 200, 2, 7, 10), (416, 130, 3, 5, 4),
                                       (520, 96, 4, 7, 10)])
@pytest.mark.parametrize("kcache", [True, False])
def test_sharded_sr_admm_matches_single(H, W, N, P, R, kcache):
    """Row-strip SR ADMM with a frozen guide (virtual ranks) == the single-GPU
    solver: v bitwise; records to float64 summation-order tolerance."""
    import paper_1901_06110_b200 as pnp
    from paper_1901_06110_b200.parallel import sharded_linearized_pnp_admm_sr
    g = torch.Generator(device="cuda").manual_seed(H + N)
    truth = torch.rand(H, W, device="cuda", generator=g)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = op.apply_device(truth) + 0.02 * torch.randn(H // 2, W // 2, device="cuda", generator=g)
    guide = (truth + 0.05 * torch.randn(H, W, device="cuda", generator=g)).clamp(0, 1)
    params = pnp.PatchParams(P, R, 0.1, 1.5)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=5, constraint=pnp.UNIT_BOX)
    prob = pnp.make_sr_problem(op, y.contiguous(), ground_truth=truth)
    v1, recs = pnp.linearized_pnp_admm(prob, cfg, denoiser=pnp.freeze_guide(guide, params)
                                       .as_denoiser())
    v2, recs2 = sharded_linearized_pnp_admm_sr(op, y, guide, params, cfg, N,
                                               ground_truth=truth, kcache=kcache)
    assert torch.equal(v1, v2)
    ref = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
    got = np.array(recs2)
    assert np.allclose(got, ref, rtol=1e-9, atol=0)
