"""The general sweep (csrc/dsg_generic.cuh): box patch distances by running
sums at any odd P <= 63, Gaussian taps beyond the P-templated kernel, search
radii beyond 32 (incl. the full-window variant when the far plane exceeds
shared memory) -- against the float64 oracle (a restatement of
pnprestore/denoise.py pinned to the reference's goldens), plus the bitwise
invariants the reference's tests hold (frozen == adaptive,
tests/test_denoise.py:256-268; batch == single; reruns)."""

import numpy as np
import pytest
import torch

import oracle
from paper_1901_06110_b200 import _lib as L

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def pnp():
    import paper_1901_06110_b200 as pnp
    return pnp


def _path(pnp, H, W, p):
    return L.dsg_geometry(H, W, p.window_radius, p.patch_side, p.is_box)[3]


CASES = [
    # H, W, R, P, bw, sigma, seed
    (40, 52, 3, 11, 0.2, None, 1),     # box from P = 11: the general kernel
    (37, 45, 2, 13, 0.25, None, 2),
    (48, 70, 5, 15, 0.2, None, 3),
    (64, 64, 8, 17, 0.15, None, 4),
    (50, 71, 6, 31, 0.3, None, 5),
    (70, 90, 4, 45, 0.4, None, 6),
    (80, 80, 5, 63, 0.5, None, 7),
    (66, 130, 21, 23, 0.15, None, 8),  # Table-1 radius, W not a multiple of 64
    (90, 75, 40, 5, 0.2, None, 9),     # R > 32, half window (shared far plane)
    (45, 60, 4, 17, 0.2, 3.0, 10),     # Gaussian taps beyond P = 15
    (40, 50, 36, 3, 0.2, 1.0, 11),     # Gaussian, R > 32
    (26, 29, 21, 11, 0.15, None, 12),  # margin = min extent: one tile, cached
]


@pytest.mark.parametrize("H,W,R,P,bw,sigma,seed", CASES)
def test_general_sweep_vs_oracle(pnp, H, W, R, P, bw, sigma, seed):
    rng = np.random.default_rng(seed)
    img = rng.random((H, W))
    p = pnp.PatchParams(P, R, bw, sigma)
    assert _path(pnp, H, W, p) in (1, 2)
    out, d, alpha = pnp.dsg_nlm_denoise(img, p, return_aux=True)
    ref, dref, mref = oracle.dsg_nlm_denoise(img, P, R, bw, patch_sigma=sigma, return_aux=True)
    assert np.abs(out - ref).max() <= TOL
    assert np.abs(d - dref).max() <= 1e-5
    assert abs(float(alpha[0]) - mref) <= 1e-5


def test_full_window_variant_vs_oracle(pnp):
    """A radius whose half-window far plane exceeds shared memory runs the
    full-window (near-only) variant of the general kernel."""
    rng = np.random.default_rng(12)
    H, W, R, P, bw = 104, 110, 100, 1, 0.3
    img = rng.random((H, W))
    p = pnp.PatchParams(P, R, bw)
    assert _path(pnp, H, W, p) == 2
    out, d, alpha = pnp.dsg_nlm_denoise(img, p, return_aux=True)
    ref, dref, mref = oracle.dsg_nlm_denoise(img, P, R, bw, return_aux=True)
    assert np.abs(out - ref).max() <= TOL
    assert np.abs(d - dref).max() <= 1e-5
    fz = pnp.freeze_guide(img, p)
    assert np.array_equal(fz.apply(img), out)


@pytest.mark.parametrize("P,R,sigma", [(17, 21, None), (5, 40, None), (19, 6, 2.5)])
def test_general_bitwise_invariants(pnp, P, R, sigma):
    g = torch.Generator(device="cuda").manual_seed(P * 100 + R)
    x = torch.rand(3, 96, 130, device="cuda", generator=g)
    p = pnp.PatchParams(P, R, 0.2, sigma)
    out, d, a = pnp.dsg_nlm_denoise(x, p, return_aux=True)
    again = pnp.dsg_nlm_denoise(x, p)
    assert torch.equal(out, again)                               # reruns
    fz = pnp.freeze_guide(x, p)
    assert torch.equal(fz.apply(x), out)                         # frozen == adaptive
    for i in range(3):                                           # batch == single
        o, di, ai = pnp.dsg_nlm_denoise(x[i].contiguous(), p, return_aux=True)
        assert torch.equal(o, out[i]) and torch.equal(di, d[i]) and float(ai[0]) == float(a[i])


def test_general_linearity_and_fixed_point(pnp):
    rng = np.random.default_rng(13)
    guide = rng.random((60, 80))
    p = pnp.PatchParams(21, 12, 0.25)
    fz = pnp.freeze_guide(guide, p)
    a, b = rng.random((60, 80)), rng.random((60, 80))
    lhs = fz.apply(2.0 * a - 0.5 * b)
    rhs = 2.0 * fz.apply(a) - 0.5 * fz.apply(b)
    assert np.abs(lhs - rhs).max() < 1e-5
    c = np.full((60, 80), 0.42)
    assert np.abs(fz.apply(c) - c).max() < 1e-6                  # W 1 = 1
    y = fz.apply(a)
    assert abs(float(y.mean()) - float(a.mean())) < 1e-6         # mean preserved


def test_general_nlm_vs_oracle(pnp):
    rng = np.random.default_rng(14)
    img = rng.random((50, 66))
    p = pnp.PatchParams(19, 7, 0.2)
    out = pnp.nlm_denoise(img, p)
    ref = oracle.nlm_denoise(img, 19, 7, 0.2)
    assert np.abs(out - ref).max() <= TOL


def test_general_sharded_equals_single(pnp):
    """Row strips over the general kernel (virtual ranks): same bits."""
    from paper_1901_06110_b200.parallel import sharded_dsg_nlm_denoise
    g = torch.Generator(device="cuda").manual_seed(15)
    x = torch.rand(256, 200, device="cuda", generator=g)
    p = pnp.PatchParams(17, 21, 0.15)
    ref = pnp.dsg_nlm_denoise(x, p)
    for n in (2, 3):
        assert torch.equal(sharded_dsg_nlm_denoise(x, p, n), ref)


@pytest.mark.parametrize("P,R,sigma", [(29, 21, None), (7, 10, 2.0), (3, 2, None)])
def test_direct_distances_match(pnp, P, R, sigma):
    """distances="direct": the brute-force per-pixel path (reference
    denoise.py:291-355) gives the fast path's result (and the oracle's)."""
    rng = np.random.default_rng(P + R)
    img = rng.random((50, 61))
    p = pnp.PatchParams(P, R, 0.2, sigma)
    fast = pnp.dsg_nlm_denoise(img, p)
    brute = pnp.dsg_nlm_denoise(img, p, distances="direct")
    ref = oracle.dsg_nlm_denoise(img, P, R, 0.2, patch_sigma=sigma)
    assert np.abs(brute - fast).max() <= 1e-5
    assert np.abs(brute - ref).max() <= TOL


def test_general_sweep_in_admm_vs_oracle(pnp):
    """Linearized ADMM with the reference's own box weights at P = 11 (the
    general sweep: adaptive iterations, then a frozen guide, dsg-fixed)
    against the float64 oracle."""
    import math

    from oracle import admm as oadmm
    from oracle import forward as ofw
    from paper_1901_06110_b200 import synth
    truth = synth.scene(96, 96, 2)
    k = ofw.gaussian_kernel(1.0, 4)
    y = ofw.sr_simulate(truth, k, 2, "symmetric", 5 / 255, 102)
    P, R, bw = 11, 6, 0.12
    den = oadmm.make_denoiser("dsg-fixed", P, R, bw, freeze_at=4)
    x0 = 4 * ofw.sr_adjoint(k, 2, "symmetric", y)
    v_ref, rec_ref = oadmm.linearized_pnp_admm(
        x0, lambda x: ofw.sr_gradient(k, 2, "symmetric", x, y), den, rho=1.0, alpha=1.0,
        max_iters=8, lo=0.0, hi=1.0, ground_truth=truth)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=8, freeze_at=4,
                           constraint=pnp.UNIT_BOX, denoiser="dsg-fixed", patch_side=P,
                           window_radius=R, bandwidth=bw)
    v, recs = pnp.linearized_pnp_admm(pnp.make_sr_problem(op, y, ground_truth=truth), cfg)
    assert np.abs(v - v_ref).max() < 1e-4
    assert abs(recs[-1].psnr - rec_ref[-1][3]) < 0.02
    assert not math.isnan(recs[-1].psnr)


def test_general_sweep_sharded_sr_admm_bitwise(pnp):
    """Row-strip SR ADMM over the general sweep (box P = 13, virtual ranks)
    equals the single-GPU solver bit for bit."""
    from paper_1901_06110_b200.parallel import sharded_linearized_pnp_admm_sr
    g = torch.Generator(device="cuda").manual_seed(41)
    H, W = 256, 130
    truth = torch.rand(H, W, device="cuda", generator=g)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = (op.apply_device(truth) + 0.02 * torch.randn(H // 2, W // 2, device="cuda",
                                                       generator=g)).contiguous()
    guide = (truth + 0.05 * torch.randn(H, W, device="cuda", generator=g)).clamp(0, 1)
    params = pnp.PatchParams(13, 8, 0.15)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=4, constraint=pnp.UNIT_BOX)
    prob = pnp.make_sr_problem(op, y, ground_truth=truth)
    v1, _ = pnp.linearized_pnp_admm(prob, cfg,
                                    denoiser=pnp.freeze_guide(guide, params).as_denoiser())
    v2, _ = sharded_linearized_pnp_admm_sr(op, y, guide, params, cfg, 2, ground_truth=truth)
    assert torch.equal(v1, v2)


@pytest.mark.parametrize("P,R,sigma,shape", [(17, 21, None, (2, 90, 140)),
                                             (11, 21, None, (256, 256)),
                                             (19, 6, 2.5, (70, 100)),
                                             (11, 21, None, (26, 29)),
                                             (29, 21, None, (3, 50, 200))])
def test_general_kcache_is_bitwise_neutral(pnp, P, R, sigma, shape):
    """The general sweep's pair-weight cache (sweep A stores, sweep B and
    frozen applies stream it): same bits as recomputing, adaptive and frozen."""
    from paper_1901_06110_b200 import profiling
    g = torch.Generator(device="cuda").manual_seed(P + R)
    x = torch.rand(*shape, device="cuda", generator=g)
    y = torch.rand(*shape, device="cuda", generator=g)
    p = pnp.PatchParams(P, R, 0.2, sigma)
    out, d, a = pnp.dsg_nlm_denoise(x, p, return_aux=True)
    fz = pnp.freeze_guide(x, p)
    info = fz.cache_info()
    assert info["rows_cached"] == info["tile_rows"] and info["bytes"] > 0
    fy = fz.apply(y)
    profiling.set_cache_limit(0)
    try:
        out0, d0, a0 = pnp.dsg_nlm_denoise(x, p, return_aux=True)
        fz0 = pnp.freeze_guide(x, p)
        assert fz0.cache_info()["rows_cached"] == 0
        fy0 = fz0.apply(y)
    finally:
        profiling.set_cache_limit(None)
    assert torch.equal(out, out0) and torch.equal(d, d0) and torch.equal(a, a0)
    assert torch.equal(fy, fy0)
