"""GPU linearized PnP-ADMM vs the reference goldens / float64 oracle, plus the
reference's solver properties (solver.py:199-235; tests/test_solver.py).

North-star bar: final ADMM PSNR within 0.02 dB of the float64 oracle."""

import math

import numpy as np
import pytest

import oracle
from oracle import admm as oadmm
from oracle import forward as ofw

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pnp():
    import paper_1901_06110_b200 as pnp
    return pnp


def quadratic_problem(pnp, y):
    return pnp.Problem(shape=y.shape, gradient=lambda x: x - y, x0=np.zeros(y.shape),
                       objective=lambda x: 0.5 * float(((x - y) ** 2).sum()))


def _rec(recs):
    return np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])


def test_sr_dsg_fixed_matches_reference(pnp, golden_admm):
    a = golden_admm
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    prob = pnp.make_sr_problem(op, a["sr_y"], ground_truth=a["sr_truth"])
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=8, freeze_at=3,
                           constraint=pnp.UNIT_BOX, denoiser="dsg-fixed",
                           patch_side=3, window_radius=3, bandwidth=0.1)
    v, recs = pnp.linearized_pnp_admm(prob, cfg)
    ref = a["sr_fixed_rec"]
    got = _rec(recs)
    assert np.abs(v - a["sr_fixed_v"]).max() < 1e-4
    assert np.abs(got[:, 3] - ref[:, 3]).max() < 0.02            # PSNR (dB)
    assert np.allclose(got[:, 4], ref[:, 4], rtol=1e-3)           # objective
    assert np.allclose(got[:, 1:3], ref[:, 1:3], rtol=2e-2, atol=1e-9)


def test_sr_gaussian_frozen_plugin(pnp, golden_admm):
    a = golden_admm
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    prob = pnp.make_sr_problem(op, a["sr_y"], ground_truth=a["sr_truth"])
    params = pnp.PatchParams.from_h(5, 4, 8 / 255, 2.0)
    fz = pnp.freeze_guide(a["sr_gauss_guide"], params)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=6, constraint=pnp.UNIT_BOX)
    v1, r1 = pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
    v2, r2 = pnp.linearized_pnp_admm(prob, cfg, denoiser=lambda im, k: fz.apply(im))
    assert np.abs(v1 - a["sr_gauss_v"]).max() < 1e-4
    assert abs(r1[-1].psnr - a["sr_gauss_rec"][-1, 3]) < 0.02
    assert np.abs(v1 - v2).max() < 1e-6     # host plug-in path == device path


def test_qis_dsg_fixed_matches_reference(pnp, golden_admm):
    a = golden_admm
    model = pnp.QisModel(128, 64.0)
    ones = a["qis_ones"]
    counts = pnp.QisCounts(ones, 128 - ones)
    prob = pnp.make_qis_problem(counts, model, ground_truth=a["qis_truth"])
    alpha = pnp.default_qis_alpha(counts, model)
    assert alpha == float(a["qis_alpha"])
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=alpha, max_iters=6, freeze_at=4,
                           constraint=pnp.UNIT_BOX, denoiser="dsg-fixed",
                           patch_side=3, window_radius=3, bandwidth=0.15)
    v, recs = pnp.linearized_pnp_admm(prob, cfg)
    got, ref = _rec(recs), a["qis_rec"]
    assert np.abs(v - a["qis_v"]).max() < 1e-4
    assert np.abs(got[:, 3] - ref[:, 3]).max() < 0.02
    assert np.allclose(got[:, 4], ref[:, 4], rtol=1e-5)


def test_fixed_point_zero_residuals(pnp):
    y = np.full((6, 6), 0.5)
    prob = pnp.Problem(shape=(6, 6), gradient=lambda x: np.zeros((6, 6)), x0=y)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.0, alpha=1.0, max_iters=3, denoiser="identity")
    v, recs = pnp.linearized_pnp_admm(prob, cfg)
    assert recs[0].primal == 0.0 and recs[0].dual == 0.0
    assert np.array_equal(v, y)


def test_identity_quadratic_converges_to_clamp(pnp, rng):
    y = rng.standard_normal((10, 10)) * 0.8 + 0.5
    cfg = pnp.SolverConfig(rho=1.0, lam=0.0, alpha=1.05, max_iters=500,
                           denoiser="identity", constraint=pnp.Box(0.0, 1.0))
    v, recs = pnp.linearized_pnp_admm(quadratic_problem(pnp, y), cfg)
    assert np.abs(v - np.clip(y, 0.0, 1.0)).max() < 1e-5
    assert len(recs) == 500


def test_multiplier_bookkeeping(pnp, rng):
    y = rng.random((6, 6))
    cfg = pnp.SolverConfig(rho=0.7, lam=0.0, alpha=1.2, max_iters=12, denoiser="identity")
    gaps = []
    pnp.linearized_pnp_admm(quadratic_problem(pnp, y), cfg, denoiser=lambda img, k: 0.9 * img,
                            callback=lambda k, x, v, u: gaps.append((x - v, u)))
    acc = np.zeros((6, 6))
    for gap, u in gaps:
        acc = acc + gap
        assert np.abs(acc - u).max() < 1e-6


def test_divergence_guard_and_early_stop(pnp):
    prob = pnp.Problem(shape=(4, 4), gradient=lambda x: np.full((4, 4), np.nan), x0=np.zeros((4, 4)))
    cfg = pnp.SolverConfig(rho=1.0, lam=0.0, alpha=1.0, max_iters=5, denoiser="identity")
    with pytest.raises(pnp.DivergenceError, match="iteration 1"):
        pnp.linearized_pnp_admm(prob, cfg)
    y = np.full((6, 6), 0.25)
    prob = pnp.Problem(shape=(6, 6), gradient=lambda x: np.zeros((6, 6)), x0=y)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.0, alpha=1.0, max_iters=100, denoiser="identity",
                           stop_tol=1e-12)
    _, recs = pnp.linearized_pnp_admm(prob, cfg)
    assert len(recs) == 1


def test_divergence_same_iteration_as_oracle(pnp):
    """A gradient that turns non-finite on its 3rd call: both raise at k=3."""
    y = np.linspace(0, 1, 64).reshape(8, 8)

    def make_grad():
        calls = {"n": 0}

        def grad(x):
            calls["n"] += 1
            return (x - y) * (np.inf if calls["n"] == 3 else 1.0)
        return grad

    with pytest.raises(oadmm.DivergenceError) as er:
        oracle.linearized_pnp_admm(np.zeros((8, 8)), make_grad(), lambda im, k: im.copy(),
                                   rho=1.0, alpha=1.0, max_iters=20)
    prob = pnp.Problem(shape=(8, 8), gradient=make_grad(), x0=np.zeros((8, 8)))
    cfg = pnp.SolverConfig(rho=1.0, lam=0.0, alpha=1.0, max_iters=20, denoiser="identity")
    with pytest.raises(pnp.DivergenceError) as ei:
        pnp.linearized_pnp_admm(prob, cfg)
    assert str(ei.value) == str(er.value) == "non-finite iterate at iteration 3"


def test_deterministic(pnp):
    from paper_1901_06110_b200 import synth
    truth = synth.scene(48, 48, 5)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.5, 3), 2, "periodic")
    y = pnp.sr_simulate(truth, op, 2 / 255, seed=5)
    cfg = pnp.SolverConfig(rho=0.05, lam=0.0002, alpha=0.3, max_iters=12, freeze_at=5,
                           constraint=pnp.UNIT_BOX, patch_side=3, window_radius=3)
    v1, r1 = pnp.linearized_pnp_admm(pnp.make_sr_problem(op, y, ground_truth=truth), cfg)
    v2, r2 = pnp.linearized_pnp_admm(pnp.make_sr_problem(op, y, ground_truth=truth), cfg)
    assert np.array_equal(v1, v2)
    assert [r.primal for r in r1] == [r.primal for r in r2]


def test_config2_shape_psnr_vs_oracle(pnp):
    """Config-2 pipeline at 128^2 (R=10, P=7 Gaussian, frozen bicubic-ish guide)."""
    from paper_1901_06110_b200 import synth
    truth = synth.scene(128, 128, 2).astype(np.float32).astype(np.float64)
    k = ofw.gaussian_kernel(1.0, 4)
    y = ofw.sr_simulate(truth, k, 2, "symmetric", 5 / 255, 102).astype(np.float32).astype(np.float64)
    guide = np.clip(np.kron(y, np.ones((2, 2))), 0, 1).astype(np.float32).astype(np.float64)
    bw = (8 / 255) / math.sqrt(2)
    fz_ref = oracle.freeze_guide(guide, 7, 10, bw, 2.0)
    x0 = 4 * ofw.sr_adjoint(k, 2, "symmetric", y)
    v_ref, rec_ref = oracle.linearized_pnp_admm(
        x0, lambda x: ofw.sr_gradient(k, 2, "symmetric", x, y), lambda im, kk: fz_ref.apply(im),
        rho=1.0, alpha=1.0, max_iters=30, lo=0.0, hi=1.0, ground_truth=truth)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    fz = pnp.freeze_guide(guide, pnp.PatchParams(7, 10, bw, 2.0))
    prob = pnp.make_sr_problem(op, y, ground_truth=truth)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=30, constraint=pnp.UNIT_BOX)
    v, recs = pnp.linearized_pnp_admm(prob, cfg, denoiser=fz.as_denoiser())
    assert abs(recs[-1].psnr - rec_ref[-1][3]) < 0.02
    assert np.abs(v - v_ref).max() < 1e-4


def test_batched_admm_matches_single(pnp):
    import torch
    from paper_1901_06110_b200 import synth
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    truths = [synth.scene(64, 64, 1000 + i) for i in range(3)]
    ys = [pnp.sr_simulate(t, op, 5 / 255, seed=1100 + i) for i, t in enumerate(truths)]
    p = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=5, constraint=pnp.UNIT_BOX)
    Y = torch.tensor(np.stack(ys), dtype=torch.float32, device="cuda")
    G = torch.clamp(torch.nn.functional.interpolate(Y[:, None], scale_factor=2, mode="bicubic",
                                                    align_corners=False)[:, 0], 0, 1).contiguous()
    T = torch.tensor(np.stack(truths), dtype=torch.float32, device="cuda")
    fzb = pnp.freeze_guide(G, p)
    vb, rb = pnp.linearized_pnp_admm(pnp.make_sr_problem(op, Y, ground_truth=T), cfg,
                                     denoiser=fzb.as_denoiser())
    for i in range(3):
        fz = pnp.freeze_guide(G[i].contiguous(), p)
        vi, ri = pnp.linearized_pnp_admm(
            pnp.make_sr_problem(op, Y[i].contiguous(), ground_truth=T[i].contiguous()), cfg,
            denoiser=fz.as_denoiser())
        assert torch.equal(vb[i], vi)
        # per-image statistics (each image's partials reduced by its own last
        # CTA in the batched fixup): the same doubles as the single solve
        for k in range(len(ri)):
            for f in ("primal", "dual", "psnr", "objective"):
                assert np.asarray(getattr(rb[k], f))[i] == getattr(ri[k], f), (k, f)


@pytest.mark.parametrize("schedule", ["frozen-plugin", "dsg-fixed", "dsg-adaptive", "nlm"])
def test_graph_replay_is_bitwise_eager(pnp, golden_admm, schedule):
    """Iterations captured into one CUDA graph == the eager loop, bit for bit."""
    import torch
    a = golden_admm
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = torch.from_numpy(np.asarray(a["sr_y"], dtype=np.float32)).cuda()
    gt = torch.from_numpy(np.asarray(a["sr_truth"], dtype=np.float32)).cuda()
    prob = pnp.make_sr_problem(op, y, ground_truth=gt)
    den = None
    kw = dict(rho=1.0, lam=0.01, alpha=1.0, max_iters=9, constraint=pnp.UNIT_BOX,
              patch_side=5, window_radius=4, bandwidth=0.1, patch_sigma=1.5)
    if schedule == "frozen-plugin":
        fz = pnp.freeze_guide(a["sr_gauss_guide"], pnp.PatchParams(5, 4, 0.1, 1.5))
        den = fz.as_denoiser()
    else:
        kw.update(denoiser=schedule, freeze_at=3)
    cfg = pnp.SolverConfig(**kw)
    ve, re_ = pnp.linearized_pnp_admm(prob, cfg, denoiser=den, graph=False)
    vg, rg = pnp.linearized_pnp_admm(prob, cfg, denoiser=den, graph=True)
    assert torch.equal(ve, vg)
    for r1, r2 in zip(re_, rg):
        assert (r1.primal, r1.dual, r1.psnr, r1.objective) == (r2.primal, r2.dual, r2.psnr,
                                                               r2.objective)
        assert math.isfinite(r2.time_ms)


def test_fused_admm_steps_match_unfused(pnp, golden_admm):
    """gradient + x-update and frozen apply + u-update fused into one kernel
    epilogue each: x, z, v, u bitwise equal to the separate kernels; stats
    (float64 partial sums in another order) to 1e-12 relative."""
    import torch
    from paper_1901_06110_b200 import _lib as L
    a = golden_admm
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = torch.from_numpy(np.asarray(a["sr_y"], dtype=np.float32)).cuda()
    g = torch.Generator(device="cuda").manual_seed(7)
    H, W = y.shape[0] * 2, y.shape[1] * 2
    x0, v0, u0 = (torch.rand(H, W, device="cuda", generator=g) for _ in range(3))
    u0 = u0 - 0.5
    gt = torch.rand(H, W, device="cuda", generator=g)
    mu, al, rho, lo, hi = 0.5, 1.0, 1.0, 0.0, 1.0
    # unfused
    x1, z1, f1 = x0.clone(), torch.empty_like(x0), torch.zeros(1, dtype=torch.int32, device="cuda")
    grad = op.gradient_device(x1, y, torch.empty_like(x1))
    ctx = L.context(0)
    L.call("pnp_admm_xupdate", ctx, L.ptr(x1), L.ptr(v0), L.ptr(u0), L.ptr(grad), L.ptr(z1),
           x1.numel(), mu, al, rho, lo, hi, L.ptr(f1))
    # fused
    x2, z2, f2 = x0.clone(), torch.empty_like(x0), torch.zeros(1, dtype=torch.int32, device="cuda")
    op.gradient_xupdate_device(x2, y, v0, u0, z2, mu, al, rho, lo, hi, f2)
    assert torch.equal(x1, x2) and torch.equal(z1, z2) and int(f1) == int(f2) == 0
    fz = pnp.freeze_guide(a["sr_gauss_guide"], pnp.PatchParams(5, 4, 0.1, 1.5))
    v1 = fz.apply_device(z1)
    u1 = u0.clone()
    s1 = torch.zeros(1, 4, dtype=torch.float64, device="cuda")
    L.call("pnp_admm_uupdate", ctx, L.ptr(u1), L.ptr(x1), L.ptr(v1), L.ptr(v0), L.ptr(gt), 1,
           H * W, rho, L.ptr(s1), L.ptr(f1))
    v2, u2 = torch.empty_like(z1), u0.clone()
    s2 = torch.zeros(1, 4, dtype=torch.float64, device="cuda")
    fz.apply_admm(z1, v2, u2, x1, v0, gt, rho, s2, f2)
    assert torch.equal(v1, v2) and torch.equal(u1, u2) and int(f1) == int(f2) == 0
    assert torch.allclose(s1[:, :3], s2[:, :3], rtol=1e-12, atol=0)


@pytest.mark.parametrize("case", ["sr-frozen", "sr-dsg-fixed", "sr-batch", "qis-dsg-fixed"])
def test_native_loop_is_bitwise_python_loop(pnp, golden_admm, case):
    """The C++ iteration loop (pnp_admm_run) == the Python loop, bit for bit:
    same fused calls with the same per-iteration arguments."""
    import torch
    a = golden_admm
    kw = dict(rho=1.0, lam=0.01, alpha=1.0, max_iters=11, constraint=pnp.UNIT_BOX,
              patch_side=5, window_radius=4, bandwidth=0.1, patch_sigma=1.5)
    den = None
    if case.startswith("qis"):
        ones = np.asarray(a["qis_ones"])
        counts = pnp.QisCounts(ones, 128 - ones)
        model = pnp.QisModel(128, 64.0)
        prob = pnp.make_qis_problem(counts, model, ground_truth=a["qis_truth"])
        kw.update(alpha=pnp.default_qis_alpha(counts, model), denoiser="dsg-fixed", freeze_at=4)
    else:
        op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
        y = torch.from_numpy(np.asarray(a["sr_y"], dtype=np.float32)).cuda()
        gt = torch.from_numpy(np.asarray(a["sr_truth"], dtype=np.float32)).cuda()
        if case == "sr-batch":
            y = torch.stack([y, y.flip(0)])
            gt = torch.stack([gt, gt.flip(0)])
        prob = pnp.make_sr_problem(op, y, ground_truth=gt)
        if case == "sr-dsg-fixed":
            kw.update(denoiser="dsg-fixed", freeze_at=3)
        else:
            guide = torch.from_numpy(np.asarray(a["sr_gauss_guide"], dtype=np.float32)).cuda()
            if case == "sr-batch":
                guide = torch.stack([guide, guide.flip(0)])
            den = pnp.freeze_guide(guide, pnp.PatchParams(5, 4, 0.1, 1.5)).as_denoiser()
    cfg = pnp.SolverConfig(**kw)
    vp, rp = pnp.linearized_pnp_admm(prob, cfg, denoiser=den, native=False)
    vn, rn = pnp.linearized_pnp_admm(prob, cfg, denoiser=den, native=True)
    if isinstance(vp, torch.Tensor):
        assert torch.equal(vp, vn)
    else:
        assert np.array_equal(vp, vn)
    assert len(rp) == len(rn) == 11
    last = 0.0
    for r1, r2 in zip(rp, rn):
        for f in ("primal", "dual", "psnr", "objective"):
            assert np.array_equal(np.asarray(getattr(r1, f)), np.asarray(getattr(r2, f)),
                                  equal_nan=True), f
        assert math.isfinite(r2.time_ms) and r2.time_ms >= last
        last = r2.time_ms


def test_native_loop_on_a_side_stream(pnp, golden_admm):
    """The pipelined C++ loop on a non-default torch stream (its own side
    stream and events hang off the context): same bits as the Python loop."""
    import torch
    a = golden_admm
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = torch.from_numpy(np.asarray(a["sr_y"], dtype=np.float32)).cuda()
    prob = pnp.make_sr_problem(op, y)
    guide = torch.from_numpy(np.asarray(a["sr_gauss_guide"], dtype=np.float32)).cuda()
    den = pnp.freeze_guide(guide, pnp.PatchParams(5, 4, 0.1, 1.5)).as_denoiser()
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=7, constraint=pnp.UNIT_BOX)
    vp, _ = pnp.linearized_pnp_admm(prob, cfg, denoiser=den, native=False)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        vn, rn = pnp.linearized_pnp_admm(prob, cfg, denoiser=den, native=True)
    s.synchronize()
    assert torch.equal(vp, vn) and len(rn) == 7


@pytest.mark.parametrize("shape,factor,boundary,batch,ksig,krad", [
    ((96, 160), 2, "periodic", 1, 1.0, 4),
    ((128, 96), 4, "symmetric", 3, 1.5, 3),
    ((64, 64), 2, "symmetric", 2, 0.8, 2),
    ((200, 136), 4, "periodic", 1, 2.0, 5),
])
def test_pipelined_loop_bitwise_across_shapes(pnp, shape, factor, boundary, batch, ksig, krad):
    """The pipelined C++ SR loop (next gradient on the side stream, x-update
    fused into the frozen apply's fixup) == the Python loop, bit for bit,
    over factors, boundaries, batches and non-square images."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(shape[0] * 7 + factor)
    H, W = shape
    op = pnp.SuperResOp(pnp.gaussian_kernel(ksig, krad), factor, boundary)
    truth = torch.rand(batch, H, W, device="cuda", generator=g)
    y = torch.stack([op.apply_device(truth[i].contiguous()) for i in range(batch)])
    y = (y + 0.02 * torch.rand(y.shape, device="cuda", generator=g)).contiguous()
    guide = torch.rand(batch, H, W, device="cuda", generator=g)
    if batch == 1:
        y, truth, guide = y[0].contiguous(), truth[0].contiguous(), guide[0].contiguous()
    prob = pnp.make_sr_problem(op, y, ground_truth=truth)
    den = pnp.freeze_guide(guide, pnp.PatchParams(7, 6, 0.15, 2.0)).as_denoiser()
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=9, constraint=pnp.UNIT_BOX)
    vp, rp = pnp.linearized_pnp_admm(prob, cfg, denoiser=den, native=False)
    vn, rn = pnp.linearized_pnp_admm(prob, cfg, denoiser=den, native=True)
    assert torch.equal(vp, vn)
    for r1, r2 in zip(rp, rn):
        for f in ("primal", "dual", "psnr", "objective"):
            assert np.array_equal(np.asarray(getattr(r1, f)), np.asarray(getattr(r2, f)),
                                  equal_nan=True), f
