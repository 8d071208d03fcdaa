"""Standard PnP-ADMM + conjugate-gradients baseline on the GPU vs the
reference goldens (solver.py:244-328; tests/golden/cg.npz from the real
reference).  The native CG runs in fp32 with float64 dot products, so its
iterates are compared with tolerances, not bitwise."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pnp():
    import paper_1901_06110_b200 as pnp
    return pnp


def _op(pnp):
    return pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")


def test_native_cg_matches_reference(pnp, golden_cg):
    g = golden_cg
    op = _op(pnp)
    rhs = torch.tensor(g["rhs"], dtype=torch.float32, device="cuda")
    for name, tol, its, warm in (("tight", 1e-8, 200, False), ("capped", 1e-12, 7, False),
                                 ("warm", 1e-6, 200, True)):
        x = torch.tensor(g["x0"], dtype=torch.float32, device="cuda")
        it, res, st = op.cg_device(rhs, x, 0.7, tol, its, warm)
        ref_x, meta = g[f"cg_{name}_x"], g[f"cg_{name}_meta"]
        assert st == [0]
        assert np.abs(x.cpu().numpy() - ref_x).max() <= 2e-5 * max(1.0, np.abs(ref_x).max())
        if name == "capped":
            assert it[0] == 7 and res[0] == pytest.approx(float(meta[1]), rel=1e-3)
        if name == "warm":   # fp32 reaches 1e-6 within a couple of iterations of float64
            assert abs(it[0] - int(meta[0])) <= 2 and res[0] <= 1e-6


def test_gram_operator(pnp, golden_cg):
    op = _op(pnp)
    x = torch.tensor(golden_cg["x0"], dtype=torch.float32, device="cuda")
    out = op.gram_device(x, torch.empty_like(x), 0.7)
    ref = op.adjoint_device(op.apply_device(x)) + 0.7 * x
    assert float((out - ref).abs().max()) < 1e-6


def test_generic_cg_solve(pnp, golden_cg):
    g = golden_cg
    op = _op(pnp)
    apply = lambda z: op.gram_device(z, torch.empty_like(z), 0.7)  # noqa: E731
    rhs = torch.tensor(g["rhs"], dtype=torch.float32, device="cuda")
    r = pnp.cg_solve(apply, rhs, 1e-6, 200)
    assert r.converged and r.residual <= 1e-6
    assert np.abs(r.x.cpu().numpy() - g["cg_tight_x"]).max() < 1e-4
    z = pnp.cg_solve(lambda v: v, np.zeros((4, 4)), 1e-10, 5)   # reference: zero rhs
    assert z.iterations == 0 and z.converged and not z.x.any()
    with pytest.raises(ValueError):
        pnp.cg_solve(apply, rhs, 0.0, 5)


def test_breakdown_and_batch(pnp, golden_cg):
    op = _op(pnp)
    rhs = torch.tensor(golden_cg["rhs"], dtype=torch.float32, device="cuda")
    x = torch.zeros_like(rhs)
    _, _, st = op.cg_device(rhs, x, -5.0, 1e-6, 50, False)   # A^T A - 5 I: indefinite
    assert st == [2]
    # batch of 3 independent systems == one at a time
    rb = torch.stack([rhs, 2 * rhs, torch.zeros_like(rhs)])
    xb = torch.zeros_like(rb)
    it, res, st = op.cg_device(rb, xb, 0.7, 1e-6, 200, False)
    assert st == [0, 0, 0] and it[2] == 0 and res[2] == 0.0 and not bool(xb[2].any())
    for i in range(2):
        xi = torch.zeros_like(rhs)
        it_i, res_i, _ = op.cg_device(rb[i].contiguous(), xi, 0.7, 1e-6, 200, False)
        assert it_i[0] == it[i] and torch.equal(xi, xb[i])


def test_standard_admm_matches_reference(pnp, golden_cg):
    g = golden_cg
    op = _op(pnp)
    prob = pnp.make_sr_problem(op, g["y"], ground_truth=g["truth"])
    cfg = pnp.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=5, freeze_at=3,
                           constraint=pnp.UNIT_BOX, denoiser="dsg-fixed", patch_side=3,
                           window_radius=3, bandwidth=0.1, cg_tol=1e-7, cg_max_iters=100)
    v, recs = pnp.standard_pnp_admm_cg(prob, cfg)
    rec = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
    assert np.abs(v - g["std_v"]).max() < 1e-4
    assert np.abs(rec[:, 3] - g["std_rec"][:, 3]).max() < 0.02
    assert np.allclose(rec[:, 4], g["std_rec"][:, 4], rtol=1e-3)
    cfg2 = pnp.SolverConfig(rho=0.5, lam=0.01, alpha=1.0, max_iters=4, constraint=pnp.UNIT_BOX,
                            denoiser="identity", cg_tol=1e-6, cg_max_iters=50,
                            cg_warm_start=True)
    v, recs = pnp.standard_pnp_admm_cg(prob, cfg2)
    rec = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
    assert np.abs(v - g["std_warm_v"]).max() < 1e-4
    assert np.abs(rec[:, 3] - g["std_warm_rec"][:, 3]).max() < 0.02
    with pytest.raises(ValueError):
        pnp.standard_pnp_admm_cg(pnp.Problem(shape=(4, 4), gradient=lambda x: x,
                                             x0=np.zeros((4, 4))), cfg)
