"""Pin the CPU oracle against golden vectors produced by the real reference.

The fixtures in tests/golden/ were written by tests/golden/make_golden.py,
which runs pnprestore itself (reference pkg/src).  If the oracle agrees with
them, it may serve as the checker for the CUDA path.
"""

import math

import numpy as np
import pytest

import oracle
from oracle import admm as oadmm
from oracle import dsg as odsg
from oracle import forward as ofw

from conftest import dsg_case_ids, load_golden


def _params(g, c):
    R, P, bw, sigma = g[f"{c}_params"]
    return int(R), int(P), float(bw), (None if sigma < 0 else float(sigma))


def test_dsg_cases_match_reference(golden_dsg):
    g = golden_dsg
    for c in dsg_case_ids(g):
        R, P, bw, sigma = _params(g, c)
        img = g[f"{c}_image"]
        guide = g[f"{c}_guide"] if bool(g[f"{c}_own_guide"]) else None
        out, d, m = oracle.dsg_nlm_denoise(img, P, R, bw, guide=guide,
                                           patch_sigma=sigma, return_aux=True)
        assert np.abs(out - g[f"{c}_out"]).max() < 1e-11, c
        assert np.abs(d - g[f"{c}_d"]).max() < 1e-11, c
        assert abs(m - float(g[f"{c}_m"])) < 1e-11, c


def test_known_answers(golden_extra):
    e = golden_extra
    assert np.allclose(oracle.dense_weights(np.full((1, 2), 0.9), 1, 1, 0.2), e["w1x2"], atol=1e-14)
    assert np.allclose(e["w1x2"], [[2 / 3, 1 / 3], [1 / 3, 2 / 3]], atol=1e-14)
    assert np.array_equal(oracle.dense_weights(np.array([[0.4]]), 1, 1, 0.2), e["w1x1"])
    out = oracle.dsg_nlm_denoise(np.array([[0.3, 0.9]]), 1, 1, 0.2, guide=np.full((1, 2), 0.9))
    assert np.allclose(out, [[(2 * 0.3 + 0.9) / 3, (0.3 + 2 * 0.9) / 3]], atol=1e-14)


def test_dense_frozen_nlm(golden_extra):
    e = golden_extra
    guide, img = e["dense_guide"], e["dense_img"]
    W = oracle.dense_weights(guide, 3, 2, 0.25)
    assert np.abs(W - e["dense_W"]).max() < 1e-12
    fz = oracle.freeze_guide(guide, 3, 2, 0.25)
    assert np.abs(fz.apply(img) - e["frozen_out"]).max() < 1e-12
    assert np.abs(fz.apply(fz.apply(img)) - e["frozen_twice"]).max() < 1e-12
    assert np.array_equal(fz.apply(img), oracle.dsg_nlm_denoise(img, 3, 2, 0.25, guide=guide))
    assert np.abs(oracle.nlm_denoise(img, 3, 2, 0.25, guide=guide) - e["nlm_out"]).max() < 1e-12
    assert np.abs(oracle.nlm_denoise(img, 5, 3, 0.2) - e["nlm_self"]).max() < 1e-12


def test_dense_invariants(rng):
    for _ in range(3):
        guide = rng.random((7, 9))
        W = oracle.dense_weights(guide, 3, 2, 0.2, patch_sigma=1.0)
        assert np.abs(W - W.T).max() <= 1e-12
        assert np.abs(W.sum(1) - 1).max() <= 1e-10
        ev = np.linalg.eigvalsh(W)
        assert ev.min() >= -1e-10 and ev.max() <= 1 + 1e-10


def test_param_validation():
    with pytest.raises(ValueError):
        odsg.check_params(4, 2, 0.1)
    with pytest.raises(ValueError):
        odsg.check_params(3, 0, 0.1)
    with pytest.raises(ValueError):
        odsg.check_params(3, 2, 0.0)
    with pytest.raises(ValueError):  # pad margin R + p > min(H, W)
        oracle.dsg_nlm_denoise(np.zeros((4, 4)), 3, 4, 0.2)


def test_forward_ops_match_reference(golden_forward):
    f = golden_forward
    i = 0
    while f"s{i}_cfg" in f:
        sigma, radius, factor, sym = f[f"s{i}_cfg"]
        k = ofw.gaussian_kernel(sigma, int(radius))
        b = "symmetric" if sym else "periodic"
        x, y = f[f"s{i}_x"], f[f"s{i}_y"]
        assert np.abs(ofw.sr_apply(k, int(factor), b, x) - f[f"s{i}_apply"]).max() < 1e-14
        assert np.abs(ofw.sr_adjoint(k, int(factor), b, y) - f[f"s{i}_adjoint"]).max() < 1e-14
        assert np.abs(ofw.sr_gradient(k, int(factor), b, x, y) - f[f"s{i}_grad"]).max() < 1e-14
        assert ofw.sr_data_term(k, int(factor), b, x, y) == pytest.approx(float(f[f"s{i}_data"]), rel=1e-13)
        i += 1
    assert i == 5
    k = ofw.gaussian_kernel(1.0, 4)
    assert np.array_equal(k, f["kernel_1_4"])
    y = ofw.sr_simulate(f["sim_truth"], k, 2, "symmetric", 5 / 255, 102)
    assert np.abs(y - f["sim_y"]).max() < 1e-14


def test_splitmix_and_qis_match_reference(golden_forward):
    f = golden_forward
    r = ofw.SplitMix64(1234567)
    assert [r.next_uint64() for _ in range(4)] == [int(v) for v in f["splitmix_u64"]]
    assert np.array_equal(ofw.SplitMix64(99).uniforms(1001), f["splitmix_uniforms"])
    assert np.array_equal(ofw.SplitMix64(5).normals(999), f["splitmix_normals"])
    ones, zeros = ofw.qis_simulate(f["qis_truth"], 16, 16.0, 2)
    assert np.array_equal(ones, f["qis_ones"]) and np.array_equal(zeros, f["qis_zeros"])
    x = f["qis_x"]
    assert np.abs(ofw.qis_gradient(x, ones, zeros, 16, 16.0) - f["qis_grad"]).max() < 1e-9
    assert ofw.qis_data_term(x, ones, zeros, 16, 16.0) == pytest.approx(float(f["qis_data"]), rel=1e-13)
    assert np.array_equal(ofw.qis_initial_estimate(ones, 16), f["qis_x0"])


def test_admm_runs_match_reference(golden_admm):
    a = golden_admm
    k = ofw.gaussian_kernel(1.0, 4)
    y, truth = a["sr_y"], a["sr_truth"]
    x0 = 4 * ofw.sr_adjoint(k, 2, "symmetric", y)
    grad = lambda x: ofw.sr_gradient(k, 2, "symmetric", x, y)  # noqa: E731
    obj = lambda x: ofw.sr_data_term(k, 2, "symmetric", x, y)  # noqa: E731
    den = oadmm.make_denoiser("dsg-fixed", 3, 3, 0.1, lam=0.01, freeze_at=3)
    v, recs = oracle.linearized_pnp_admm(x0, grad, den, rho=1.0, alpha=1.0, max_iters=8,
                                         lo=0.0, hi=1.0, objective=obj, ground_truth=truth)
    assert np.abs(v - a["sr_fixed_v"]).max() < 1e-11
    assert np.allclose(np.array(recs), a["sr_fixed_rec"], rtol=1e-9, atol=1e-14)

    fz = oracle.freeze_guide(a["sr_gauss_guide"], 5, 4, (8 / 255) / math.sqrt(2), 2.0)
    v, recs = oracle.linearized_pnp_admm(x0, grad, lambda im, k_: fz.apply(im), rho=1.0,
                                         alpha=1.0, max_iters=6, lo=0.0, hi=1.0,
                                         objective=obj, ground_truth=truth)
    assert np.abs(v - a["sr_gauss_v"]).max() < 1e-11
    assert np.allclose(np.array(recs), a["sr_gauss_rec"], rtol=1e-9, atol=1e-14)

    ones = a["qis_ones"]
    zeros = 128 - ones
    alpha = 2.0 * 64.0 * float(zeros.max()) / 128
    assert alpha == float(a["qis_alpha"])
    den = oadmm.make_denoiser("dsg-fixed", 3, 3, 0.15, lam=0.01, freeze_at=4)
    v, recs = oracle.linearized_pnp_admm(
        ofw.qis_initial_estimate(ones, 128),
        lambda x: ofw.qis_gradient(x, ones, zeros, 128, 64.0), den, rho=1.0, alpha=alpha,
        max_iters=6, lo=0.0, hi=1.0,
        objective=lambda x: ofw.qis_data_term(x, ones, zeros, 128, 64.0),
        ground_truth=a["qis_truth"])
    assert np.abs(v - a["qis_v"]).max() < 1e-11
    assert np.allclose(np.array(recs), a["qis_rec"], rtol=1e-9, atol=1e-14)


def test_cg_and_standard_admm_match_reference(golden_cg):
    """cg_solve / standard_pnp_admm_cg (solver.py:244-328) against the reference."""
    g = golden_cg
    k = ofw.gaussian_kernel(1.0, 4)
    y, truth = g["y"], g["truth"]
    gram = lambda z: ofw.sr_adjoint(k, 2, "symmetric", ofw.sr_apply(k, 2, "symmetric", z))  # noqa: E731
    rho = 0.7
    for name, tol, its, warm in (("tight", 1e-8, 200, False), ("capped", 1e-12, 7, False),
                                 ("warm", 1e-6, 200, True)):
        x, it, res, conv = oracle.cg_solve(lambda z: gram(z) + rho * z, g["rhs"], tol, its,
                                           x0=g["x0"] if warm else None)
        meta = g[f"cg_{name}_meta"]
        assert it == int(meta[0]) and conv == bool(meta[2])
        assert res == pytest.approx(float(meta[1]), rel=1e-6)
        assert np.abs(x - g[f"cg_{name}_x"]).max() < 1e-10
    atb = ofw.sr_adjoint(k, 2, "symmetric", y)
    obj = lambda x: ofw.sr_data_term(k, 2, "symmetric", x, y)  # noqa: E731
    den = oadmm.make_denoiser("dsg-fixed", 3, 3, 0.1, lam=0.01, freeze_at=3)
    v, recs = oracle.standard_pnp_admm_cg(4 * atb, gram, atb, den, rho=1.0, max_iters=5,
                                          cg_tol=1e-7, cg_max_iters=100, lo=0.0, hi=1.0,
                                          objective=obj, ground_truth=truth)
    assert np.abs(v - g["std_v"]).max() < 1e-10
    assert np.allclose(np.array(recs), g["std_rec"], rtol=1e-8, atol=1e-14)
    v, recs = oracle.standard_pnp_admm_cg(4 * atb, gram, atb, lambda im, k_: im.copy(), rho=0.5,
                                          max_iters=4, cg_tol=1e-6, cg_max_iters=50,
                                          cg_warm_start=True, lo=0.0, hi=1.0, objective=obj,
                                          ground_truth=truth)
    assert np.abs(v - g["std_warm_v"]).max() < 1e-10
    assert np.allclose(np.array(recs), g["std_warm_rec"], rtol=1e-8, atol=1e-14)
