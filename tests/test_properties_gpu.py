"""Property checks in the spirit of the reference's own test suite
(pnprestore tests/test_denoise.py, test_forward.py, test_solver.py), run on the
device path: dense-operator identities, NLM limits, gradient consistency with
the float64 data terms, descent and monotonicity of the solver's objective.
fp32 kernels against float64 references: absolute 1e-5 on [0,1] data unless
stated."""

import math

import numpy as np
import pytest

from oracle import forward as ofw

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pnp():
    import paper_1901_06110_b200 as pnp
    return pnp


def test_frozen_twice_equals_dense_square(pnp, rng):
    guide = rng.random((8, 9))
    p = pnp.PatchParams(3, 2, 0.25)
    W = pnp.build_dense_weights(guide, p)
    fz = pnp.freeze_guide(guide, p)
    x = rng.random((8, 9))
    twice = fz.apply(fz.apply(x))
    assert np.abs(twice.ravel() - W @ (W @ x.ravel())).max() < 1e-5


def test_nlm_limits(pnp, rng):
    g = rng.random((20, 21))
    p = pnp.PatchParams(3, 3, 0.2)
    c = np.full((20, 21), 0.37)
    assert np.abs(pnp.nlm_denoise(c, p, guide=g) - 0.37).max() < 1e-6
    x = rng.random((20, 21))
    out = pnp.nlm_denoise(x, p)
    assert out.min() >= x.min() - 1e-6 and out.max() <= x.max() + 1e-6
    # vanishing bandwidth: only the self weight survives
    tiny = pnp.nlm_denoise(x, pnp.PatchParams(3, 3, 1e-4))
    assert np.abs(tiny - x).max() < 1e-6


def test_nlm_matches_row_stochastic_dense_operator(pnp, rng):
    """Plain NLM = row-normalized patch-kernel matrix over the clipped window
    (no hat taper: denoise.py:254-269), built here from nlm_kernel."""
    h, w, R = 6, 7, 2
    g = rng.random((h, w))
    p = pnp.PatchParams(3, R, 0.3)
    n = h * w
    K = np.zeros((n, n))
    for sy in range(h):
        for sx in range(w):
            for ry in range(max(0, sy - R), min(h, sy + R + 1)):
                for rx in range(max(0, sx - R), min(w, sx + R + 1)):
                    K[sy * w + sx, ry * w + rx] = pnp.nlm_kernel(g, (sy, sx), (ry, rx), p)
    K /= K.sum(axis=1, keepdims=True)
    x = rng.random((h, w))
    assert np.abs(pnp.nlm_denoise(x, p, guide=g).ravel() - K @ x.ravel()).max() < 1e-5


@pytest.mark.parametrize("boundary", ["symmetric", "periodic"])
def test_sr_gradient_is_derivative_of_data_term(pnp, rng, boundary):
    """GPU gradient vs central differences of the float64 data term."""
    k = ofw.gaussian_kernel(1.0, 2)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 2), 2, boundary)
    x = rng.random((12, 14))
    y = rng.random((6, 7))
    g = pnp.sr_gradient(op, x, y)
    eps = 1e-6
    for (i, j) in [(0, 0), (5, 7), (11, 13), (3, 12)]:
        e = np.zeros_like(x)
        e[i, j] = eps
        fd = (ofw.sr_data_term(k, 2, boundary, x + e, y)
              - ofw.sr_data_term(k, 2, boundary, x - e, y)) / (2 * eps)
        assert g[i, j] == pytest.approx(fd, abs=1e-5)


def test_qis_gradient_is_derivative_and_descent(pnp, rng):
    model = pnp.QisModel(16, 8.0)
    truth = rng.uniform(0.1, 0.9, (10, 11))
    counts = pnp.qis_simulate(truth, model, seed=5)
    x = rng.uniform(0.2, 0.8, (10, 11))
    g = pnp.qis_gradient(x, counts, model)
    eps = 1e-6
    for (i, j) in [(0, 0), (4, 5), (9, 10)]:
        e = np.zeros_like(x)
        e[i, j] = eps
        fd = (ofw.qis_data_term(x + e, counts.ones, counts.zeros, 16, 8.0)
              - ofw.qis_data_term(x - e, counts.ones, counts.zeros, 16, 8.0)) / (2 * eps)
        assert g[i, j] == pytest.approx(fd, rel=1e-4, abs=1e-4)
    # a small step against the gradient lowers the data term
    f0 = ofw.qis_data_term(x, counts.ones, counts.zeros, 16, 8.0)
    f1 = ofw.qis_data_term(x - 1e-4 * g, counts.ones, counts.zeros, 16, 8.0)
    assert f1 < f0


def test_objective_nonincreasing_after_burn_in(pnp):
    """Quadratic SR data term with the identity denoiser (a convex problem):
    after a burn-in the recorded objective does not increase."""
    from paper_1901_06110_b200 import synth
    truth = synth.scene(64, 64, 11)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 2), 2, "symmetric")
    y = pnp.sr_simulate(truth, op, 0.0, seed=0)
    prob = pnp.make_sr_problem(op, y, ground_truth=truth)
    cfg = pnp.SolverConfig(rho=1.0, lam=0.0, alpha=1.0, max_iters=60,
                           constraint=pnp.UNIT_BOX, denoiser="identity")
    _, recs = pnp.linearized_pnp_admm(prob, cfg)
    obj = np.array([r.objective for r in recs])
    assert np.all(np.isfinite(obj))
    tail = obj[20:]
    assert np.all(np.diff(tail) <= 1e-9 * np.abs(tail[:-1]) + 1e-12)
    assert math.isfinite(recs[-1].psnr)
