"""GPU parity of the SR / QIS forward operators against reference goldens and
the float64 oracle (fp32 kernels: absolute 1e-5 on [0,1]-scaled values,
relative 1e-6 for the QIS gradient whose magnitude reaches ~1e7)."""

import numpy as np
import pytest

import oracle
from oracle import forward as ofw

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pnp():
    import paper_1901_06110_b200 as pnp
    return pnp


def test_sr_ops_match_reference(pnp, golden_forward):
    f = golden_forward
    for i in range(5):
        sigma, radius, factor, sym = f[f"s{i}_cfg"]
        op = pnp.SuperResOp(pnp.gaussian_kernel(sigma, int(radius)), int(factor),
                            "symmetric" if sym else "periodic")
        x, y = f[f"s{i}_x"], f[f"s{i}_y"]
        assert np.abs(pnp.sr_apply(op, x) - f[f"s{i}_apply"]).max() < 1e-6
        assert np.abs(pnp.sr_adjoint(op, y) - f[f"s{i}_adjoint"]).max() < 1e-6
        assert np.abs(pnp.sr_gradient(op, x, y) - f[f"s{i}_grad"]).max() < 1e-6
        assert pnp.sr_data_term(op, x, y) == pytest.approx(float(f[f"s{i}_data"]), rel=1e-5)


@pytest.mark.parametrize("factor", [2, 4])
@pytest.mark.parametrize("boundary", ["periodic", "symmetric"])
def test_adjoint_identity(pnp, rng, factor, boundary):
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.5, 4), factor, boundary)
    for _ in range(3):
        x = rng.standard_normal((32, 48))
        y = rng.standard_normal((32 // factor, 48 // factor))
        lhs = float((pnp.sr_apply(op, x) * y).sum())
        rhs = float((x * pnp.sr_adjoint(op, y)).sum())
        scale = np.linalg.norm(pnp.sr_apply(op, x)) * np.linalg.norm(y)
        assert abs(lhs - rhs) <= 1e-5 * scale


def test_sr_large_vs_oracle(pnp, rng):
    k = ofw.gaussian_kernel(1.0, 4)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    x = rng.random((130, 94))
    y = rng.random((65, 47))
    assert np.abs(pnp.sr_gradient(op, x, y) - ofw.sr_gradient(k, 2, "symmetric", x, y)).max() < 2e-6


def test_sr_edge_cases(pnp, rng):
    kk = np.zeros((3, 3))
    kk[0, 1], kk[1, 1] = 0.6, 0.4
    op = pnp.SuperResOp(kk, 2)
    with pytest.raises(ValueError):
        pnp.sr_adjoint(op, np.ones((4, 4)))
    x = rng.random((8, 8))
    ref = ofw.sr_apply(kk, 2, "periodic", x)
    assert np.abs(pnp.sr_apply(op, x) - ref).max() < 1e-6
    opc = pnp.SuperResOp(pnp.gaussian_kernel(1.5, 4), 2, "symmetric")
    assert np.abs(pnp.sr_apply(opc, np.full((12, 12), 0.37)) - 0.37).max() < 1e-6
    with pytest.raises(ValueError):
        pnp.sr_apply(opc, rng.random((9, 8)))
    delta = np.zeros((3, 3))
    delta[1, 1] = 1.0
    op1 = pnp.SuperResOp(delta, 1)
    y = rng.random((6, 6))
    assert pnp.sr_data_term(op1, y, y) == pytest.approx(0.0, abs=1e-12)


def test_sr_simulate_and_power_iteration(pnp, golden_forward):
    f = golden_forward
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = pnp.sr_simulate(f["sim_truth"], op, 5 / 255, seed=102)
    assert np.abs(y - f["sim_y"]).max() < 1e-6
    op2 = pnp.SuperResOp(pnp.gaussian_kernel(1.2, 2), 2, "periodic")
    lam = pnp.power_iteration_lipschitz(op2, (8, 8), iters=400, seed=3)
    k = ofw.gaussian_kernel(1.2, 2)
    cols = []
    for j in range(64):
        e = np.zeros(64)
        e[j] = 1
        cols.append(ofw.sr_apply(k, 2, "periodic", e.reshape(8, 8)).ravel())
    Am = np.array(cols).T
    assert lam == pytest.approx(float(np.linalg.eigvalsh(Am.T @ Am).max()), abs=1e-5)


def test_qis_ops_match_reference(pnp, golden_forward):
    f = golden_forward
    model = pnp.QisModel(16, 16.0)
    counts = pnp.qis_simulate(f["qis_truth"], model, seed=2)
    assert np.array_equal(counts.ones, f["qis_ones"])
    x = f["qis_x"]
    g = pnp.qis_gradient(x, counts, model)
    ref = f["qis_grad"]
    assert np.all(np.abs(g - ref) <= 1e-6 * np.abs(ref) + 1e-5)
    assert pnp.qis_data_term(x, counts, model) == pytest.approx(float(f["qis_data"]), rel=1e-6)
    assert np.array_equal(pnp.qis_initial_estimate(counts), f["qis_x0"])
    c2 = pnp.qis_simulate(oracle_scene16(), pnp.QisModel(128, 64.0), seed=103)
    assert np.array_equal(c2.ones, f["qis128_ones"])


def oracle_scene16():
    from paper_1901_06110_b200 import synth
    return synth.scene(16, 16, 3)


@pytest.mark.parametrize("n", [1, 2, 7, 4097, (1 << 21) + 3])
def test_device_splitmix_uniforms_bit_exact(pnp, n):
    """pnp_splitmix_uniforms == the host stream's next n uniforms, bit for bit
    (counter-based: output k of state s is mix(s + k*GOLDEN))."""
    import torch
    from paper_1901_06110_b200 import _lib as L

    for seed in (0, 12345, (1 << 64) - 1):
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        L.call("pnp_splitmix_uniforms", L.context(0), seed, n, L.ptr(out))
        assert np.array_equal(out.cpu().numpy(), oracle.forward.SplitMix64(seed).uniforms(n))


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (64, 63), (1024, 1025)])
def test_device_sr_noise_matches_host_box_muller(pnp, shape):
    """sr_simulate's noise drawn on the device equals sigma * SplitMix64.normals
    (float64 libm calls: a few ulp); odd sizes exercise the half pair."""
    import torch

    delta = np.zeros((1, 1))
    delta[0, 0] = 1.0
    op = pnp.SuperResOp(delta, 1)
    rng = np.random.default_rng(3)
    x = rng.random(shape)
    sigma = 5 / 255
    clean = x.astype(np.float32).astype(np.float64)
    y = pnp.sr_simulate(x, op, sigma, seed=77)
    n = oracle.forward.SplitMix64(77).normals(x.size).reshape(shape)
    assert y.dtype == np.float64
    assert np.abs((y - clean) - sigma * n).max() <= 1e-15 + 4e-16 * np.abs(n).max()
    yt = pnp.sr_simulate(torch.from_numpy(x).float().cuda(), op, sigma, seed=77)
    assert yt.dtype == torch.float32
    ref32 = (clean + sigma * n).astype(np.float32)
    got = yt.cpu().numpy()
    ulp = np.spacing(np.abs(ref32))
    assert np.all(np.abs(got - ref32) <= ulp)
    assert np.mean(got == ref32) > 0.999
    assert np.array_equal(pnp.sr_simulate(x, op, 0.0, seed=77), clean)


@pytest.mark.parametrize("boundary", ["periodic", "symmetric"])
def test_sr_fast_tiles_bitwise_equal_generic(pnp, rng, boundary):
    """The configs' operator (factor 2, 9x9) takes a compile-time fast path on
    tiles whose staged window needs no boundary map (the adjoint filters only
    the low-res samples); border tiles take the generic path.  Shifting the
    image inside a larger one moves every interior pixel to another tile (and
    tile kind): the interior outputs must be the same bits either way, and
    match the float64 oracle."""
    k = ofw.gaussian_kernel(1.0, 4)
    op = pnp.SuperResOp(pnp.gaussian_kernel(1.0, 4), 2, boundary)
    H, W, s = 192, 224, 20  # s: shift in low-res pixels (40 high-res)
    y = rng.random((3, H // 2, W // 2)).astype(np.float32)
    big = rng.random((3, H // 2 + 2 * s, W // 2 + 2 * s)).astype(np.float32)
    big[:, s:s + H // 2, s:s + W // 2] = y
    import torch
    dev = lambda t: torch.from_numpy(t).cuda()  # noqa: E731 (batched device path)
    a = pnp.sr_adjoint(op, dev(y)).cpu().numpy()
    b = pnp.sr_adjoint(op, dev(big)).cpu().numpy()[:, 2 * s:2 * s + H, 2 * s:2 * s + W]
    m = 8  # high-res rows / columns reached by the boundary from either side
    assert np.array_equal(a[:, m:-m, m:-m], b[:, m:-m, m:-m])
    for i in range(3):
        assert np.abs(a[i] - ofw.sr_adjoint(k, 2, boundary, y[i])).max() < 2e-6
    x = rng.random((3, H, W)).astype(np.float32)
    xb = rng.random((3, H + 4 * s, W + 4 * s)).astype(np.float32)
    xb[:, 2 * s:2 * s + H, 2 * s:2 * s + W] = x
    ra = pnp.sr_apply(op, dev(x)).cpu().numpy()
    rb = pnp.sr_apply(op, dev(xb)).cpu().numpy()[:, s:s + H // 2, s:s + W // 2]
    ml = 4
    assert np.array_equal(ra[:, ml:-ml, ml:-ml], rb[:, ml:-ml, ml:-ml])
    for i in range(3):
        assert np.abs(ra[i] - ofw.sr_apply(k, 2, boundary, x[i])).max() < 2e-6
