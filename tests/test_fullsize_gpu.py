"""Parity at BASELINE.json's full sizes (config 4: 8192^2, R=10, P=7
Gaussian sigma_p=2, h=12/255; config 5: a 64 x 1024^2 batch) through
properties that do not need a full-size oracle run:

* local parity: d and W x of the full-size denoise on windows (interior,
  edges, corners) against the float64 oracle run on a crop with a 2R+p
  margin -- d(s) depends on the guide within 2R+p of s only, and W x on d, Kx
  and the global alpha, which the GPU returns (reference denoise.py:207-241);
* doubly stochastic: W 1 = 1 (constant image is a fixed point), and the mean
  is preserved;
* the k cache (stored pair weights) is bitwise neutral at full size;
* batched images equal the single-image calls bit for bit (config 5).
"""

import math

import numpy as np
import pytest
import torch

import oracle
from oracle import dsg as odsg

pytestmark = pytest.mark.gpu

N4, R, P, SIG = 8192, 10, 7, 2.0
BW = (12 / 255) / math.sqrt(2.0)
TOL = 1e-4


@pytest.fixture(scope="module")
def pnp():
    import paper_1901_06110_b200 as pnp
    return pnp


@pytest.fixture(scope="module")
def big(pnp):
    """Config-4-sized noisy image (seeded, on device) + its denoise with aux."""
    g = torch.Generator(device="cuda").manual_seed(4)
    # piecewise-smooth content + noise 25/255, in the config's value range
    yy = torch.linspace(0, 1, N4, device="cuda")[:, None]
    xx = torch.linspace(0, 1, N4, device="cuda")[None, :]
    clean = 0.15 + 0.7 * (0.5 + 0.5 * torch.sin(6.0 * xx + 3.0 * yy) * torch.cos(5.0 * yy))
    clean = torch.where((xx - 0.3) ** 2 + (yy - 0.6) ** 2 < 0.04, 0.9, clean)
    x = (clean + (25 / 255) * torch.randn(N4, N4, device="cuda", generator=g)).contiguous()
    p = pnp.PatchParams(P, R, BW, SIG)
    out, d, alpha = pnp.dsg_nlm_denoise(x, p, return_aux=True)
    torch.cuda.synchronize()
    return x, p, out, d, float(alpha[0])


@pytest.mark.parametrize("r0,c0", [(4000, 4100), (0, 0), (0, 6000), (N4 - 48, N4 - 48),
                                   (5000, N4 - 48), (3001, 0)])
def test_local_parity_full_size(big, r0, c0):
    x, p, out, d, alpha = big
    S, M = 48, 2 * R + (P - 1) // 2
    a0, a1 = max(0, r0 - M), min(N4, r0 + S + M)
    b0, b1 = max(0, c0 - M), min(N4, c0 + S + M)
    crop = x[a0:a1, b0:b1].double().cpu().numpy()
    g, dref, _, e = odsg.dsg_sweeps(crop, P, R, BW, patch_sigma=SIG)
    wx = odsg.filter_sweep(e, crop, g, alpha)   # GPU's global alpha
    sl = (slice(r0 - a0, r0 - a0 + S), slice(c0 - b0, c0 - b0 + S))
    d_gpu = d[r0:r0 + S, c0:c0 + S].double().cpu().numpy()
    o_gpu = out[r0:r0 + S, c0:c0 + S].double().cpu().numpy()
    assert np.abs(d_gpu - dref[sl]).max() <= 1e-5
    assert np.abs(o_gpu - wx[sl]).max() <= TOL


def test_alpha_is_max_row_sum(big):
    _, _, _, d, alpha = big
    assert float(d.max()) == alpha
    assert alpha > 0.0


def test_doubly_stochastic_full_size(pnp):
    p = pnp.PatchParams(P, R, BW, SIG)
    c = torch.full((N4, N4), 0.37, device="cuda")
    assert torch.equal(pnp.dsg_nlm_denoise(c, p), c) or \
        float((pnp.dsg_nlm_denoise(c, p) - c).abs().max()) < 1e-6


def test_mean_preserved_full_size(big):
    x, _, out, _, _ = big
    mx, mo = float(x.double().mean()), float(out.double().mean())
    assert abs(mx - mo) < 2e-6


def test_k_cache_neutral_full_size(pnp, big):
    from paper_1901_06110_b200 import profiling
    x, p, out, _, _ = big
    try:
        profiling.set_cache_limit(0)
        ref = pnp.dsg_nlm_denoise(x, p)
    finally:
        profiling.set_cache_limit(None)
    assert torch.equal(ref, out)


def test_kcache_memory_is_torchs(pnp, big):
    """The adaptive k cache of an 8192^2 denoise (59 GB) comes from torch's
    caching allocator and goes back to it when the call returns: nothing
    large stays hidden in the library, and torch can hand 100 GB out
    right after the call."""
    from paper_1901_06110_b200 import profiling
    x, p, out, _, _ = big
    profiling.trim()
    torch.cuda.synchronize()
    assert torch.equal(pnp.dsg_nlm_denoise(x, p), out)
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    hidden = (total - free) - torch.cuda.memory_reserved()
    assert hidden < (4 << 30), hidden / 2 ** 30          # context + small scratch only
    t = torch.empty(100 << 30, dtype=torch.uint8, device="cuda")
    t[-1] = 1
    del t
    torch.cuda.empty_cache()


def test_config5_batch_equals_single(pnp):
    """Config-5 shape: a batch of 1024^2 images denoised in one call (per-image
    alpha) == each image on its own, bitwise; frozen batch apply too."""
    B, n = 6, 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand(B, n, n, device="cuda", generator=g)
    p = pnp.PatchParams(P, R, (8 / 255) / math.sqrt(2.0), SIG)
    outb, db, ab = pnp.dsg_nlm_denoise(x, p, return_aux=True)
    fz = pnp.freeze_guide(x, p)
    yb = fz.apply(x)
    for i in range(B):
        o, d, a = pnp.dsg_nlm_denoise(x[i].contiguous(), p, return_aux=True)
        assert torch.equal(o, outb[i]) and torch.equal(d, db[i]) and float(a[0]) == float(ab[i])
    assert torch.equal(yb, outb)
