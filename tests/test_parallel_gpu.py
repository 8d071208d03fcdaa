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
