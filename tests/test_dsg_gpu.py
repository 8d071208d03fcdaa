"""GPU parity of the DSG-NLM kernels against the CPU oracle / reference goldens.

Tolerances (north_star): fp32 GPU vs float64 reference, max abs <= 1e-4 per
denoise on [0,1] intensities.  Integer/bitwise properties (frozen == adaptive,
reruns, batch == single) are checked with array_equal.
"""

import math

import numpy as np
import pytest
import torch

import oracle
from conftest import dsg_case_ids

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def pnp():
    import paper_1901_06110_b200 as pnp
    return pnp


def _params(pnp, g, c):
    R, P, bw, sigma = g[f"{c}_params"]
    return pnp.PatchParams(int(P), int(R), float(bw), None if sigma < 0 else float(sigma))


def test_golden_cases(pnp, golden_dsg):
    g = golden_dsg
    for c in dsg_case_ids(g):
        p = _params(pnp, g, c)
        img = g[f"{c}_image"]
        guide = g[f"{c}_guide"] if bool(g[f"{c}_own_guide"]) else None
        out, d, m = pnp.dsg_nlm_denoise(img, p, guide=guide, return_aux=True)
        assert out.dtype == np.float64 and out.shape == img.shape
        assert np.abs(out - g[f"{c}_out"]).max() <= TOL, c
        assert np.abs(d - g[f"{c}_d"]).max() <= TOL, c
        assert abs(float(m[0]) - float(g[f"{c}_m"])) <= 1e-5 * float(g[f"{c}_m"]), c


def test_known_answers(pnp):
    p = pnp.PatchParams(1, 1, 0.2)
    out = pnp.dsg_nlm_denoise(np.array([[0.3, 0.9]]), p, guide=np.full((1, 2), 0.9))
    assert np.allclose(out, [[(2 * 0.3 + 0.9) / 3, (0.3 + 2 * 0.9) / 3]], atol=1e-6)
    out = pnp.dsg_nlm_denoise(np.array([[0.4]]), p)
    assert np.allclose(out, [[0.4]], atol=1e-7)


@pytest.mark.parametrize("shape,R,P,sigma,bw", [
    ((37, 29), 3, 3, None, 0.2),
    ((64, 64), 5, 5, 1.5, 0.2),
    ((70, 130), 10, 7, 2.0, 0.15),      # crosses tile rows/cols, R=10
    ((100, 66), 10, 7, None, 0.1),
    ((33, 200), 6, 9, 2.5, 0.25),
    ((26, 64), 10, 7, 2.0, 0.2),         # exactly one tile
    ((13, 15), 4, 11, None, 0.3),
    ((40, 45), 21, 3, None, 0.2),        # R larger than the tile height
    ((50, 50), 2, 13, 3.0, 0.2),
    ((24, 30), 3, 15, None, 0.3),
    ((90, 150), 16, 5, 1.5, 0.2),        # R bucket 16
    ((60, 70), 12, 9, None, 0.2),
    ((80, 100), 32, 1, None, 0.2),       # largest R, P = 1
    ((70, 75), 30, 3, 1.0, 0.25),
])
def test_random_vs_oracle(pnp, rng, shape, R, P, sigma, bw):
    img = rng.random(shape)
    guide = rng.random(shape)
    p = pnp.PatchParams(P, R, bw, sigma)
    ref, dref, mref = oracle.dsg_nlm_denoise(img, P, R, bw, guide=guide, patch_sigma=sigma,
                                             return_aux=True)
    out, d, m = pnp.dsg_nlm_denoise(img, p, guide=guide, return_aux=True)
    assert np.abs(out - ref).max() <= TOL
    assert np.abs(d - dref).max() <= TOL
    assert abs(m[0] - mref) <= 1e-5 * mref


def test_config1_shape_both_regimes(pnp):
    from paper_1901_06110_b200 import synth

    img = synth.noisy(synth.scene(256, 256, 1), 20 / 255, 2)
    for bw in ((10 / 255) / math.sqrt(2), 0.2):
        p = pnp.PatchParams(5, 5, bw, 1.5)
        ref, dref, mref = oracle.dsg_nlm_denoise(img, 5, 5, bw, patch_sigma=1.5, return_aux=True)
        out, d, m = pnp.dsg_nlm_denoise(img, p, return_aux=True)
        assert np.abs(out - ref).max() <= TOL
        assert np.abs(d - dref).max() <= TOL
        assert abs(m[0] - mref) <= 1e-5 * mref


def test_frozen_bit_identical_to_adaptive(pnp, rng):
    for shape, R, P, s in [((9, 9), 2, 3, None), ((77, 90), 10, 7, 2.0), ((300, 140), 5, 5, 1.5)]:
        p = pnp.PatchParams(P, R, 0.2, s)
        guide = rng.random(shape)
        img = rng.random(shape)
        fz = pnp.freeze_guide(guide, p)
        assert np.array_equal(fz.apply(img), pnp.dsg_nlm_denoise(img, p, guide=guide))
        assert np.array_equal(fz.apply(guide), pnp.dsg_nlm_denoise(guide, p))
        ref = oracle.freeze_guide(guide, P, R, 0.2, s)
        assert np.abs(fz.apply(img) - ref.apply(img)).max() <= TOL
        assert abs(fz.alpha[0] - ref.m) <= 1e-5 * ref.m


def test_frozen_linear_and_immutable(pnp, rng):
    p = pnp.PatchParams(3, 2, 0.3)
    guide = rng.random((8, 8))
    fz = pnp.freeze_guide(guide, p)
    a, b = rng.random((8, 8)), rng.random((8, 8))
    combo = fz.apply(1.7 * a - 0.4 * b)
    split = 1.7 * fz.apply(a) - 0.4 * fz.apply(b)
    assert np.abs(combo - split).max() < 1e-5
    guide[0, 0] += 1.0
    with pytest.raises(ValueError):
        fz.guide[0, 0] = 0.0
    with pytest.raises(ValueError):
        fz.apply(rng.random((8, 9)))


def test_invariants_fixed_point_mean(pnp, rng):
    p = pnp.PatchParams(3, 2, 0.2)
    out = pnp.dsg_nlm_denoise(np.full((10, 10), 0.5), p, guide=rng.random((10, 10)))
    assert np.abs(out - 0.5).max() < 2e-6
    img = rng.random((140, 150))
    out = pnp.dsg_nlm_denoise(img, pnp.PatchParams(5, 6, 0.2, 1.0))
    assert out.mean() == pytest.approx(img.mean(), rel=2e-6)


def test_deterministic_and_batch_consistent(pnp, rng):
    p = pnp.PatchParams(7, 10, 0.15, 2.0)
    imgs = torch.tensor(rng.random((3, 90, 100)), dtype=torch.float32, device="cuda")
    a = pnp.dsg_nlm_denoise(imgs, p)
    b = pnp.dsg_nlm_denoise(imgs, p)
    assert torch.equal(a, b)
    for i in range(3):
        assert torch.equal(a[i], pnp.dsg_nlm_denoise(imgs[i].contiguous(), p))
    fz = pnp.freeze_guide(imgs, p)
    assert torch.equal(fz.apply(imgs), a)


def test_errors(pnp, rng):
    p = pnp.PatchParams(3, 4, 0.2)
    with pytest.raises(ValueError):          # margin 5 > 4
        pnp.dsg_nlm_denoise(rng.random((4, 8)), p)
    with pytest.raises(ValueError):
        pnp.dsg_nlm_denoise(rng.random((8, 8)), p, guide=rng.random((8, 9)))
    bad = rng.random((8, 8))
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        pnp.dsg_nlm_denoise(bad, p)
    with pytest.raises(ValueError):
        pnp.dsg_nlm_denoise(rng.random((8, 8)), p, distances="sat")
    with pytest.raises(ValueError):
        pnp.dsg_nlm_denoise(rng.random((8,)), p)


def test_nlm_vs_oracle(pnp, golden_extra, rng):
    e = golden_extra
    out = pnp.nlm_denoise(e["dense_img"], pnp.PatchParams(3, 2, 0.25), guide=e["dense_guide"])
    assert np.abs(out - e["nlm_out"]).max() <= TOL
    img = rng.random((50, 70))
    p = pnp.PatchParams(5, 4, 0.15, 1.2)
    ref = oracle.nlm_denoise(img, 5, 4, 0.15, patch_sigma=1.2)
    assert np.abs(pnp.nlm_denoise(img, p) - ref).max() <= TOL


def test_k_cache_is_bitwise_neutral(pnp, rng):
    """k-cache (stored pair weights) vs recompute: identical bits everywhere."""
    from paper_1901_06110_b200 import profiling
    p = pnp.PatchParams(7, 10, 0.15, 2.0)
    x = torch.tensor(rng.random((2, 130, 200)), dtype=torch.float32, device="cuda")
    g = torch.tensor(rng.random((2, 130, 200)), dtype=torch.float32, device="cuda")
    try:
        profiling.set_cache_limit(None)
        a = pnp.dsg_nlm_denoise(x, p, guide=g)
        fa = pnp.freeze_guide(g, p)
        assert pnp._lib.lib.pnp_frozen_cached(fa._h) == 1
        info = fa.cache_info()
        assert info["rows_cached"] == info["tile_rows"] == 5 and info["bytes"] > 0
        ya = fa.apply(x)
        profiling.set_cache_limit(0)
        b = pnp.dsg_nlm_denoise(x, p, guide=g)
        fb = pnp.freeze_guide(g, p)
        assert pnp._lib.lib.pnp_frozen_cached(fb._h) == 0
        assert fb.cache_info() == {"rows_cached": 0, "tile_rows": 5, "bytes": 0}
        yb = fb.apply(x)
        # a budget for 2 of the 5 tile rows: those cached, the rest recomputed
        row_bytes = 220 * 2 * 26 * 4 * 64 * 4
        profiling.set_cache_limit(int(2.5 * row_bytes))
        c = pnp.dsg_nlm_denoise(x, p, guide=g)
        fc = pnp.freeze_guide(g, p)
        assert pnp._lib.lib.pnp_frozen_cached(fc._h) == 1
        assert fc.cache_info()["rows_cached"] == 2
        yc = fc.apply(x)
        tall = torch.tensor(rng.random((700, 130)), dtype=torch.float32).pin_memory()
        st = pnp.DenoiseStream(p, (700, 130))
        profiling.set_cache_limit(int(6.5 * 220 * 26 * 3 * 64 * 4))  # 6 of 27 tile rows
        sc = st.run([tall])[0]
        profiling.set_cache_limit(0)
        sd = st.run([tall])[0]
    finally:
        profiling.set_cache_limit(None)
    assert torch.equal(a, b) and torch.equal(ya, yb) and torch.equal(a, ya)
    assert torch.equal(a, c) and torch.equal(ya, yc)
    assert torch.equal(sc, sd)


def test_denoise_stream_pipeline(pnp, rng):
    """Pipelined H2D / denoise / D2H over a sequence == per-image calls,
    bitwise; a non-finite image is reported by index."""
    p = pnp.PatchParams(7, 10, 0.05, 2.0)
    imgs = [torch.tensor(rng.random((150, 210)), dtype=torch.float32).pin_memory()
            for _ in range(5)]
    outs = pnp.DenoiseStream(p, (150, 210), depth=2).run(imgs)
    for im, o in zip(imgs, outs):
        assert torch.equal(o, pnp.dsg_nlm_denoise(im.cuda(), p).cpu())
    bad = [im.clone() for im in imgs]
    bad[3][10, 20] = float("nan")
    with pytest.raises(ValueError, match="image 3"):
        pnp.DenoiseStream(p, (150, 210)).run(bad)
    # tall enough for the banded first upload (>= 16 tile rows): same bits
    tall = [torch.tensor(rng.random((700, 130)), dtype=torch.float32).pin_memory()
            for _ in range(3)]
    st = pnp.DenoiseStream(p, (700, 130))
    assert st._bands is not None
    for im, o in zip(tall, st.run(tall)):
        assert torch.equal(o, pnp.dsg_nlm_denoise(im.cuda(), p).cpu())
    bad = [im.clone() for im in tall]
    bad[0][600, 5] = float("inf")
    with pytest.raises(ValueError, match="image 0"):
        st.run(bad)


def test_distance_helpers_match_reference_semantics(pnp, rng):
    """pad_symmetric / integral_image bitwise equal to numpy; patch distances
    bitwise equal to the reference's method="direct" shifted-add order
    (restated here), box_sum / nlm_kernel against direct sums
    (reference tests/test_image.py, tests/test_denoise.py)."""
    img = rng.random((13, 17))
    for m in (0, 1, 5, 13):
        assert np.array_equal(pnp.pad_symmetric(img, m), np.pad(img, m, mode="symmetric"))
    with pytest.raises(ValueError):
        pnp.pad_symmetric(img, 14)
    ii = pnp.integral_image(img)
    ref = np.zeros((14, 18))
    np.cumsum(img, axis=0, out=ref[1:, 1:])
    np.cumsum(ref[1:, 1:], axis=1, out=ref[1:, 1:])
    assert np.array_equal(ii, ref)
    assert pnp.box_sum(ii, 2, 3, 4) == pytest.approx(img[2:6, 3:7].sum(), abs=1e-12)
    with pytest.raises(ValueError):
        pnp.box_sum(ii, 10, 0, 4)
    p = pnp.PatchParams(5, 3, 0.2)
    g = rng.random((20, 23))
    half, M = 2, 5
    pad = np.pad(g, M, mode="symmetric")
    for t in [(0, 0), (1, -2), (-3, 3), (3, 0)]:
        got = pnp.patch_distance_map(g, t, p, method="direct")
        a = M - half
        base = pad[a:a + 24, a:a + 27]
        d = base - pad[a + t[0]:a + t[0] + 24, a + t[1]:a + t[1] + 27]
        d *= d
        want = np.zeros((20, 23))
        for py in range(5):
            for px in range(5):
                want += d[py:py + 20, px:px + 23]
        assert np.array_equal(got, want)
        assert np.abs(pnp.patch_distance_map(g, t, p) - want).max() < 1e-9
    with pytest.raises(ValueError):
        pnp.patch_distance_map(g, (4, 0), p)
    assert pnp.nlm_kernel(g, (4, 4), (4, 4), p) == 1.0
    assert pnp.nlm_kernel(np.full((9, 9), 0.3), (1, 2), (7, 5), p) == 1.0
    k = pnp.nlm_kernel(g, (2, 3), (10, 15), p)
    ps, pr = np.pad(g, 2, mode="symmetric")[2:7, 3:8], np.pad(g, 2, mode="symmetric")[10:15, 15:20]
    assert k == pytest.approx(float(np.exp(-((ps - pr) ** 2).sum() / (2 * 25 * 0.04))), abs=1e-14)
    assert k == pytest.approx(pnp.nlm_kernel(g, (10, 15), (2, 3), p), abs=1e-14)


def test_dense_weights_match_reference_golden(pnp, golden_extra, rng):
    """build_dense_weights on the device (float64) against the real
    reference's dense W (golden) and the known 1x1 / 1x2 answers; W x equals
    the denoiser (reference tests/test_denoise.py:186-230)."""
    e = golden_extra
    W = pnp.build_dense_weights(e["dense_guide"], pnp.PatchParams(3, 2, 0.25))
    assert np.abs(W - e["dense_W"]).max() < 1e-12
    assert np.array_equal(pnp.build_dense_weights(np.array([[0.4]]), pnp.PatchParams(1, 1, 0.2)),
                          e["w1x1"])
    assert np.abs(pnp.build_dense_weights(np.full((1, 2), 0.9), pnp.PatchParams(1, 1, 0.2))
                  - e["w1x2"]).max() < 1e-14
    guide = rng.random((9, 11))
    p = pnp.PatchParams(3, 2, 0.2)
    W = pnp.build_dense_weights(guide, p)
    assert np.abs(W - W.T).max() < 1e-12 and np.abs(W.sum(axis=1) - 1).max() < 1e-12
    x = rng.random((9, 11))
    assert np.abs((W @ x.ravel()).reshape(9, 11) - pnp.dsg_nlm_denoise(x, p, guide=guide)).max() < 1e-4
    with pytest.raises(ValueError):
        pnp.build_dense_weights(rng.random((65, 64)), p)


def test_large_numpy_inputs_take_the_pinned_path(pnp, rng):
    """>= 1 M-element numpy arrays go through pinned staging with threaded
    casts: same values as the tensor path, float64 out, non-finite rejected."""
    p = pnp.PatchParams(5, 4, 0.2, 1.5)
    img = rng.random((1100, 1000))
    out = pnp.dsg_nlm_denoise(img, p)
    ref = pnp.dsg_nlm_denoise(torch.tensor(img, dtype=torch.float32, device="cuda"), p)
    assert out.dtype == np.float64 and out.flags.writeable
    assert np.array_equal(out, ref.cpu().numpy().astype(np.float64))
    ro = img.copy()
    ro.setflags(write=False)
    assert np.array_equal(pnp.dsg_nlm_denoise(ro, p), out)
    bad = img.copy()
    bad[700, 3] = np.inf
    with pytest.raises(ValueError):
        pnp.dsg_nlm_denoise(bad, p)
    bad[700, 3] = np.nan
    with pytest.raises(ValueError):
        pnp.dsg_nlm_denoise(bad, p)


def test_numpy_banded_upload_path(pnp, rng, monkeypatch):
    """Large numpy images take the banded path (host cast + upload of band
    j+1 overlapping sweep A of band j, pnp_dsg_band_sweep / _finish): same
    bits as the device-tensor path for float64 and integer inputs, a fresh
    writeable float64 result, ValueError for non-finite input and for finite
    values the float32 device path cannot hold; C-ABI misuse is rejected."""
    from paper_1901_06110_b200 import _lib as L
    from paper_1901_06110_b200 import denoise as D
    calls = []
    real = D._dsg_numpy_banded
    monkeypatch.setattr(D, "_dsg_numpy_banded", lambda *a: calls.append(1) or real(*a))
    p = pnp.PatchParams.from_h(7, 10, 12 / 255, 2.0)
    img = rng.random((1300, 1032))
    out = pnp.dsg_nlm_denoise(img, p)
    assert calls and out.dtype == np.float64 and out.flags.writeable
    ref = pnp.dsg_nlm_denoise(torch.tensor(img, dtype=torch.float32, device="cuda"), p)
    assert np.array_equal(out, ref.cpu().numpy().astype(np.float64))
    assert np.array_equal(pnp.dsg_nlm_denoise(img, p), out)  # rerun: same bits
    ints = rng.integers(0, 256, (1024, 1024)).astype(np.uint8)
    got = pnp.dsg_nlm_denoise(ints, pnp.PatchParams(5, 4, 20.0, 1.5))
    ref = pnp.dsg_nlm_denoise(torch.tensor(ints, dtype=torch.float32, device="cuda"),
                              pnp.PatchParams(5, 4, 20.0, 1.5))
    assert np.array_equal(got, ref.cpu().numpy().astype(np.float64))
    n_calls = len(calls)
    for v in (np.nan, -np.inf, 1e300):
        bad = img.copy()
        bad[1200, 1031] = v
        with pytest.raises(ValueError):
            pnp.dsg_nlm_denoise(bad, p)
    assert len(calls) == n_calls + 3
    # sweeping out of order / finishing early fails loudly
    ctx = L.context(torch.cuda.current_device())
    x = torch.zeros(1300, 1032, device="cuda")
    args = (1300, 1032, p.window_radius, p.patch_side, p._ctaps(), float(p.bandwidth))
    assert L.lib.pnp_dsg_band_sweep(ctx, L.ptr(x), *args, 8, 1) != 0
    assert L.lib.pnp_dsg_band_finish(ctx, L.ptr(x), L.ptr(x), *args) != 0
    assert L.lib.pnp_dsg_band_sweep(ctx, L.ptr(x), *args, 8, 0) == 0
    assert L.lib.pnp_dsg_band_finish(ctx, L.ptr(x), L.ptr(x), *args) != 0
    assert L.lib.pnp_dsg_band_sweep(ctx, L.ptr(x), *args, 8, 2) != 0
    assert L.lib.pnp_dsg_band_sweep(ctx, L.ptr(x), *args, 8, 0) == 0  # restart is allowed
    for j in range(1, 8):
        assert L.lib.pnp_dsg_band_sweep(ctx, L.ptr(x), *args, 8, j) == 0
    assert L.lib.pnp_dsg_band_finish(ctx, L.ptr(x), L.ptr(x), *args) == 0
    torch.cuda.synchronize()


def test_helpers_match_reference_goldens(pnp):
    """Distance-engine helpers against the real reference's outputs
    (tests/golden/helpers.npz, make_golden.py --helpers): pad / SAT / box sums
    and the direct distance maps bitwise, the SAT-based maps and nlm_kernel to
    the reference's own fast-vs-direct agreement, dense W to 1e-12."""
    from conftest import load_golden
    h = load_golden("helpers.npz")
    g = h["g"]
    for m in (0, 2, 9):
        assert np.array_equal(pnp.pad_symmetric(g, m), h[f"pad{m}"])
    ii = pnp.integral_image(g)
    assert np.array_equal(ii, h["ii"])
    boxes = [pnp.box_sum(ii, t, l, sz) for t, l, sz in ((0, 0, 3), (2, 5, 7), (10, 12, 4))]
    assert np.array_equal(np.array(boxes), h["box"])
    p = pnp.PatchParams(5, 3, 0.21)
    for i, t in enumerate(h["offs"]):
        t = (int(t[0]), int(t[1]))
        assert np.array_equal(pnp.patch_distance_map(g, t, p, method="direct"), h[f"dmap_direct{i}"])
        assert np.abs(pnp.patch_distance_map(g, t, p) - h[f"dmap{i}"]).max() < 1e-9
    for (sy, sx, ry, rx), want in zip(h["pairs"], h["nlmk"]):
        got = pnp.nlm_kernel(g, (int(sy), int(sx)), (int(ry), int(rx)), p)
        assert got == pytest.approx(float(want), abs=1e-14)
    W = pnp.build_dense_weights(h["gw"], pnp.PatchParams(3, 2, 0.25))
    assert np.abs(W - h["W"]).max() < 1e-12


def test_two_streams_share_a_context_safely(pnp, rng):
    """One thread issuing denoises / frozen applies on two torch streams uses
    one native context (per thread and device) whose scratch every call
    shares: switching streams orders the new call after the context's work on
    the old stream, so the results equal the serial ones bit for bit."""
    p = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
    xs = [torch.from_numpy(rng.random((1024, 1536)).astype(np.float32)).cuda() for _ in range(4)]
    fz = [pnp.freeze_guide(x, p) for x in xs[:2]]
    ser_d = [pnp.dsg_nlm_denoise(x, p) for x in xs]
    ser_f = [f.apply(x) for f, x in zip(fz, xs[2:])]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    cur = torch.cuda.current_stream()
    for _ in range(3):
        outs = []
        for s in streams:
            s.wait_stream(cur)
        for i, x in enumerate(xs):
            with torch.cuda.stream(streams[i % 2]):
                outs.append(pnp.dsg_nlm_denoise(x, p))
        for i, (f, x) in enumerate(zip(fz, xs[2:])):
            with torch.cuda.stream(streams[i % 2]):
                outs.append(f.apply(x))
        for s in streams:
            cur.wait_stream(s)
        torch.cuda.synchronize()
        for a, b in zip(outs, ser_d + ser_f):
            assert torch.equal(a, b)


def test_frozen_kcache_is_torch_memory(pnp, rng):
    """A frozen guide's pair-weight cache is torch memory held by the
    FrozenGuide: torch counts it while the handle lives, takes it back when
    the handle goes, and re-freezing (old handle alive during the new freeze,
    as in an ADMM loop) recycles blocks instead of growing."""
    p = pnp.PatchParams.from_h(7, 10, 8 / 255, 2.0)
    x = torch.from_numpy(rng.random((1024, 1024)).astype(np.float32)).cuda()
    ref = pnp.dsg_nlm_denoise(x, p)
    torch.cuda.synchronize()
    a0 = torch.cuda.memory_allocated()
    fz = pnp.freeze_guide(x, p)
    info = fz.cache_info()
    assert info["rows_cached"] == info["tile_rows"] and info["bytes"] > 0
    assert torch.cuda.memory_allocated() - a0 >= info["bytes"]
    assert torch.equal(fz.apply(x), ref)
    for _ in range(2):
        fz = pnp.freeze_guide(x, p)
    r1 = torch.cuda.memory_reserved()
    for _ in range(4):
        fz = pnp.freeze_guide(x, p)
        assert torch.equal(fz.apply(x), ref)
    assert torch.cuda.memory_reserved() <= r1 + (64 << 20)  # no new cache-sized blocks
    del fz
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() - a0 < info["bytes"]
