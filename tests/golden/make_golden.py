"""Generate golden vectors by running the REAL reference (pnprestore).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports pnprestore read-only from /root/reference/pkg/src and writes
small ``.npz`` fixtures next to this file.  The GPU box never runs this
script; tests there read the committed fixtures.  Inputs are seeded
(np.random.default_rng / the package's splitmix scene generator), outputs are
exactly what the reference returns.

Gaussian patch weights are not in the reference.  They are generated here
the way SURVEY.md §7 step 1 prescribes: subclass the reference's
``_DistanceEngine`` so ``map`` returns ``P^2 * sum w_a w_b D`` and install it
as ``_WeightEngine._dist``; the reference's own three sweeps then run
unchanged.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parent.parent))

import pnprestore as ref  # noqa: E402
from pnprestore import denoise as rden  # noqa: E402

from paper_1901_06110_b200 import synth  # noqa: E402


def gauss_taps(P, sigma):
    a = np.arange(P, dtype=np.float64) - (P - 1) // 2
    w = np.exp(-(a * a) / (2.0 * sigma * sigma))
    return w / w.sum()


class GaussDistance(rden._DistanceEngine):
    """P^2 * separable-Gaussian-weighted patch SSD (box when taps = 1/P)."""

    def __init__(self, guide, params, taps):
        super().__init__(guide, params, "direct")
        self.taps = taps

    def map(self, dy, dx):
        a, rh, rw = self._a, self._rh, self._rw
        shifted = self._pad[a + dy:a + dy + rh, a + dx:a + dx + rw]
        d = (self._base - shifted) ** 2
        P, h, w = self.side, self.h, self.w
        out = np.zeros((h, w))
        for py in range(P):
            for px in range(P):
                out += self.taps[py] * self.taps[px] * d[py:py + h, px:px + w]
        return out * (P * P)


def ref_engine(guide, params, sigma):
    guide = ref.validate_image(guide)
    eng = rden._WeightEngine(guide, params)
    if sigma is not None:
        eng._dist = GaussDistance(guide, params, gauss_taps(params.patch_side, sigma))
        eng._cache = {} if eng._cache is not None else None
    return eng


def ref_dsg(image, guide, params, sigma):
    """Reference three sweeps (denoise.py:207-241) + the rowsum map d."""
    image = ref.validate_image(image)
    guide = image if guide is None else ref.validate_image(guide)
    eng = ref_engine(guide, params, sigma)
    g = np.maximum(rden._mass_sweep(eng), rden._MASS_FLOOR)
    m = rden._scale_sweep(eng, g)
    out = rden._filter_sweep(eng, image, g, m)
    # rowsum map: the quantity _scale_sweep maximizes (denoise.py:217-223)
    rs = 1.0 / np.sqrt(g)
    d = np.zeros(g.shape)
    for dy, dx, dst, src in eng.offsets():
        d[dst] += eng.hat(dy, dx) * eng.kernel_map(dy, dx)[dst] * rs[dst] * rs[src]
    assert float(d.max()) == m
    if sigma is None:
        assert np.array_equal(out, ref.dsg_nlm_denoise(image, params, guide=guide))
    return out, d, m, g


def dsg_cases():
    rng = np.random.default_rng(20260808)
    cases = []
    for (h, w, R, P, bw, sigma, own_guide) in [
        (8, 8, 2, 3, 0.25, None, False),
        (9, 13, 3, 5, 0.2, None, False),
        (16, 16, 3, 3, 0.2, None, True),
        (12, 10, 2, 5, 0.3, None, False),
        (24, 20, 5, 5, 0.2, None, False),
        (17, 23, 4, 7, 0.15, None, False),
        (20, 20, 3, 5, 0.2, 1.5, False),
        (21, 18, 5, 7, 0.2, 2.0, True),
        (15, 15, 10, 5, 0.2, 1.5, False),
        (11, 11, 1, 1, 0.2, None, False),
    ]:
        img = rng.random((h, w))
        guide = rng.random((h, w)) if own_guide else None
        cases.append((img, guide, R, P, bw, sigma))
    # scene-based, config-1 shape scaled down, both bandwidth regimes
    clean = synth.scene(64, 64, 1)
    img = synth.noisy(clean, 20 / 255, 2)
    cases.append((img, None, 5, 5, (10 / 255) / math.sqrt(2), 1.5))
    cases.append((img, None, 5, 5, 0.2, 1.5))
    cases.append((img, None, 5, 5, 0.2, None))
    # config-2/3 window at reduced size (R=10, P=7)
    clean = synth.scene(48, 40, 3)
    img = synth.noisy(clean, 10 / 255, 4)
    cases.append((img, None, 10, 7, 0.1, 2.0))
    return cases


def main():
    out = {}
    for i, (img, guide, R, P, bw, sigma) in enumerate(dsg_cases()):
        params = ref.PatchParams(P, R, bw)
        o, d, m, g = ref_dsg(img, guide, params, sigma)
        out[f"c{i}_image"] = img
        out[f"c{i}_guide"] = img if guide is None else guide
        out[f"c{i}_own_guide"] = np.array(guide is not None)
        out[f"c{i}_params"] = np.array([R, P, bw, -1.0 if sigma is None else sigma])
        out[f"c{i}_out"] = o
        out[f"c{i}_d"] = d
        out[f"c{i}_m"] = np.array(m)
        out[f"c{i}_g"] = g
    np.savez_compressed(HERE / "dsg.npz", **out)

    # known answers + dense W + frozen + nlm
    rng = np.random.default_rng(7)
    extra = {}
    extra["w1x2"] = ref.build_dense_weights(np.full((1, 2), 0.9), ref.PatchParams(1, 1, 0.2))
    extra["w1x1"] = ref.build_dense_weights(np.array([[0.4]]), ref.PatchParams(1, 1, 0.2))
    guide = rng.random((7, 8))
    img = rng.random((7, 8))
    p = ref.PatchParams(3, 2, 0.25)
    extra["dense_guide"], extra["dense_img"] = guide, img
    extra["dense_W"] = ref.build_dense_weights(guide, p)
    fz = ref.freeze_guide(guide, p)
    extra["frozen_out"] = fz.apply(img)
    extra["frozen_twice"] = fz.apply(fz.apply(img))
    extra["nlm_out"] = ref.nlm_denoise(img, p, guide=guide)
    extra["nlm_self"] = ref.nlm_denoise(img, ref.PatchParams(5, 3, 0.2))
    np.savez_compressed(HERE / "dsg_extra.npz", **extra)

    # forward operators
    fw = {}
    rng = np.random.default_rng(11)
    ci = 0
    for sigma, radius, factor, boundary, (h, w) in [
        (1.0, 4, 2, "symmetric", (16, 16)),
        (1.0, 4, 2, "periodic", (24, 16)),
        (1.5, 3, 4, "symmetric", (16, 24)),
        (1.5, 3, 4, "periodic", (16, 16)),
        (1.2, 2, 1, "symmetric", (10, 12)),
    ]:
        op = ref.SuperResOp(ref.gaussian_kernel(sigma, radius), factor, boundary)
        x = rng.random((h, w))
        y = rng.random((h // factor, w // factor))
        fw[f"s{ci}_cfg"] = np.array([sigma, radius, factor, 1.0 if boundary == "symmetric" else 0.0])
        fw[f"s{ci}_x"], fw[f"s{ci}_y"] = x, y
        fw[f"s{ci}_apply"] = ref.sr_apply(op, x)
        fw[f"s{ci}_adjoint"] = ref.sr_adjoint(op, y)
        fw[f"s{ci}_grad"] = ref.sr_gradient(op, x, y)
        fw[f"s{ci}_data"] = np.array(ref.sr_data_term(op, x, y))
        ci += 1
    op = ref.SuperResOp(ref.gaussian_kernel(1.0, 4), 2, "symmetric")
    truth = synth.scene(32, 32, 9)
    fw["sim_truth"] = truth
    fw["sim_y"] = ref.sr_simulate(truth, op, 5 / 255, seed=102)
    fw["kernel_1_4"] = ref.gaussian_kernel(1.0, 4)
    r = ref.SplitMix64(1234567)
    fw["splitmix_u64"] = np.array([r.next_uint64() for _ in range(4)], dtype=np.uint64)
    fw["splitmix_uniforms"] = ref.SplitMix64(99).uniforms(1001)
    fw["splitmix_normals"] = ref.SplitMix64(5).normals(999)
    model = ref.QisModel(16, 16.0)
    qtruth = rng.random((12, 10))
    counts = ref.qis_simulate(qtruth, model, seed=2)
    fw["qis_truth"], fw["qis_ones"], fw["qis_zeros"] = qtruth, counts.ones, counts.zeros
    xq = 0.1 + 0.8 * rng.random((12, 10))
    xq[0, 0] = 0.0
    xq[0, 1] = -0.3
    fw["qis_x"] = xq
    fw["qis_grad"] = ref.qis_gradient(xq, counts, model)
    fw["qis_data"] = np.array(ref.qis_data_term(xq, counts, model))
    fw["qis_x0"] = ref.qis_initial_estimate(counts)
    model2 = ref.QisModel(128, 64.0)
    c2 = ref.qis_simulate(synth.scene(16, 16, 3), model2, seed=103)
    fw["qis128_ones"] = c2.ones
    np.savez_compressed(HERE / "forward.npz", **fw)

    # ADMM end-to-end runs (small)
    ad = {}
    truth = synth.scene(32, 32, 2)
    op = ref.SuperResOp(ref.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = ref.sr_simulate(truth, op, 5 / 255, seed=102)
    ad["sr_truth"], ad["sr_y"] = truth, y
    prob = ref.make_sr_problem(op, y, ground_truth=truth)
    cfg = ref.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=8, freeze_at=3,
                           constraint=ref.UNIT_BOX, denoiser="dsg-fixed",
                           patch_side=3, window_radius=3, bandwidth=0.1)
    v, recs = ref.linearized_pnp_admm(prob, cfg)
    ad["sr_fixed_v"] = v
    ad["sr_fixed_rec"] = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
    # config-2 style: frozen Gaussian-weight guide from an upsampled y
    guide = np.clip(np.kron(y, np.ones((2, 2))), 0, 1)
    params = ref.PatchParams(5, 4, (8 / 255) / math.sqrt(2))
    eng = ref_engine(guide, params, 2.0)
    g = np.maximum(rden._mass_sweep(eng), rden._MASS_FLOOR)
    m = rden._scale_sweep(eng, g)
    ad["sr_gauss_guide"] = guide
    cfg2 = ref.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=6,
                            constraint=ref.UNIT_BOX, denoiser="dsg-fixed",
                            patch_side=5, window_radius=4, bandwidth=params.bandwidth)
    v, recs = ref.linearized_pnp_admm(prob, cfg2,
                                      denoiser=lambda im, k: rden._filter_sweep(eng, ref.validate_image(im), g, m))
    ad["sr_gauss_v"] = v
    ad["sr_gauss_rec"] = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
    # QIS, adaptive then frozen
    qt = synth.scene(24, 24, 3)
    model = ref.QisModel(128, 64.0)
    counts = ref.qis_simulate(qt, model, seed=103)
    ad["qis_truth"], ad["qis_ones"] = qt, counts.ones
    qprob = ref.make_qis_problem(counts, model, ground_truth=qt)
    alpha = ref.default_qis_alpha(counts, model)
    ad["qis_alpha"] = np.array(alpha)
    cfg3 = ref.SolverConfig(rho=1.0, lam=0.01, alpha=alpha, max_iters=6, freeze_at=4,
                            constraint=ref.UNIT_BOX, denoiser="dsg-fixed",
                            patch_side=3, window_radius=3, bandwidth=0.15)
    v, recs = ref.linearized_pnp_admm(qprob, cfg3)
    ad["qis_v"] = v
    ad["qis_rec"] = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
    np.savez_compressed(HERE / "admm.npz", **ad)
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)


def cg_goldens():
    """Conjugate gradients and the standard PnP-ADMM + CG baseline
    (solver.py:244-328), run by the reference on small SR problems."""
    cg = {}
    truth = synth.scene(32, 40, 7)
    op = ref.SuperResOp(ref.gaussian_kernel(1.0, 4), 2, "symmetric")
    y = ref.sr_simulate(truth, op, 5 / 255, seed=107)
    prob = ref.make_sr_problem(op, y, ground_truth=truth)
    cg["truth"], cg["y"] = truth, y
    rho = 0.7
    rng = np.random.default_rng(11)
    rhs = prob.atb + rho * rng.standard_normal(truth.shape) * 0.1
    x0 = rng.random(truth.shape)
    cg["rhs"], cg["x0"] = rhs, x0
    for name, tol, its, warm in (("tight", 1e-8, 200, False), ("capped", 1e-12, 7, False),
                                 ("warm", 1e-6, 200, True)):
        res = ref.cg_solve(lambda z: prob.gram(z) + rho * z, rhs, tol, its,
                           x0=x0 if warm else None)
        cg[f"cg_{name}_x"] = res.x
        cg[f"cg_{name}_meta"] = np.array([res.iterations, res.residual, float(res.converged)])
    # standard PnP-ADMM + CG, frozen DSG schedule, box weights
    cfg = ref.SolverConfig(rho=1.0, lam=0.01, alpha=1.0, max_iters=5, freeze_at=3,
                           constraint=ref.UNIT_BOX, denoiser="dsg-fixed", patch_side=3,
                           window_radius=3, bandwidth=0.1, cg_tol=1e-7, cg_max_iters=100)
    v, recs = ref.standard_pnp_admm_cg(prob, cfg)
    cg["std_v"] = v
    cg["std_rec"] = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective] for r in recs])
    cfg2 = ref.SolverConfig(rho=0.5, lam=0.01, alpha=1.0, max_iters=4, constraint=ref.UNIT_BOX,
                            denoiser="identity", cg_tol=1e-6, cg_max_iters=50,
                            cg_warm_start=True)
    v, recs = ref.standard_pnp_admm_cg(prob, cfg2)
    cg["std_warm_v"] = v
    cg["std_warm_rec"] = np.array([[r.index, r.primal, r.dual, r.psnr, r.objective]
                                   for r in recs])
    np.savez_compressed(HERE / "cg.npz", **cg)
    print("cg.npz", (HERE / "cg.npz").stat().st_size)


def io_goldens():
    """PGM / PFM files written by the reference (image.py:169-280) and what its
    reader returns for them, plus malformed inputs and the error it raises."""
    from pnprestore import image as rimg
    d = HERE / "io"
    d.mkdir(exist_ok=True)
    rng = np.random.default_rng(5)
    img = rng.random((7, 11))
    img[0, 0], img[0, 1], img[1, 0] = -0.2, 1.3, 0.5 / 255  # clamping / rounding edges
    rimg.write_image(img, d / "w8.pgm", "pgm8")
    rimg.write_image(img, d / "wf.pfm", "pfm")
    files = {
        "p2_comment.pgm": b"P2\n# a comment\n3 2 # trailing\n7\n0 1 2\n3 4 7\n",
        "p5_16bit.pgm": b"P5 2 2 1000\n" + np.array([0, 1000, 500, 1], ">u2").tobytes(),
        "p5_8bit.pgm": b"P5\n4 1\n255\n" + bytes([0, 128, 255, 7]),
        "pf_be.pfm": b"Pf\n2 2\n1.0\n" + np.array([1, 2, 3, 4], ">f4").tobytes(),
        "bad_magic.pgm": b"P3\n1 1\n255\n0\n",
        "bad_header.pgm": b"P5\n4 x\n255\n\0\0\0\0",
        "truncated.pgm": b"P5\n4 4\n255\n\0\0",
        "bad_maxval.pgm": b"P2\n1 1\n70000\n1\n",
        "ascii_junk.pgm": b"P2\n2 1\n9\n1 q\n",
        "too_big.pgm": b"P2\n2 1\n9\n1 10\n",
    }
    out = {}
    for name, data in files.items():
        (d / name).write_bytes(data)
    for name in sorted(p.name for p in d.iterdir()):
        try:
            out["read_" + name] = rimg.read_image(d / name)
        except rimg.ImageFormatError as exc:
            out["error_" + name] = np.array(type(exc).__name__)
    out["written_image"] = img
    np.savez_compressed(HERE / "io.npz", **out)
    print("io.npz", (HERE / "io.npz").stat().st_size)


CLI_WORK = Path("/tmp/pnp_cli_golden")  # absolute: run-dir fingerprints hash resolved paths

CLI_CONFIGS = {
    "sim_sr.ini": ("simulate-sr", "[run]\nground_truth = {w}/truth.pgm\noutput_dir = {w}/runs\n"
                   "seed = 3\n[sr]\nfactor = 2\nblur_sigma = 1.0\nblur_radius = 4\n"
                   "boundary = symmetric\nnoise_sigma = 0.02\n"),
    "restore_sr.ini": ("restore", "[run]\nobservation = {w}/obs.pfm\nground_truth = {w}/truth.pgm\n"
                       "output_dir = {w}/runs\n[sr]\nfactor = 2\nblur_sigma = 1.0\n"
                       "blur_radius = 4\nboundary = symmetric\n[patch]\npatch_side = 3\n"
                       "window_radius = 3\nbandwidth = 0.1\n[solver]\nrho = 1.0\n"
                       "lambda = 0.01\nalpha = 1.0\nmax_iters = 6\nfreeze_at = 3\n"
                       "constraint = box01\n"),
    "restore_cg.ini": ("restore", "[run]\nobservation = {w}/obs.pfm\nground_truth = {w}/truth.pgm\n"
                       "output_dir = {w}/runs\n[sr]\nfactor = 2\nblur_sigma = 1.0\n"
                       "blur_radius = 4\nboundary = symmetric\n[patch]\npatch_side = 3\n"
                       "window_radius = 3\nbandwidth = 0.1\n[solver]\nsolver = standard-cg\n"
                       "denoiser = dsg-adaptive\nmax_iters = 4\ncg_tol = 1e-6\n"
                       "cg_max_iters = 80\nalpha = 1.0\n"),
    "denoise.ini": ("denoise", "[run]\ninput = {w}/truth.pgm\noutput_dir = {w}/runs\n"
                    "[patch]\npatch_side = 5\nwindow_radius = 4\nbandwidth = 0.15\n"
                    "[solver]\ndenoiser = dsg-adaptive\n"),
}


def cli_goldens():
    """Run the reference CLI (cli.py) on small configs: run-directory names and
    outputs the GPU CLI must reproduce (tests/golden/cli/)."""
    import json
    import shutil
    from pnprestore import cli as rcli
    from pnprestore import image as rimg
    w = CLI_WORK
    shutil.rmtree(w, ignore_errors=True)
    w.mkdir(parents=True)
    rimg.write_image(synth.scene(32, 32, 21), w / "truth.pgm", "pgm8")
    out = HERE / "cli"
    shutil.rmtree(out, ignore_errors=True)
    out.mkdir()
    shutil.copy(w / "truth.pgm", out / "truth.pgm")
    meta = {}
    for name, (cmd, text) in CLI_CONFIGS.items():
        (w / name).write_text(text.format(w=w))
        (out / name).write_text(text)
    for name in ("sim_sr.ini", "restore_sr.ini", "restore_cg.ini", "denoise.ini"):
        cmd = CLI_CONFIGS[name][0]
        before = set((w / "runs").glob("*")) if (w / "runs").exists() else set()
        rc = rcli.main([cmd, str(w / name)])
        assert rc == 0, (name, rc)
        (d,) = set((w / "runs").glob("*")) - before
        meta[name] = d.name
        for f in sorted(d.iterdir()):
            shutil.copy(f, out / f"{name[:-4]}__{f.name}")
        if name == "sim_sr.ini":
            shutil.copy(d / "observation.pfm", w / "obs.pfm")
    (out / "runs.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("cli fixtures", sorted(p.name for p in out.iterdir()))


def helper_goldens():
    """The reference's distance-engine helpers on small seeded inputs:
    pad_symmetric, integral_image, box_sum, patch_distance_map (both methods),
    nlm_kernel, build_dense_weights (helpers.npz)."""
    from pnprestore import image as rimg
    rng = np.random.default_rng(77)
    out = {}
    g = rng.random((14, 17))
    out["g"] = g
    for m in (0, 2, 9):
        out[f"pad{m}"] = rimg.pad_symmetric(g, m)
    ii = rimg.integral_image(g)
    out["ii"] = ii
    out["box"] = np.array([rimg.box_sum(ii, t, l, sz) for t, l, sz in
                           ((0, 0, 3), (2, 5, 7), (10, 12, 4))])
    p = ref.PatchParams(5, 3, 0.21)
    offs = [(0, 0), (2, -1), (-3, 3), (1, 2)]
    out["offs"] = np.array(offs)
    for i, t in enumerate(offs):
        out[f"dmap{i}"] = rden.patch_distance_map(g, t, p)
        out[f"dmap_direct{i}"] = rden.patch_distance_map(g, t, p, method="direct")
    pairs = [((0, 0), (13, 16)), ((4, 5), (6, 9)), ((7, 7), (7, 7)), ((13, 0), (0, 16))]
    out["pairs"] = np.array([[a[0], a[1], b[0], b[1]] for a, b in pairs])
    out["nlmk"] = np.array([ref.nlm_kernel(g, a, b, p) for a, b in pairs])
    gw = rng.random((6, 7))
    out["gw"] = gw
    out["W"] = ref.build_dense_weights(gw, ref.PatchParams(3, 2, 0.25))
    np.savez_compressed(HERE / "helpers.npz", **out)
    print("helpers", sorted(out))


if __name__ == "__main__":
    if "--cg" in sys.argv:   # only the CG / standard-ADMM fixtures
        cg_goldens()
    elif "--helpers" in sys.argv:
        helper_goldens()
    elif "--io" in sys.argv:
        io_goldens()
    elif "--cli" in sys.argv:
        cli_goldens()
    else:
        main()
        cg_goldens()
        io_goldens()
        cli_goldens()
        helper_goldens()
