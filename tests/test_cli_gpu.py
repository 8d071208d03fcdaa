"""The batch CLI end to end on the GPU backend vs the reference CLI's outputs
for the same configs (tests/golden/cli/): run-directory names, observation /
restored / denoised images (within the fp32 tolerances) and log.csv."""

import json

import numpy as np
import pytest

from test_cli_cpu import CLI, WORK, stage

pytestmark = pytest.mark.gpu


def _log(path):
    lines = path.read_text().splitlines()
    assert lines[0] == "iter,primal,dual,psnr,time_ms,objective"
    return np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])


def test_cli_commands_match_reference():
    from paper_1901_06110_b200 import cli, read_image
    runs = stage()
    obs = WORK / "obs.pfm"
    for name, cmd in (("sim_sr.ini", "simulate-sr"), ("restore_sr.ini", "restore"),
                      ("restore_cg.ini", "restore"), ("denoise.ini", "denoise")):
        if name == "sim_sr.ini":
            obs.unlink()  # restore must read this run's own observation
        assert cli.main([cmd, str(WORK / name)]) == 0, name
        d = WORK / "runs" / runs[name]
        assert d.is_dir(), name
        tag = name[:-4]
        for f in d.iterdir():
            ref = CLI / f"{tag}__{f.name}"
            assert ref.exists(), f.name
            if f.suffix == ".pfm":
                err = np.abs(read_image(f) - read_image(ref)).max()
                assert err <= (2e-6 if cmd == "simulate-sr" else 1e-4), (name, f.name, err)
            elif f.suffix == ".pgm":
                assert np.abs(read_image(f) - read_image(ref)).max() <= 1.0 / 255 + 1e-12
            elif f.name == "log.csv":
                got, want = _log(f), _log(ref)
                assert got.shape == want.shape
                assert np.array_equal(got[:, 0], want[:, 0])
                assert np.abs(got[:, 3] - want[:, 3]).max() < 0.02      # PSNR (dB)
                assert np.allclose(got[:, 5], want[:, 5], rtol=1e-3)    # objective
                assert not got[:, 4].any()                              # no --timing
        if name == "sim_sr.ini":
            obs.write_bytes((d / "observation.pfm").read_bytes())
    assert json.loads((CLI / "runs.json").read_text()) == runs


def test_denoise_oracle_flag(tmp_path, capsys):
    """denoise --oracle: the dense-W brute force (built on the device) agrees
    with the fast denoiser; too-large images and non-DSG denoisers are config
    errors (reference cli.py denoise --oracle)."""
    import numpy as np

    from paper_1901_06110_b200 import cli, write_image
    rng = np.random.default_rng(3)
    write_image(rng.random((24, 30)), tmp_path / "small.pfm", "pfm")
    write_image(rng.random((70, 70)), tmp_path / "big.pfm", "pfm")
    ini = tmp_path / "d.ini"
    ini.write_text(f"[run]\ninput = small.pfm\noutput_dir = {tmp_path}/runs\n"
                   "[patch]\npatch_side = 3\nwindow_radius = 3\nbandwidth = 0.2\n"
                   "[solver]\ndenoiser = dsg-adaptive\n")
    assert cli.main(["denoise", str(ini), "--oracle"]) == 0
    line = [ln for ln in capsys.readouterr().out.splitlines() if "oracle max-abs diff" in ln][0]
    assert float(line.split("=")[1]) < 1e-4
    assert cli.main(["denoise", str(ini), "--oracle", "--denoiser", "nlm"]) == 2
    ini.write_text(ini.read_text().replace("small.pfm", "big.pfm"))
    assert cli.main(["denoise", str(ini), "--oracle"]) == 2


def test_bench_denoiser_default_shape(tmp_path):
    """bench-denoiser with the reference's default bench section (256^2,
    R = 21, P in {11, 17, 23, 29}, bandwidth 0.15; cli.py:115-120): all four
    rows written, GPU times within the reference's criterion-4 ratio (< 2,
    tests/test_acceptance.py:131-153); the brute-force columns the GPU does not
    time are nan."""
    from paper_1901_06110_b200 import cli
    ini = tmp_path / "b.ini"
    ini.write_text(f"[run]\noutput_dir = {tmp_path}/runs\n[bench]\nrepeats = 5\n")
    assert cli.main(["bench-denoiser", str(ini)]) == 0
    (d,) = list((tmp_path / "runs").iterdir())
    rows = (d / "bench.csv").read_text().splitlines()
    assert rows[0] == "np,fast_s,brute_s,speedup"
    vals = [r.split(",") for r in rows[1:]]
    assert [int(v[0]) for v in vals] == [11, 17, 23, 29]
    t = [float(v[1]) for v in vals]
    assert max(t) / min(t) < 2.0, t
    brute = [float(v[2]) for v in vals]
    speed = [float(v[3]) for v in vals]
    assert all(b > f for b, f in zip(brute, t)) and speed[-1] > speed[0] > 1.0
