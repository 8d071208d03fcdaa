"""The batch CLI's host logic (reference cli.py): INI parsing, overrides,
validation and run-directory fingerprints, against the reference CLI's own
run directories for the same configs (tests/golden/cli/runs.json)."""

import json
import shutil
from pathlib import Path

import pytest

from conftest import GOLDEN

CLI = GOLDEN / "cli"
WORK = Path("/tmp/pnp_cli_golden")   # the absolute path the fixtures were made under


def stage():
    """Recreate the fixture tree at the absolute path the goldens used."""
    shutil.rmtree(WORK, ignore_errors=True)
    WORK.mkdir(parents=True)
    shutil.copy(CLI / "truth.pgm", WORK / "truth.pgm")
    shutil.copy(CLI / "sim_sr__observation.pfm", WORK / "obs.pfm")
    for ini in CLI.glob("*.ini"):
        (WORK / ini.name).write_text(ini.read_text().format(w=WORK))
    return json.loads((CLI / "runs.json").read_text())


@pytest.fixture(scope="module")
def cli():
    from paper_1901_06110_b200 import cli
    return cli


def test_fingerprints_match_reference(cli):
    runs = stage()
    for name, want in runs.items():
        cmd = want.split("-")[0] if not want.startswith("simulate") else "simulate-sr"
        args = cli.build_parser().parse_args([cmd, str(WORK / name)])
        s = cli.load_settings(cmd, args.config, args)
        assert f"{cmd}-{s.fingerprint()}-{s.seed}" == want, name


def test_config_errors_exit_2(cli, tmp_path, capsys):
    bad = tmp_path / "bad.ini"
    bad.write_text("[run]\nproblem = sr\nnonsense = 1\n")
    assert cli.main(["restore", str(bad)]) == 2
    assert "unknown config key" in capsys.readouterr().err
    assert cli.main(["restore", str(tmp_path / "missing.ini")]) == 2
    bad.write_text("[solver]\nsolver = magic\n")
    assert cli.main(["restore", str(bad)]) == 2
    bad.write_text("[run]\ninput = nowhere.pgm\n")
    assert cli.main(["denoise", str(bad)]) == 2
    bad.write_text("[solver]\nconstraint = box:1\n")
    assert cli.main(["restore", str(bad)]) == 2


def test_overrides(cli):
    stage()
    args = cli.build_parser().parse_args(["restore", str(WORK / "restore_sr.ini"), "--iters", "9",
                                          "--lambda", "0.5", "--seed", "4"])
    s = cli.load_settings("restore", args.config, args)
    assert (s.max_iters, s.lam, s.seed) == (9, 0.5, 4)
    assert s.constraint_set().lo == 0.0
