"""Kernel hygiene without compute-sanitizer (closed on this pool): the
PNP_CHECKS + PNP_JITTER debug build of the library (device asserts on every
shared-memory index and global write of the sweeps; a pseudo-random pause
per warp before every barrier, so warps reach the ordered flushes in a
different order each run) must run every device path without an assert and
produce the product library's bits, twice."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
VARIANT = ROOT / "build" / "var_checks" / "libpnpb200.so"


def _run(out, lib=None):
    env = dict(os.environ)
    if lib:
        env["PNP_B200_LIB"] = str(lib)
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "checks_run.py"), str(out)],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    return dict(np.load(out))


def test_debug_build_asserts_and_jitter_bitwise(tmp_path):
    if not VARIANT.exists():
        subprocess.run([sys.executable, str(ROOT / "scripts" / "build_variant.py"), "checks",
                        "--", "-DPNP_CHECKS", "-DPNP_JITTER"], cwd=ROOT, check=True,
                       timeout=1800)
    ref = _run(tmp_path / "ref.npz")
    for i in range(2):
        got = _run(tmp_path / f"chk{i}.npz", VARIANT)
        assert set(got) == set(ref)
        for k in ref:
            assert np.array_equal(got[k], ref[k], equal_nan=True), (i, k)
