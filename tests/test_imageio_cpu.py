"""PGM / PFM I/O (reference image.py:169-280) against files and reads produced
by the reference itself (tests/golden/io/, io.npz from make_golden.py)."""

from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

IO = GOLDEN / "io"


@pytest.fixture(scope="module")
def io():
    from paper_1901_06110_b200 import imageio
    return imageio


def test_reads_match_reference(io):
    g = load_golden("io.npz")
    names = sorted(p.name for p in IO.iterdir())
    assert names
    for name in names:
        if "read_" + name in g:
            got = io.read_image(IO / name)
            assert got.dtype == np.float64
            assert np.array_equal(got, g["read_" + name]), name
        else:
            want = str(g["error_" + name])
            with pytest.raises(io.ImageFormatError) as ei:
                io.read_image(IO / name)
            assert type(ei.value).__name__ == want, name


def test_writes_are_byte_identical(io, tmp_path):
    img = load_golden("io.npz")["written_image"]
    io.write_image(img, tmp_path / "a.pgm", "pgm8")
    io.write_image(img, tmp_path / "a.pfm", "pfm")
    assert (tmp_path / "a.pgm").read_bytes() == (IO / "w8.pgm").read_bytes()
    assert (tmp_path / "a.pfm").read_bytes() == (IO / "wf.pfm").read_bytes()
    with pytest.raises(ValueError):
        io.write_image(img, tmp_path / "a.x", "png")
    with pytest.raises(ValueError):
        io.write_image(np.full((2, 2), np.nan), tmp_path / "b.pgm")


def test_roundtrip(io, tmp_path):
    rng = np.random.default_rng(1)
    img = rng.random((5, 9))
    io.write_image(img, tmp_path / "r.pfm", "pfm")
    assert np.array_equal(io.read_image(tmp_path / "r.pfm"), img.astype(np.float32))
    io.write_image(img, tmp_path / "r.pgm", "pgm8")
    assert np.abs(io.read_image(tmp_path / "r.pgm") - img).max() <= 0.5 / 255 + 1e-12
