"""Recipe: install the UNMODIFIED reference into oracle/_ref — TEST/BENCH INFRASTRUCTURE ONLY.

The reference (``pnprestore`` 0.1.0, /root/reference/pkg) is pure Python +
numpy, so "building" it is a plain offline pip install of its own source
tree (no network, no dependency resolution: numpy is already in the image):

    python -m pip install --no-index --no-deps --no-build-isolation \
        --target oracle/_ref /root/reference/pkg

``oracle/_ref/`` is git-ignored (not product source, never committed) but
travels to the GPU box with the gpurun snapshot, where ``bench.py --impl
reference`` and the ``cpu_baseline`` leg import it to time the reference's
own code path (oracle/refcpu.py).  Nothing in the product package imports it.
``__graft_entry__.build()`` runs this when /root/reference is present.
"""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg")
TARGET = HERE / "_ref"


def built() -> bool:
    return (TARGET / "pnprestore" / "denoise.py").exists()


def build(force: bool = False) -> Path | None:
    if built() and not force:
        return TARGET
    if not (REF_SRC / "pyproject.toml").exists():
        return None  # GPU box: the prebuilt copy travels with the snapshot
    cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-deps",
           "--no-build-isolation", "--upgrade", "--target", str(TARGET), str(REF_SRC)]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd="/tmp")
    if r.returncode != 0:
        sys.stderr.write(r.stdout[-2000:] + r.stderr[-2000:])
        raise RuntimeError("pip install of the reference into oracle/_ref failed")
    return TARGET


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
