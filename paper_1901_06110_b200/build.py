"""Build the native library in-tree: paper_1901_06110_b200/libpnpb200.so.

Plain nvcc (no torch extension machinery): the library exposes a C ABI
(include/pnp_b200.h) with no torch types, and is loaded with ctypes.
Compiled for sm_100a only, with -lineinfo so ncu's source page maps to code.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libpnpb200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "pnp_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def build(force: bool = False, verbose: bool = False, extra=()) -> Path:
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    build_dir = PKG / "build"
    build_dir.mkdir(exist_ok=True)
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-I", str(ROOT / "include"), "--expt-relaxed-constexpr",
                     "-Xptxas", "-v" if verbose else "-O3"] + list(extra)

    def one(src: Path):
        obj = build_dir / (src.stem + ".o")
        if src.suffix == ".cpp":  # host-only code (runtime dispatch to AVX2 inside)
            cmd = [os.environ.get("CXX", "g++"), "-c", str(src), "-o", str(obj), "-O3", "-g",
                   "-std=c++17", "-fPIC", "-pthread", "-I", str(ROOT / "include")]
        else:
            cmd = [nvcc(), "-c", str(src), "-o", str(obj)] + common
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, r

    objs = []
    with ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 4))) as ex:
        for src, obj, r in ex.map(one, sources()):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src.name}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", "-o", str(tmp)] + objs + ARCH + ["-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
