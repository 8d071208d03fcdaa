"""Build libpnpb200.so from another git revision (or with extra nvcc flags)
into build/var_<name>/ for A/B kernel timing (development aid).

usage: build_variant.py <name> [git-rev] [-- extra nvcc flags...]
then:  PNP_B200_LIB=build/var_<name>/libpnpb200.so python scripts/...
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
argv = sys.argv[1:]
extra = []
if "--" in argv:
    i = argv.index("--")
    argv, extra = argv[:i], argv[i + 1:]
name = argv[0]
rev = argv[1] if len(argv) > 1 else None
out = ROOT / "build" / f"var_{name}"
src = out / "src"
src.mkdir(parents=True, exist_ok=True)
if rev:
    for sub in ("paper_1901_06110_b200/csrc", "include"):
        tar = subprocess.run(["git", "-C", str(ROOT), "archive", rev, sub], check=True,
                             capture_output=True).stdout
        subprocess.run(["tar", "-x", "-C", str(src)], input=tar, check=True)
    csrc, inc = src / "paper_1901_06110_b200/csrc", src / "include"
else:
    csrc, inc = ROOT / "paper_1901_06110_b200/csrc", ROOT / "include"
arch = ["-gencode", "arch=compute_100a,code=sm_100a"]
flags = arch + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(inc),
                "--expt-relaxed-constexpr"] + extra
objs = []
procs = []
for cu in sorted(csrc.glob("*.cu")):
    obj = out / (cu.stem + ".o")
    objs.append(str(obj))
    procs.append(subprocess.Popen(["nvcc", "-c", str(cu), "-o", str(obj)] + flags))
for cpp in sorted(csrc.glob("*.cpp")):  # host-only sources (as in build.py)
    obj = out / (cpp.stem + ".o")
    objs.append(str(obj))
    procs.append(subprocess.Popen(["g++", "-c", str(cpp), "-o", str(obj), "-O3", "-g",
                                   "-std=c++17", "-fPIC", "-pthread", "-I", str(inc)]))
if any(p.wait() for p in procs):
    sys.exit("compile failed")
subprocess.run(["nvcc", "-shared", "-o", str(out / "libpnpb200.so")] + objs + arch +
               ["-cudart", "static"], check=True)
print(out / "libpnpb200.so")
