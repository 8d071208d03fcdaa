"""CPU-side checks of the native boundary: the C-ABI library loads and exports
every symbol include/pnp_b200.h declares (no compute without a GPU)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "pnp_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|const char\*)\s+(pnp_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_1901_06110_b200 import _lib

    syms = header_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.pnp_version() == 1


def test_error_path_without_gpu_or_bad_args():
    from paper_1901_06110_b200 import _lib

    with pytest.raises(ValueError):
        _lib.call("pnp_dsg_denoise", ctypes.c_void_p(), None, None, None, 1, 8, 8, 2, 3,
                  None, 0.2, None, None)
    assert "null" in _lib.lib.pnp_last_error().decode()


def test_qis_simulate_host_matches_reference_golden(golden_forward):
    """Host-native Knuth sampler is bit-exact with the reference (forward.py:263-298)."""
    from paper_1901_06110_b200 import _lib

    f = golden_forward
    x = f["qis_truth"]
    stop = np.ascontiguousarray(np.exp(-16.0 * np.clip(x, 0.0, 1.0) / 16).ravel())
    ones = np.zeros(x.size)
    _lib.call("pnp_qis_simulate_host", stop.ctypes.data_as(ctypes.c_void_p), x.size, 16,
              2, ones.ctypes.data_as(ctypes.c_void_p))
    assert np.array_equal(ones.reshape(x.shape), f["qis_ones"])


def test_patch_params_validation():
    from paper_1901_06110_b200 import PatchParams

    with pytest.raises(ValueError):
        PatchParams(4, 2, 0.1)
    with pytest.raises(ValueError):
        PatchParams(3, 0, 0.1)
    with pytest.raises(ValueError):
        PatchParams(3, 2, 0.0)
    with pytest.raises(ValueError):
        PatchParams(3, 2, 0.1, patch_sigma=0.0)
    assert PatchParams(7, 10, 0.1).pad_margin == 13
    p = PatchParams(5, 5, 0.2, 1.5)
    assert abs(p.taps().sum() - 1) < 1e-15


def test_synth_splitmix_matches_reference(golden_forward):
    from paper_1901_06110_b200.synth import SplitMix64

    f = golden_forward
    r = SplitMix64(1234567)
    assert [r.next_uint64() for _ in range(4)] == [int(v) for v in f["splitmix_u64"]]
    assert np.array_equal(SplitMix64(99).uniforms(1001), f["splitmix_uniforms"])
    assert np.array_equal(SplitMix64(5).normals(999), f["splitmix_normals"])


def test_sweep_path_routing():
    """pnp_dsg_geometry (host logic, no GPU): box taps run the P-templated
    kernel up to P = 9 and the running-sum general kernel from P = 11 (the
    reference's Table-1 range, P = 11..29, in one kernel whose cost is flat in
    P); Gaussian taps the P-templated kernel up to P = 15, R <= 32; the
    full-window variant once the half-window far plane exceeds shared memory."""
    from paper_1901_06110_b200 import _lib as L
    for P, box, R, want in [(1, True, 3, 0), (7, True, 10, 0), (9, True, 10, 0),
                            (11, True, 10, 1), (29, True, 21, 1), (63, True, 5, 1),
                            (7, False, 10, 0), (15, False, 10, 0), (17, False, 10, 1),
                            (7, False, 40, 1), (1, True, 100, 2)]:
        g = L.dsg_geometry(256, 256, R, P, box)
        assert g[3] == want, (P, box, R, g)
        assert g[0] in (8, 16, 32) or g[3] == 0
    import pytest
    with pytest.raises(ValueError):
        L.dsg_geometry(256, 256, 5, 65, True)


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 31, 1000, (1 << 20) + 5])
def test_host_casts_are_c_casts(n):
    """The numpy path's streaming host casts (pnp_host_cast_*) give numpy's
    astype bits: misaligned ends, overflow to inf, nan, denormals."""
    import torch

    from paper_1901_06110_b200 import _arrays as A

    rng = np.random.default_rng(n)
    s64 = rng.standard_normal(n) * 10.0 ** rng.integers(-45, 45, n)
    if n > 4:
        s64[:4] = [np.inf, -np.nan, 1e300, -1e-320]
    buf32 = np.full(n + 3, -7.0, dtype=np.float32)
    o32 = buf32[3:]                     # 12-byte offset: scalar head + vector body
    A.cast_into(torch.from_numpy(o32), torch.from_numpy(s64))
    with np.errstate(over="ignore"):
        want = s64.astype(np.float32)
    assert np.array_equal(o32.view(np.uint32), want.view(np.uint32))
    assert np.all(buf32[:3] == -7.0)
    buf64 = np.full(n + 1, -7.0)
    o64 = buf64[1:]
    A.cast_into(torch.from_numpy(o64), torch.from_numpy(want))
    assert np.array_equal(o64.view(np.uint64), want.astype(np.float64).view(np.uint64))
    assert buf64[0] == -7.0


@pytest.mark.filterwarnings("ignore::DeprecationWarning")
def test_host_casts_in_a_forked_child():
    """The cast pool's workers do not survive fork(): a child process runs
    the casts inline instead of waiting for them."""
    import os

    import torch

    from paper_1901_06110_b200 import _arrays as A

    s = np.arange(1 << 20, dtype=np.float32)
    d = np.empty(1 << 20)
    A.cast_into(torch.from_numpy(d), torch.from_numpy(s))   # pool started in the parent
    pid = os.fork()
    if pid == 0:
        try:
            d2 = np.empty(1 << 20)
            A.cast_into(torch.from_numpy(d2), torch.from_numpy(s))
            os._exit(0 if np.array_equal(d2, s) else 1)
        except BaseException:
            os._exit(2)
    _, status = os.waitpid(pid, 0)
    assert os.WIFEXITED(status) and os.WEXITSTATUS(status) == 0
