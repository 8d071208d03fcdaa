"""B200-native DSG-NLM / linearized plug-and-play ADMM (arXiv 1901.06110 hot path).

Drop-in for the reference package ``pnprestore`` on its hot path: the same
public names, backed by hand-written sm_100a CUDA kernels in
``libpnpb200.so`` (C ABI: include/pnp_b200.h) through ctypes.  Loading the
package loads the native library; there is no CPU fallback.
"""

from . import _lib  # noqa: F401  (loads libpnpb200.so, fails loudly if missing)
from .denoise import (  # noqa: F401
    FrozenGuide,
    PatchParams,
    dsg_nlm_denoise,
    freeze_guide,
    hat_weight,
    nlm_denoise,
)
from .synth import SplitMix64  # noqa: F401

__version__ = "0.1.0"
