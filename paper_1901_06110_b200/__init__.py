"""B200-native DSG-NLM / linearized plug-and-play ADMM (arXiv 1901.06110 hot path).

Drop-in for the reference package ``pnprestore`` on its hot path: the same
public names, backed by hand-written sm_100a CUDA kernels in
``libpnpb200.so`` (C ABI: include/pnp_b200.h) through ctypes.  Loading the
package loads the native library; there is no CPU fallback.
"""

from . import _lib  # noqa: F401  (loads libpnpb200.so, fails loudly if missing)
from .denoise import (  # noqa: F401
    DENSE_WEIGHTS_MAX_PIXELS,
    FrozenGuide,
    build_dense_weights,
    PatchParams,
    dsg_nlm_denoise,
    freeze_guide,
    hat_weight,
    nlm_denoise,
    nlm_kernel,
    patch_distance_map,
)
from .forward import (  # noqa: F401
    QIS_FLOOR,
    QisCounts,
    QisModel,
    SuperResOp,
    gaussian_kernel,
    power_iteration_lipschitz,
    qis_data_term,
    qis_gradient,
    qis_initial_estimate,
    qis_simulate,
    sr_adjoint,
    sr_apply,
    sr_data_term,
    sr_gradient,
    sr_simulate,
)
from .imageio import (  # noqa: F401
    ImageFormatError,
    MalformedHeaderError,
    TruncatedPayloadError,
    UnsupportedFormatError,
    read_image,
    write_image,
)
from .image import (  # noqa: F401
    NON_NEGATIVE,
    UNCONSTRAINED,
    UNIT_BOX,
    Box,
    NonNegative,
    Unconstrained,
    box_sum,
    integral_image,
    pad_symmetric,
    project,
    psnr,
    validate_image,
)
from .solver import (  # noqa: F401
    CgBreakdownError,
    CgResult,
    DivergenceError,
    IterationRecord,
    Problem,
    SolverConfig,
    default_qis_alpha,
    default_sr_alpha,
    device_callable,
    linearized_pnp_admm,
    make_qis_problem,
    make_sr_problem,
    residuals,
    cg_solve,
    standard_pnp_admm_cg,
    write_log_csv,
)
from .stream import DenoiseStream, denoise_host_sequence  # noqa: F401
from .synth import SplitMix64  # noqa: F401


__version__ = "0.1.0"
