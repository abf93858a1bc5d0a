"""B200-native per-pixel whitening pipeline (arXiv 1408.3526).

A drop-in for the reference ``clutterwhiten`` hot path: the public names a
caller of ``Pipeline.process_frame`` needs, with the same signatures and
errors (/root/reference/pkg/src/clutterwhiten/__init__.py:11-95).  The
frame path runs as one fused sm_100a kernel per frame behind the C ABI in
include/cw_b200.h; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .params import (
    FilterParams,
    ParamError,
    default_params,
    load_params,
    save_params,
    validate,
)
from .parallel import ExecStrategy
from .design import (
    FilterBank,
    FreqKernel,
    SampleKernel,
    build_bank,
    dirichlet,
    kernel_to_freq,
    retained_bin_indices,
    sample_kernel,
)
from .flow import VelocityField, pick_gains
from .pipeline import Pipeline, WhitenedOutput, apply_pef, valid_bounds, valid_mask

__all__ = [
    "__version__",
    "FilterParams",
    "ParamError",
    "default_params",
    "load_params",
    "save_params",
    "validate",
    "ExecStrategy",
    "FilterBank",
    "FreqKernel",
    "SampleKernel",
    "build_bank",
    "dirichlet",
    "kernel_to_freq",
    "retained_bin_indices",
    "sample_kernel",
    "VelocityField",
    "pick_gains",
    "Pipeline",
    "WhitenedOutput",
    "apply_pef",
    "valid_bounds",
    "valid_mask",
]
