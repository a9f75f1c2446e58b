"""approxrv-b200: B200-native hot path of approxrv (arXiv 2012.09715).

Approximate Gaussian / non-central chi-squared random variables from cheap
piecewise inverse-CDF tables, fused with PCG32 generation, and the nested
multilevel Monte Carlo path kernels that consume them -- hand-written sm_100a
CUDA behind the C ABI in include/approxrv_b200.h, with the reference's
Python API (approxrv) mirrored on top.
"""

__version__ = "0.1.0"

from . import _native  # noqa: F401  (loads libarv_b200.so; fails loudly)
from ._backend import backend_name, get_kernels
from .errors import (
    ApproxRvError, BadMagicError, ChecksumError, ConfigError, DeviceError, DomainError,
    NumericalError, TableIOError, TruncatedFileError, VersionError,
)
from .mlmc import (
    Allocation, CirParams, GbmParams, LevelSpec, LevelStats, PathBatch, difference, estimate_level,
    estimate_level_suite, estimate_level_suites, level_stream, optimal_allocation, optimal_allocation_nested, simulate,
    simulate_cir_coupled, simulate_gbm_coupled, speedup_report, telescoped_mean,
)
from .sampler import (
    CoupledGaussianBatch, GaussianSamplePair, Pcg32Stream, PhiloxStream, UniformStream, dyadic_index,
    eval_constant, eval_dyadic, eval_ncchi2, eval_subdyadic, evaluate, gaussian_exact_batch, gaussian_inv_cdf,
    sample_coupled, shard_range,
)
from .tables import ConstantTable, DyadicPolyTable, NcChi2Table, SubDyadicTable, load_table, shipped_names
from .tableio import export_table, import_table

__all__ = [
    "ApproxRvError", "BadMagicError", "ChecksumError", "ConfigError", "DeviceError", "DomainError",
    "NumericalError", "TableIOError", "TruncatedFileError", "VersionError",
    "Allocation", "CirParams", "GbmParams", "LevelSpec", "LevelStats", "PathBatch", "difference",
    "estimate_level", "estimate_level_suite", "estimate_level_suites", "level_stream", "optimal_allocation", "optimal_allocation_nested",
    "simulate", "simulate_cir_coupled", "simulate_gbm_coupled", "speedup_report", "telescoped_mean",
    "CoupledGaussianBatch", "GaussianSamplePair", "Pcg32Stream", "PhiloxStream", "UniformStream", "dyadic_index",
    "eval_constant", "eval_dyadic", "eval_ncchi2", "eval_subdyadic", "evaluate", "gaussian_exact_batch",
    "gaussian_inv_cdf", "sample_coupled", "shard_range",
    "ConstantTable", "DyadicPolyTable", "NcChi2Table", "SubDyadicTable", "load_table", "shipped_names",
    "export_table", "import_table",
    "backend_name", "get_kernels",
]
