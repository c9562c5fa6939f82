"""B200-native SkyCell skyline path (arXiv 2107.09993).

The product is ``lib/libskycell_gpu.so`` (sm_100a kernels behind the C ABI in
``include/skycell_gpu.h``); this package is its Python mirror of the reference
API.  See DESIGN.md.
"""
from .skycell import (  # noqa: F401
    ConfigError, CudaError, Dataset, Engine, InputError, IoError, LayerCounts, Mode, MultiEngine, MultiLayerGrid,
    SkycellError, SkylineResult, StageTimes, UnsupportedError, UsageError, bin_header, compute_skyline, default_rho, engine,
    load_library, quadrant_skyline, validate,
)

__all__ = [
    "ConfigError", "CudaError", "Dataset", "Engine", "InputError", "IoError", "LayerCounts", "Mode",
    "MultiEngine", "MultiLayerGrid", "SkycellError", "SkylineResult", "StageTimes", "UnsupportedError", "UsageError", "bin_header", "compute_skyline",
    "default_rho", "engine", "load_library", "quadrant_skyline", "validate",
]
