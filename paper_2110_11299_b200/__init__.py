"""B200-native Dynamic Sparse Attention hot path (arXiv 2110.11299).

predict (projection + quantisation) -> select (exact-integer approximate
scores -> row / vector / block / threshold masks) -> sparse attention
(SDDMM -> online softmax -> SpMM), as hand-written sm_100a kernels behind the
C-ABI in include/dsa_b200.h.  This package is the Python host mirror used by
the tests and bench.py; the C++ host mirror of the reference API is
include/dsattn_gpu.hpp.
"""
from .errors import (ConfigError, CudaError, DsaError, IoError, ParamError, ShapeError,
                     UnsupportedError)
from .presets import Preset, baseline_configs, load_preset, parse_preset, CONFIG_NAMES

__all__ = ["ConfigError", "CudaError", "DsaError", "IoError", "ParamError", "ShapeError",
           "UnsupportedError", "Preset", "baseline_configs", "load_preset", "parse_preset",
           "CONFIG_NAMES", "ops"]


def __getattr__(name):
    if name == "ops":
        import importlib
        return importlib.import_module(".ops", __name__)
    raise AttributeError(name)
