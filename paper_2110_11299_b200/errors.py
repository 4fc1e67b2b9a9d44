"""Exception types mirroring P/include/dsattn/errors.hpp:9-31, plus the two
B200-side codes (CUDA failure, unsupported configuration).  dsa_status codes
from include/dsa_b200.h map onto these one to one."""


class DsaError(RuntimeError):
    code = -1


class ShapeError(DsaError, ValueError):
    code = 1


class ParamError(DsaError, ValueError):
    code = 2


class ConfigError(DsaError):
    code = 3


class CudaError(DsaError):
    code = 4


class IoError(DsaError):
    code = 5


class UnsupportedError(DsaError):
    code = 6


BY_CODE = {c.code: c for c in (ShapeError, ParamError, ConfigError, CudaError, IoError,
                               UnsupportedError)}
