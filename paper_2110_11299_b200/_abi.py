"""ctypes binding of include/dsa_b200.h (the C-ABI).  Loads the in-tree
libdsa_b200.so; there is no fallback: a missing library raises immediately."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

from . import errors

PKG = Path(__file__).resolve().parent
import os

# DSA_LIB: an alternative build of the same library (tools/ablate.py variants)
LIB_PATH = Path(os.environ["DSA_LIB"]) if os.environ.get("DSA_LIB") else PKG / "libdsa_b200.so"
HEADER = PKG.parent / "include" / "dsa_b200.h"


class DsaConfig(C.Structure):
    _fields_ = [("batch", C.c_int64), ("heads", C.c_int64), ("L", C.c_int64), ("d", C.c_int64),
                ("k", C.c_int64), ("dtype", C.c_int32), ("bits", C.c_int32),
                ("quant_scope", C.c_int32), ("round_proj_f32", C.c_int32),
                ("mask_mode", C.c_int32), ("scale", C.c_int32), ("keep", C.c_int64),
                ("vec_v", C.c_int32), ("block", C.c_int32), ("force_diag", C.c_int32),
                ("causal", C.c_int32), ("frac_num", C.c_int64), ("frac_den", C.c_int64),
                ("cap", C.c_int64)]


class DsaMask(C.Structure):
    _fields_ = [("cols", C.c_void_p), ("rowptr", C.c_void_p), ("capacity", C.c_int64),
                ("empty_rows", C.c_void_p)]


class DsaCounts(C.Structure):
    _fields_ = [("nnz", C.c_uint64), ("sddmm_mults", C.c_uint64), ("spmm_mults", C.c_uint64),
                ("softmax_exps", C.c_uint64), ("empty_rows", C.c_uint64),
                ("flops_predict", C.c_double), ("flops_score", C.c_double),
                ("flops_attention", C.c_double), ("bytes_predict", C.c_double),
                ("bytes_attention", C.c_double)]


_P = C.c_void_p
_SIGS = {
    "dsa_abi_version": (C.c_int, []),
    "dsa_last_error": (C.c_char_p, []),
    "dsa_build_info": (C.c_char_p, []),
    "dsa_config_validate": (C.c_int, [C.POINTER(DsaConfig)]),
    "dsa_workspace_bytes": (C.c_size_t, [C.POINTER(DsaConfig)]),
    "dsa_mask_capacity": (C.c_int64, [C.POINTER(DsaConfig)]),
    "dsa_predict": (C.c_int, [C.POINTER(DsaConfig), _P, _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "dsa_select": (C.c_int, [C.POINTER(DsaConfig), _P, _P, _P, _P, C.POINTER(DsaMask), _P,
                             C.c_size_t, _P]),
    "dsa_sparse_attention": (C.c_int, [C.POINTER(DsaConfig), _P, _P, _P, C.POINTER(DsaMask), _P, _P]),
    "dsa_pipeline": (C.c_int, [C.POINTER(DsaConfig), _P, _P, _P, _P, _P, C.POINTER(DsaMask), _P,
                               C.c_size_t, _P]),
    "dsa_launch_counter": (C.c_uint64, []),
    "dsa_predict_wtilde_workspace_bytes": (C.c_size_t, [C.POINTER(DsaConfig)]),
    "dsa_predict_wtilde": (C.c_int, [C.POINTER(DsaConfig), C.c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                     C.c_size_t, _P]),
    "dsa_pipeline_fused": (C.c_int, [C.POINTER(DsaConfig)]),
    "dsa_prediction_accuracy": (C.c_int, [C.POINTER(DsaConfig), C.POINTER(DsaMask), C.POINTER(DsaMask),
                                          C.POINTER(C.c_double), _P]),
    "dsa_project_qkv": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                  C.c_int64, _P, _P, _P, _P, _P, _P, _P]),
    "dsa_counters": (C.c_int, [C.POINTER(DsaConfig), C.POINTER(DsaMask), C.POINTER(DsaCounts), _P]),
    "dsa_dataflow_trace": (C.c_int, [C.POINTER(DsaConfig), C.POINTER(DsaMask), C.c_int32, C.c_int64, _P, _P, _P]),
    "dsa_row_topk_f64": (C.c_int, [C.c_int64, C.c_int64, _P, C.c_int64, _P, _P]),
    "dsa_colvec_mask_f64": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, _P, _P, _P]),
    "dsa_threshold_mask_f64": (C.c_int, [C.c_int64, C.c_int64, _P, C.c_double, C.c_int32, C.c_int32, _P, _P]),
    "dsa_sddmm_f64": (C.c_int, [C.c_int64, C.c_int64, _P, _P, _P, _P, C.c_int32, _P, _P]),
    "dsa_sparse_softmax_f64": (C.c_int, [C.c_int64, _P, _P, _P, _P, _P]),
    "dsa_spmm_f64": (C.c_int, [C.c_int64, C.c_int64, _P, _P, _P, _P, _P, _P]),
    "dsa_generate": (C.c_int, [C.POINTER(DsaConfig), C.c_uint64, C.c_int32, C.c_int32, C.c_int64,
                               C.c_int64, _P, _P, _P, _P, C.c_int32]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise errors.CudaError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().dsa_last_error().decode()
        raise errors.BY_CODE.get(status, errors.DsaError)(msg)


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(dsa_[a-z0-9_]+)\s*\(", text)) - {"dsa_status"})
