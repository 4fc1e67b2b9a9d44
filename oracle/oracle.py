"""ctypes front-end of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module -- as the checker, never as the product.

* ``Oracle``: our C restatement (oracle/dsa_oracle.c -> build/libdsa_oracle.so)
* ``Reference``: the unmodified reference sources compiled by oracle/Makefile
  into _ref/libdsattn_ref.so with our extern "C" shim (ref_shim.cpp).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "build" / "libdsa_oracle.so"
REF_SO = HERE / "_ref" / "libdsattn_ref.so"
REF_SRC = Path("/root/reference/proj")

_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
I64, I32, D = C.c_int64, C.c_int, C.c_double


def build(ref: bool = True) -> None:
    targets = ["oracle"] + (["ref", "shim_test", "eval_test"] if ref and REF_SRC.exists() else [])
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    def __init__(self):
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        sig = {
            "dsa_oracle_project": (None, [_d, _d, I64, I64, I64, I32, _d]),
            "dsa_oracle_round_half_away": (D, [D]),
            "dsa_oracle_quantize_levels": (D, [_d, I64, I32, _i32]),
            "dsa_oracle_quantize_levels_rows": (None, [_d, I64, I64, I32, _i32, _d]),
            "dsa_oracle_dequantize": (None, [_i32, I64, D, I32, _d]),
            "dsa_oracle_scores_int": (None, [_i32, _i32, I64, I64, _i32]),
            "dsa_oracle_row_topk": (I32, [_d, I64, I64, _u32]),
            "dsa_oracle_mask_topk": (I32, [_i32, _i32, I64, I64, I64, _u32]),
            "dsa_oracle_mask_topk_rowscaled": (I32, [_i32, _i32, _d, I64, I64, I64, _u32]),
            "dsa_oracle_mask_colvec": (I32, [_i32, _i32, I64, I64, I64, I64, _u32]),
            "dsa_oracle_mask_block": (I32, [_i32, _i32, I64, I64, I64, I64, I32, _u32]),
            "dsa_oracle_exp": (D, [D]),
            "dsa_oracle_exp_table": (None, [D, I64, _i64]),
            "dsa_oracle_mask_threshold": (I64, [_i32, _i32, I64, I64, D, I64, I64, I64, I32, _u64, C.c_void_p]),
            "dsa_oracle_sparse_attention": (None, [_d, _d, _d, I64, I64, I64, _u64, _u32, I32, I32, _d, _u8]),
            "dsa_oracle_masked_dense_attention": (None, [_d, _d, _d, I64, I64, I64, _u64, _u32, I32, _d]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        self.L = L

    # -- predictor
    def project(self, x, p, round_f32=False) -> np.ndarray:
        x, p = _f64(x), _f64(p)
        out = np.empty((x.shape[0], p.shape[1]))
        self.L.dsa_oracle_project(x, p, x.shape[0], x.shape[1], p.shape[1], int(round_f32), out)
        return out

    def quantize_levels(self, x, bits) -> tuple[np.ndarray, float]:
        x = _f64(x)
        lv = np.empty(x.shape, np.int32)
        s = self.L.dsa_oracle_quantize_levels(x, x.size, bits, lv)
        return lv, s

    def quantize_levels_rows(self, x, bits) -> tuple[np.ndarray, np.ndarray]:
        x = _f64(x)
        lv = np.empty(x.shape, np.int32)
        s = np.empty(x.shape[0])
        self.L.dsa_oracle_quantize_levels_rows(x, x.shape[0], x.shape[1], bits, lv, s)
        return lv, s

    def round_half_away(self, v: float) -> float:
        return self.L.dsa_oracle_round_half_away(v)

    def levels(self, x, p, bits, per_row=False, round_f32=False):
        xp = self.project(x, p, round_f32)
        return self.quantize_levels_rows(xp, bits) if per_row else self.quantize_levels(xp, bits)

    # -- scores / masks
    def scores_int(self, lq, lk) -> np.ndarray:
        lq, lk = np.ascontiguousarray(lq, np.int32), np.ascontiguousarray(lk, np.int32)
        out = np.empty((lq.shape[0], lk.shape[0]), np.int32)
        self.L.dsa_oracle_scores_int(lq, lk, lq.shape[0], lq.shape[1], out)
        return out

    def row_topk(self, row, keep) -> np.ndarray:
        row = _f64(row)
        out = np.empty(keep, np.uint32)
        if self.L.dsa_oracle_row_topk(row, row.size, keep, out) != 0:
            raise ValueError("row_topk_indices: k_keep out of range")
        return out

    def mask_topk(self, lq, lk, keep, sk=None) -> np.ndarray:
        lq, lk = np.ascontiguousarray(lq, np.int32), np.ascontiguousarray(lk, np.int32)
        L = lq.shape[0]
        out = np.empty((L, keep), np.uint32)
        if sk is None:
            r = self.L.dsa_oracle_mask_topk(lq, lk, L, lq.shape[1], keep, out)
        else:
            r = self.L.dsa_oracle_mask_topk_rowscaled(lq, lk, _f64(sk), L, lq.shape[1], keep, out)
        if r != 0:
            raise ValueError("row_topk_indices: k_keep out of range")
        return out

    def mask_colvec(self, lq, lk, v, keep) -> np.ndarray:
        lq, lk = np.ascontiguousarray(lq, np.int32), np.ascontiguousarray(lk, np.int32)
        L = lq.shape[0]
        out = np.empty((-(-L // v), keep), np.uint32)
        if self.L.dsa_oracle_mask_colvec(lq, lk, L, lq.shape[1], v, keep, out) != 0:
            raise ValueError("colvec_mask: bad parameters")
        return out

    def mask_block(self, lq, lk, bs, keep, force_diag) -> np.ndarray:
        lq, lk = np.ascontiguousarray(lq, np.int32), np.ascontiguousarray(lk, np.int32)
        L = lq.shape[0]
        out = np.empty((-(-L // bs), keep), np.uint32)
        if self.L.dsa_oracle_mask_block(lq, lk, L, lq.shape[1], bs, keep, int(force_diag), out) != 0:
            raise ValueError("block mask: bad parameters")
        return out

    def exp(self, x: float) -> float:
        return self.L.dsa_oracle_exp(x)

    def exp_table(self, c: float, n: int) -> np.ndarray:
        out = np.empty(n, np.int64)
        self.L.dsa_oracle_exp_table(c, n, out)
        return out

    def mask_threshold(self, lq, lk, c, frac_num, frac_den, cap, causal):
        lq, lk = np.ascontiguousarray(lq, np.int32), np.ascontiguousarray(lk, np.int32)
        L = lq.shape[0]
        rp = np.zeros(L + 1, np.uint64)
        self.L.dsa_oracle_mask_threshold(lq, lk, L, lq.shape[1], c, frac_num, frac_den, cap,
                                         int(causal), rp, None)
        cols = np.empty(max(int(rp[-1]), 1), np.uint32)
        empty = self.L.dsa_oracle_mask_threshold(lq, lk, L, lq.shape[1], c, frac_num, frac_den,
                                                 cap, int(causal), rp,
                                                 cols.ctypes.data_as(C.c_void_p))
        return rp, cols[: int(rp[-1])], int(empty)

    # -- attention
    def sparse_attention(self, q, k, v, rowptr, cols, scale=True, round_f32=False):
        q, k, v = _f64(q), _f64(k), _f64(v)
        L, d = q.shape
        z = np.empty((L, v.shape[1]))
        er = np.empty(L, np.uint8)
        cols = np.ascontiguousarray(cols, np.uint32)
        if cols.size == 0:
            cols = np.zeros(1, np.uint32)
        self.L.dsa_oracle_sparse_attention(q, k, v, L, d, v.shape[1],
                                           np.ascontiguousarray(rowptr, np.uint64), cols,
                                           int(scale), int(round_f32), z, er)
        return z, er

    def masked_dense_attention(self, q, k, v, rowptr, cols, scale=True):
        q, k, v = _f64(q), _f64(k), _f64(v)
        L, d = q.shape
        z = np.empty((L, v.shape[1]))
        self.L.dsa_oracle_masked_dense_attention(q, k, v, L, d, v.shape[1],
                                                 np.ascontiguousarray(rowptr, np.uint64),
                                                 np.ascontiguousarray(cols, np.uint32),
                                                 int(scale), z)
        return z


class Reference:
    """The reference implementation itself (oracle/_ref/libdsattn_ref.so)."""

    def __init__(self):
        if not REF_SO.exists():
            if REF_SRC.exists():
                build(ref=True)
            else:
                raise FileNotFoundError(f"{REF_SO} not built and {REF_SRC} absent")
        L = C.CDLL(str(REF_SO))
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_isa_name": (C.c_char_p, []),
            "ref_project": (I32, [_d, _d, I64, I64, I64, I32, _d]),
            "ref_quantize": (I32, [_d, I64, I64, I32, I32, _d]),
            "ref_quantize_levels": (I32, [_d, I64, I64, I32, I32, _i32, C.POINTER(C.c_double)]),
            "ref_row_topk": (I32, [_d, I64, I64, _u32]),
            "ref_topk_mask": (I32, [_d, I64, I64, _u32]),
            "ref_colvec_mask": (I32, [_d, I64, I64, I32, D, _u64, C.c_void_p]),
            "ref_threshold_mask": (I32, [_d, I64, D, I32, _u64, C.c_void_p]),
            "ref_colvec_maxpool_mask": (I32, [_d, I64, I64, I64, _u32]),
            "ref_sparse_attention": (I32, [_d, _d, _d, I64, I64, I64, I32, _u64, _u32, I32, _d, _u8, _u64]),
            "ref_masked_attention": (I32, [_d, _d, _d, I64, I64, I64, _u64, _u32, I32, _d]),
            "ref_pipeline": (I32, [I64, I32, _d, _d, _d, _d, I64, I64, I64, I32, I32, I32, I32, I64, I64,
                                   I64, I32, I64, I64, I64, I32, _d]),
            "ref_levels_wtilde": (I32, [C.c_void_p, C.c_void_p, C.c_void_p, _d, I64, I64, I64, I32, I32,
                                        C.c_void_p, _i32, C.POINTER(C.c_double)]),
            "ref_init_projection": (I32, [I64, I64, C.c_uint64, _d]),
            "ref_prediction_accuracy": (I32, [I64, _u64, _u32, _u64, _u32, C.POINTER(C.c_double)]),
            "ref_dataflow_simulate": (I32, [I64, _u64, _u32, I32, I64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
            "ref_block_mask": (I32, [_i32, _i32, I64, I64, I64, I64, I32, _u32]),
            "ref_causal_threshold_mask": (I32, [_i32, _i32, I64, I64, D, D, I64, I32, _u64, C.c_void_p]),
            "ref_threshold_row_probs": (I32, [_i32, _i32, I64, I64, D, I64, I32, _d]),
            "ref_generate": (I32, [I64, I64, I64, I32, C.c_uint64, I32, I32, I64, I64, _d, _d, _d, _d]),
            "ref_write_mask": (I32, [C.c_char_p, I64, _u64, _u32]),
            "ref_read_mask": (I32, [C.c_char_p, C.POINTER(I64), C.POINTER(I64), C.c_void_p, C.c_void_p]),
            "ref_write_sparse_scores": (I32, [C.c_char_p, I64, _u64, _u32, _d]),
            "ref_read_sparse_scores": (I32, [C.c_char_p, C.POINTER(I64), C.POINTER(I64), C.c_void_p,
                                             C.c_void_p, C.c_void_p]),
            "ref_write_container1": (I32, [C.c_char_p, C.c_char_p, I64, I64, I32, _d, C.c_char_p]),
            "ref_read_container1": (I32, [C.c_char_p, C.c_char_p, C.POINTER(I64), C.POINTER(I64),
                                          C.POINTER(I32), C.c_void_p, C.POINTER(I64), C.c_void_p]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        self.L = L

    def _chk(self, r):
        if r != 0:
            msg = self.L.ref_last_error().decode()
            raise {1: ValueError, 2: ValueError, 5: IOError}.get(r, RuntimeError)(f"[ref code {r}] {msg}")

    def isa(self) -> str:
        return self.L.ref_isa_name().decode()

    # ---- the reference's fixture formats (mask.cpp / sparse.cpp / serialize.cpp)
    def write_mask(self, path, rowptr, cols):
        rp = np.ascontiguousarray(rowptr, np.uint64)
        c = np.ascontiguousarray(cols if len(cols) else np.zeros(1), np.uint32)
        self._chk(self.L.ref_write_mask(str(path).encode(), len(rp) - 1, rp, c))

    def read_mask(self, path):
        l, nnz = I64(), I64()
        self._chk(self.L.ref_read_mask(str(path).encode(), C.byref(l), C.byref(nnz), None, None))
        rp = np.zeros(l.value + 1, np.uint64)
        cols = np.zeros(max(nnz.value, 1), np.uint32)
        self._chk(self.L.ref_read_mask(str(path).encode(), C.byref(l), C.byref(nnz),
                                       rp.ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p)))
        return rp, cols[: nnz.value]

    def write_sparse_scores(self, path, rowptr, cols, values):
        rp = np.ascontiguousarray(rowptr, np.uint64)
        c = np.ascontiguousarray(cols if len(cols) else np.zeros(1), np.uint32)
        v = np.ascontiguousarray(values if len(values) else np.zeros(1), np.float64)
        self._chk(self.L.ref_write_sparse_scores(str(path).encode(), len(rp) - 1, rp, c, v))

    def read_sparse_scores(self, path):
        l, nnz = I64(), I64()
        self._chk(self.L.ref_read_sparse_scores(str(path).encode(), C.byref(l), C.byref(nnz), None, None, None))
        rp = np.zeros(l.value + 1, np.uint64)
        cols = np.zeros(max(nnz.value, 1), np.uint32)
        vals = np.zeros(max(nnz.value, 1), np.float64)
        self._chk(self.L.ref_read_sparse_scores(str(path).encode(), C.byref(l), C.byref(nnz),
                                                rp.ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p),
                                                vals.ctypes.data_as(C.c_void_p)))
        return rp, cols[: nnz.value], vals[: nnz.value]

    def write_container1(self, path, name, arr, f32=False, meta=""):
        a = _f64(arr)
        self._chk(self.L.ref_write_container1(str(path).encode(), name.encode(), a.shape[0], a.shape[1],
                                              int(f32), a, meta.encode()))

    def read_container1(self, path, name):
        r, c, m = I64(), I64(), I64()
        f32 = I32()
        self._chk(self.L.ref_read_container1(str(path).encode(), name.encode(), C.byref(r), C.byref(c),
                                             C.byref(f32), None, C.byref(m), None))
        out = np.zeros((r.value, c.value))
        meta = C.create_string_buffer(max(m.value, 1))
        self._chk(self.L.ref_read_container1(str(path).encode(), name.encode(), C.byref(r), C.byref(c),
                                             C.byref(f32), out.ctypes.data_as(C.c_void_p), C.byref(m), meta))
        return out, bool(f32.value), meta.raw[: m.value].decode()

    def project(self, x, p, f32=False):
        x, p = _f64(x), _f64(p)
        out = np.empty((x.shape[0], p.shape[1]))
        self._chk(self.L.ref_project(x, p, x.shape[0], x.shape[1], p.shape[1], int(f32), out))
        return out

    def quantize(self, x, bits, f32=False):
        x = _f64(x)
        out = np.empty(x.shape)
        self._chk(self.L.ref_quantize(x, x.shape[0], x.shape[1], bits, int(f32), out))
        return out

    def quantize_levels(self, x, bits, f32=False):
        x = _f64(x)
        lv = np.empty(x.shape, np.int32)
        s = C.c_double()
        self._chk(self.L.ref_quantize_levels(x, x.shape[0], x.shape[1], bits, int(f32), lv, C.byref(s)))
        return lv, s.value

    def row_topk(self, row, keep):
        row = _f64(row)
        out = np.empty(keep, np.uint32)
        self._chk(self.L.ref_row_topk(row, row.size, keep, out))
        return out

    def topk_mask(self, s, keep):
        s = _f64(s)
        out = np.empty((s.shape[0], keep), np.uint32)
        self._chk(self.L.ref_topk_mask(s, s.shape[0], keep, out))
        return out

    def colvec_mask(self, s, v, sparsity, row_orient=False):
        s = _f64(s)
        L = s.shape[0]
        rp = np.zeros(L + 1, np.uint64)
        self._chk(self.L.ref_colvec_mask(s, L, v, int(row_orient), sparsity, rp, None))
        cols = np.empty(max(int(rp[-1]), 1), np.uint32)
        self._chk(self.L.ref_colvec_mask(s, L, v, int(row_orient), sparsity, rp,
                                         cols.ctypes.data_as(C.c_void_p)))
        return rp, cols[: int(rp[-1])]

    def threshold_mask(self, s, theta, post_softmax):
        s = _f64(s)
        L = s.shape[0]
        rp = np.zeros(L + 1, np.uint64)
        self._chk(self.L.ref_threshold_mask(s, L, theta, int(post_softmax), rp, None))
        cols = np.empty(max(int(rp[-1]), 1), np.uint32)
        self._chk(self.L.ref_threshold_mask(s, L, theta, int(post_softmax), rp,
                                            cols.ctypes.data_as(C.c_void_p)))
        return rp, cols[: int(rp[-1])]

    def colvec_maxpool_mask(self, s_int, v, keep):
        s = _f64(s_int)
        L = s.shape[0]
        out = np.empty((-(-L // v), keep), np.uint32)
        self._chk(self.L.ref_colvec_maxpool_mask(s, L, v, keep, out))
        return out

    def sparse_attention(self, q, k, v, rowptr, cols, scale=True, f32=False):
        q, k, v = _f64(q), _f64(k), _f64(v)
        L, d = q.shape
        z = np.empty((L, v.shape[1]))
        er = np.empty(L, np.uint8)
        cnt = np.zeros(3, np.uint64)
        cols = np.ascontiguousarray(cols, np.uint32)
        if cols.size == 0:
            cols = np.zeros(1, np.uint32)
        self._chk(self.L.ref_sparse_attention(q, k, v, L, d, v.shape[1], int(f32),
                                              np.ascontiguousarray(rowptr, np.uint64), cols,
                                              int(scale), z, er, cnt))
        return z, er, cnt

    def masked_attention(self, q, k, v, rowptr, cols, scale=True):
        q, k, v = _f64(q), _f64(k), _f64(v)
        L, d = q.shape
        z = np.empty((L, v.shape[1]))
        self._chk(self.L.ref_masked_attention(q, k, v, L, d, v.shape[1],
                                              np.ascontiguousarray(rowptr, np.uint64),
                                              np.ascontiguousarray(cols, np.uint32), int(scale), z))
        return z

    def pipeline(self, q, k, v, p, bits, f32, mode, keep, vec_v=8, block=32, force_diag=False,
                 threads=1, per_row=False, frac_num=1, frac_den=1, cap=1, causal=False):
        """[pairs, L, d] doubles -> Z [pairs, L, d] through reference functions.
        mode 0 row top-k (per_row scales optional), 1 colvec, 2 block, 3 threshold."""
        q, k, v, p = _f64(q), _f64(k), _f64(v), _f64(p)
        pairs, L, d = q.shape
        z = np.empty_like(q)
        self._chk(self.L.ref_pipeline(pairs, threads, q, k, v, p, L, d, p.shape[1], bits, int(f32),
                                      mode, int(per_row), keep, vec_v, block, int(force_diag), frac_num,
                                      frac_den, cap, int(causal), z))
        return z

    # ---- the reference predictor (approx_scores / approx_scores_from_r)
    def levels_wtilde(self, w, bits, f32=False, x=None, p=None, r=None):
        """Levels / scale of quantize(matmul(R, W~)), R = matmul(x, p) when x is
        given (returned too), else r."""
        w = _f64(w)
        k = w.shape[0]
        xp = _f64(x) if x is not None else None
        L = xp.shape[0] if xp is not None else r.shape[0]
        dm = xp.shape[1] if xp is not None else 0
        pp = _f64(p) if p is not None else None
        rin = _f64(r) if r is not None else None
        rout = np.empty((L, k))
        lv = np.empty((L, k), np.int32)
        s = C.c_double()
        ptr = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None  # noqa: E731
        self._chk(self.L.ref_levels_wtilde(ptr(xp), ptr(pp), ptr(rin), w, L, dm, k, bits, int(f32),
                                           rout.ctypes.data_as(C.c_void_p), lv, C.byref(s)))
        return lv, s.value, rout

    def prediction_accuracy(self, rp_pred, c_pred, rp_orc, c_orc):
        out = C.c_double()
        f = lambda a, t: np.ascontiguousarray(a if len(a) else np.zeros(1), t)  # noqa: E731
        self._chk(self.L.ref_prediction_accuracy(len(rp_pred) - 1, f(rp_pred, np.uint64), f(c_pred, np.uint32),
                                                 f(rp_orc, np.uint64), f(c_orc, np.uint32), C.byref(out)))
        return out.value

    def dataflow_simulate(self, rp, cols, schedule, band):
        """dataflow::simulate (P/src/dataflow.cpp:48-62): (operand_fetches, pe_idle_steps)."""
        f, i = C.c_uint64(), C.c_uint64()
        kind = {"row_by_row": 0, "row_parallel": 1, "row_parallel_reordered": 2}[schedule]
        cc = np.ascontiguousarray(cols if len(cols) else np.zeros(1), np.uint32)
        self._chk(self.L.ref_dataflow_simulate(len(rp) - 1, np.ascontiguousarray(rp, np.uint64), cc, kind, band,
                                               C.byref(f), C.byref(i)))
        return f.value, i.value

    def init_projection(self, d, k, seed):
        out = np.empty((d, k))
        self._chk(self.L.ref_init_projection(d, k, seed, out))
        return out

    # ---- O5 / O6 compositions of reference primitives (block, causal threshold)
    def block_mask(self, lq, lk, bs, keep, force_diag):
        lq, lk = np.ascontiguousarray(lq, np.int32), np.ascontiguousarray(lk, np.int32)
        L = lq.shape[0]
        out = np.empty((-(-L // bs), keep), np.uint32)
        self._chk(self.L.ref_block_mask(lq, lk, L, lq.shape[1], bs, keep, int(force_diag), out))
        return out

    def causal_threshold_mask(self, lq, lk, c, theta, cap, causal):
        lq, lk = np.ascontiguousarray(lq, np.int32), np.ascontiguousarray(lk, np.int32)
        L = lq.shape[0]
        rp = np.zeros(L + 1, np.uint64)
        self._chk(self.L.ref_causal_threshold_mask(lq, lk, L, lq.shape[1], c, theta, cap, int(causal), rp, None))
        cols = np.empty(max(int(rp[-1]), 1), np.uint32)
        self._chk(self.L.ref_causal_threshold_mask(lq, lk, L, lq.shape[1], c, theta, cap, int(causal), rp,
                                                   cols.ctypes.data_as(C.c_void_p)))
        return rp, cols[: int(rp[-1])]

    def threshold_row_probs(self, lq, lk, c, i, causal):
        lq, lk = np.ascontiguousarray(lq, np.int32), np.ascontiguousarray(lk, np.int32)
        L = lq.shape[0]
        out = np.empty(i + 1 if causal else L)
        self._chk(self.L.ref_threshold_row_probs(lq, lk, L, lq.shape[1], c, i, int(causal), out))
        return out

    def generate(self, L, d, kdim, bf16, seed, planted_pm, band_w, pair0, npairs):
        """Seeded BASELINE inputs drawn with the reference Rng (doubles rounded
        to the dtype): q, k, v [npairs, L, d], P [d, kdim]."""
        q, k, v = (np.empty((npairs, L, d)) for _ in range(3))
        p = np.empty((d, kdim))
        self._chk(self.L.ref_generate(L, d, kdim, int(bf16), seed, planted_pm, band_w, pair0, npairs,
                                      q, k, v, p))
        return q, k, v, p
