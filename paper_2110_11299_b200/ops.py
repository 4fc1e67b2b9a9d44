"""Host-side mirror of the reference attention-operator interface over the
C-ABI (PyTorch is used only for device memory and streams).

Names follow the reference entry points (P/include/dsattn/predictor.hpp:31-49,
maskgen.hpp:14-31, sparse.hpp:47-59): ``quantize``-style prediction
(``predict``), mask selection (``predicted_topk_mask``, ``colvec_mask``,
``block_mask``, ``threshold_mask`` -> ``select``), ``sparse_attention`` and
the fused ``pipeline``.  Errors surface as the reference exception types
(errors.py).  Everything runs batched over (b, h) pairs with tensors shaped
[pairs, L, d] on one CUDA device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from .errors import ParamError, ShapeError
from .presets import DTYPES, MASK_MODES, QUANT_SCOPES, Preset


def config_of(p: Preset, pairs: int | None = None) -> _abi.DsaConfig:
    """dsa_config for a preset; `pairs` overrides batch*heads (heads := 1)."""
    c = _abi.DsaConfig()
    if pairs is None:
        c.batch, c.heads = p.batch, p.heads
    else:
        c.batch, c.heads = pairs, 1
    c.L, c.d, c.k = p.L, p.d, p.k
    c.dtype = DTYPES[p.dtype]
    c.bits = p.bits
    c.quant_scope = QUANT_SCOPES[p.quant_scope]
    c.round_proj_f32 = int(p.round_proj_f32)
    c.mask_mode = MASK_MODES[p.mask_mode]
    c.scale = int(p.scale)
    c.keep = p.keep
    c.vec_v, c.block, c.force_diag = p.vec_v, p.block, int(p.force_diag)
    c.causal = int(p.causal)
    c.frac_num, c.frac_den, c.cap = p.frac_num, p.frac_den, p.cap
    return c


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream


def torch_dtype(p: Preset) -> torch.dtype:
    return torch.bfloat16 if p.dtype == "bf16" else torch.float32


def validate(p: Preset, pairs: int | None = None) -> None:
    c = config_of(p, pairs)
    _abi.check(_abi.lib().dsa_config_validate(C.byref(c)))


def workspace_bytes(p: Preset, pairs: int | None = None) -> int:
    c = config_of(p, pairs)
    n = _abi.lib().dsa_workspace_bytes(C.byref(c))
    if n == 0:
        _abi.check(_abi.lib().dsa_config_validate(C.byref(c)))
    return int(n)


def mask_capacity(p: Preset, pairs: int | None = None) -> int:
    c = config_of(p, pairs)
    n = _abi.lib().dsa_mask_capacity(C.byref(c))
    if n < 0:
        _abi.check(_abi.lib().dsa_config_validate(C.byref(c)))
    return int(n)


# ------------------------------------------------------------------ inputs
def generate(p: Preset, pair0: int = 0, npairs: int | None = None, threads: int = 0,
             pinned: bool = False):
    """Seeded BASELINE inputs on the host: q, k, v as torch CPU tensors
    [npairs, L, d] in the preset dtype, plus P [d, k] float32."""
    import os
    npairs = p.pairs if npairs is None else npairs
    dt = torch_dtype(p)
    shape = (npairs, p.L, p.d)
    q = torch.empty(shape, dtype=dt, pin_memory=pinned)
    k = torch.empty(shape, dtype=dt, pin_memory=pinned)
    v = torch.empty(shape, dtype=dt, pin_memory=pinned)
    P = torch.empty((p.d, p.k), dtype=torch.float32, pin_memory=pinned)
    c = config_of(p)
    _abi.check(_abi.lib().dsa_generate(C.byref(c), p.seed, p.planted_per_mille, p.band_width,
                                       pair0, npairs, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                       P.data_ptr(), threads or (os.cpu_count() or 1)))
    return q, k, v, P


# ------------------------------------------------------------------ phases
def levels_rows(t: torch.Tensor) -> torch.Tensor:
    """Chunk-planar levels [pairs, k/8, L, 8] -> row-major [pairs, L, k]."""
    pairs, kc, L, _ = t.shape
    return t.permute(0, 2, 1, 3).reshape(pairs, L, kc * 8)


@dataclass
class Levels:
    lq: torch.Tensor   # [pairs, k/8, L, 8] bf16 chunk-planar (exact integer levels)
    lk: torch.Tensor
    sq: torch.Tensor   # f64 [pairs] or [pairs, L]
    sk: torch.Tensor


@dataclass
class Mask:
    mode: str
    cols: torch.Tensor
    rowptr: torch.Tensor | None
    empty_rows: torch.Tensor | None

    def as_c(self) -> _abi.DsaMask:
        m = _abi.DsaMask()
        m.cols = _ptr(self.cols)
        m.rowptr = _ptr(self.rowptr)
        m.capacity = self.cols.numel()
        m.empty_rows = _ptr(self.empty_rows)
        return m


def _check_inputs(p: Preset, pairs: int, *ts: torch.Tensor) -> None:
    for t in ts:
        if t.shape != (pairs, p.L, p.d):
            raise ShapeError(f"dsa: expected [{pairs}, {p.L}, {p.d}], got {list(t.shape)}")
        if t.dtype != torch_dtype(p):
            raise ParamError(f"dsa: expected {torch_dtype(p)}, got {t.dtype}")
        if not t.is_cuda or not t.is_contiguous():
            raise ParamError("dsa: inputs must be contiguous CUDA tensors")


def _ws(nbytes: int, device, stream=None) -> torch.Tensor:
    """Scratch for one call.  The caching allocator hands out memory per
    stream, so a buffer used by a launch on another stream is tied to it
    (record_stream) and is not reused before that stream's work is done."""
    t = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
    if stream is not None and t.is_cuda:
        t.record_stream(stream)
    return t


def _check_projection(p: Preset, P: torch.Tensor) -> None:
    if P.shape != (p.d, p.k) or P.dtype != torch.float32 or not P.is_cuda or not P.is_contiguous():
        raise ParamError(f"dsa: P must be a contiguous CUDA float32 tensor of shape [{p.d}, {p.k}]")


def predict(p: Preset, q: torch.Tensor, k: torch.Tensor, P: torch.Tensor, stream=None) -> Levels:
    pairs = q.shape[0]
    _check_inputs(p, pairs, q, k)
    _check_projection(p, P)
    c = config_of(p, pairs)
    dev = q.device
    lq = torch.empty((pairs, p.k // 8, p.L, 8), dtype=torch.bfloat16, device=dev)
    lk = torch.empty_like(lq)
    ns = (pairs,) if p.quant_scope == "tensor" else (pairs, p.L)
    sq = torch.empty(ns, dtype=torch.float64, device=dev)
    sk = torch.empty_like(sq)
    ws = _ws(workspace_bytes(p, pairs), dev, stream)
    _abi.check(_abi.lib().dsa_predict(C.byref(c), _ptr(q), _ptr(k), _ptr(P), _ptr(lq),
                                      _ptr(lk), _ptr(sq), _ptr(sk), _ptr(ws), ws.numel(),
                                      _stream(stream)))
    return Levels(lq, lk, sq, sk)


def predict_wtilde(p: Preset, wq: torch.Tensor, wk: torch.Tensor, x: torch.Tensor | None = None,
                   P: torch.Tensor | None = None, r: torch.Tensor | None = None, stream=None):
    """The reference predictor, approx_scores / approx_scores_from_r
    (P/src/predictor.cpp:67-80): R = X P once per sample (returned), then per
    head Q~ = quantize(R W~_Q[h]), K~ = quantize(R W~_K[h]), bit-exact fp64
    chains.  x [batch, L, d_model] f64, P [d_model, k] f64 (or r [batch, L, k]
    f64 instead), wq/wk [heads, k, k] f64, all CUDA.  Returns (Levels, r)."""
    batch = (x if x is not None else r).shape[0]
    if p.batch != batch:
        raise ShapeError(f"predict_wtilde: preset batch {p.batch} != input batch {batch}")
    for t in (wq, wk):
        if t.shape != (p.heads, p.k, p.k) or t.dtype != torch.float64 or not t.is_cuda:
            raise ShapeError(f"predict_wtilde: W~ must be [{p.heads}, {p.k}, {p.k}] float64 CUDA")
    c = config_of(p)
    dev = wq.device
    dm = 0
    if x is not None:
        dm = x.shape[2]
        if x.shape != (batch, p.L, dm) or P is None or P.shape != (dm, p.k):
            raise ShapeError("approx_scores: X feature dim != d")
        r = torch.empty((batch, p.L, p.k), dtype=torch.float64, device=dev)
    elif r is None or r.shape != (batch, p.L, p.k):
        raise ShapeError("approx_scores: R width != projection k")
    pairs = p.pairs
    lq = torch.empty((pairs, p.k // 8, p.L, 8), dtype=torch.bfloat16, device=dev)
    lk = torch.empty_like(lq)
    ns = (pairs,) if p.quant_scope == "tensor" else (pairs, p.L)
    sq = torch.empty(ns, dtype=torch.float64, device=dev)
    sk = torch.empty_like(sq)
    ws = _ws(int(_abi.lib().dsa_predict_wtilde_workspace_bytes(C.byref(c))), dev, stream)
    _abi.check(_abi.lib().dsa_predict_wtilde(C.byref(c), dm, _ptr(x), _ptr(P), _ptr(r), _ptr(wq.contiguous()),
                                             _ptr(wk.contiguous()), _ptr(lq), _ptr(lk), _ptr(sq), _ptr(sk),
                                             _ptr(ws), ws.numel(), _stream(stream)))
    return Levels(lq, lk, sq, sk), r


def alloc_mask(p: Preset, pairs: int, device, empty_rows: bool = True) -> Mask:
    cap = mask_capacity(p, pairs)
    cols = torch.empty(cap, dtype=torch.int32, device=device)
    rowptr = (torch.empty(pairs * p.L + 1, dtype=torch.int64, device=device)
              if p.mask_mode == "threshold" else None)
    er = torch.zeros(pairs * p.L, dtype=torch.uint8, device=device) if empty_rows else None
    return Mask(p.mask_mode, cols, rowptr, er)


def select(p: Preset, lv: Levels, stream=None, mask: Mask | None = None) -> Mask:
    pairs = lv.lq.shape[0]
    c = config_of(p, pairs)
    dev = lv.lq.device
    m = mask or alloc_mask(p, pairs, dev)
    ws = _ws(workspace_bytes(p, pairs), dev, stream)
    cm = m.as_c()
    _abi.check(_abi.lib().dsa_select(C.byref(c), _ptr(lv.lq), _ptr(lv.lk), _ptr(lv.sq),
                                     _ptr(lv.sk), C.byref(cm), _ptr(ws), ws.numel(),
                                     _stream(stream)))
    return m


def sparse_attention(p: Preset, q, k, v, mask: Mask, stream=None, out=None) -> torch.Tensor:
    pairs = q.shape[0]
    _check_inputs(p, pairs, q, k, v)
    c = config_of(p, pairs)
    z = out if out is not None else torch.empty_like(q)
    cm = mask.as_c()
    _abi.check(_abi.lib().dsa_sparse_attention(C.byref(c), _ptr(q), _ptr(k), _ptr(v), C.byref(cm),
                                               _ptr(z), _stream(stream)))
    return z


class Pipeline:
    """predict -> select -> sparse attention with a pre-sized workspace
    (allocation-free per call; capturable in a CUDA graph)."""

    def __init__(self, p: Preset, pairs: int | None = None, device="cuda", keep_mask=False):
        self.p = p
        self.pairs = p.pairs if pairs is None else pairs
        self.cfg = config_of(p, self.pairs)
        self.ws = _ws(workspace_bytes(p, self.pairs), device)
        self.mask = alloc_mask(p, self.pairs, device) if keep_mask else None
        self._cmask = self.mask.as_c() if self.mask else None

    def __call__(self, q, k, v, P, out=None, stream=None) -> torch.Tensor:
        z = out if out is not None else torch.empty_like(q)
        mp = C.byref(self._cmask) if self._cmask is not None else None
        _abi.check(_abi.lib().dsa_pipeline(C.byref(self.cfg), _ptr(q), _ptr(k), _ptr(v), _ptr(P),
                                           _ptr(z), mp, _ptr(self.ws), self.ws.numel(),
                                           _stream(stream)))
        return z


class Phases:
    """The three phases as separate, allocation-free calls on preallocated
    buffers (bench.py times each with CUDA events)."""

    def __init__(self, p: Preset, pairs: int, device="cuda"):
        self.p, self.pairs = p, pairs
        self.cfg = config_of(p, pairs)
        self.ws = _ws(workspace_bytes(p, pairs), device)
        self.lq = torch.empty((pairs, p.k // 8, p.L, 8), dtype=torch.bfloat16, device=device)
        self.lk = torch.empty_like(self.lq)
        ns = (pairs,) if p.quant_scope == "tensor" else (pairs, p.L)
        self.sq = torch.empty(ns, dtype=torch.float64, device=device)
        self.sk = torch.empty_like(self.sq)
        self.mask = alloc_mask(p, pairs, device, empty_rows=False)
        self._cm = self.mask.as_c()

    def predict(self, q, k, P, stream=None):
        _abi.check(_abi.lib().dsa_predict(C.byref(self.cfg), _ptr(q), _ptr(k), _ptr(P), _ptr(self.lq),
                                          _ptr(self.lk), _ptr(self.sq), _ptr(self.sk), _ptr(self.ws),
                                          self.ws.numel(), _stream(stream)))

    def select(self, stream=None):
        _abi.check(_abi.lib().dsa_select(C.byref(self.cfg), _ptr(self.lq), _ptr(self.lk),
                                         _ptr(self.sq), _ptr(self.sk), C.byref(self._cm),
                                         _ptr(self.ws), self.ws.numel(), _stream(stream)))

    def attend(self, q, k, v, z, stream=None):
        _abi.check(_abi.lib().dsa_sparse_attention(C.byref(self.cfg), _ptr(q), _ptr(k), _ptr(v),
                                                   C.byref(self._cm), _ptr(z), _stream(stream)))


# ------------------------------------------------- step before the path
def pack_qkv_weights(wq, wk, wv, p_model=None) -> torch.Tensor:
    """Reference per-head weights (lists of [d_model, d] matrices, as in
    AttentionParams wq/wk/wv, P/include/dsattn/attention.hpp) and the
    optional predictor projection P [d_model, npred] -> the K-major packed
    operand [H*(2dk+dv) + npred, d_model] bf16 of dsa_project_qkv."""
    rows = [w.t() for w in wq] + [w.t() for w in wk] + [w.t() for w in wv]
    if p_model is not None:
        rows.append(p_model.t())
    return torch.cat([r.to(torch.bfloat16) for r in rows], 0).contiguous()


def project_qkv(x: torch.Tensor, w: torch.Tensor, heads: int, dk: int, dv: int, npred: int = 0,
                stream=None, out=None):
    """project_qkv (P/src/attention.cpp:36-46) for every head plus the
    predictor input R = X P (P/src/trainer.cpp:162) in one tensor-core GEMM.
    x: [batch, L, d_model] bf16 CUDA; w: pack_qkv_weights(...).  Returns
    (q, k, v, r): q/k [batch*heads, L, dk], v [batch*heads, L, dv] bf16 (the
    (b,h)-pair layout the hot path consumes), r [batch, L, npred] f32 or None."""
    if x.dim() != 3 or x.dtype != torch.bfloat16 or not x.is_cuda or not x.is_contiguous():
        raise ParamError("project_qkv: x must be a contiguous [batch, L, d_model] bf16 CUDA tensor")
    batch, L, dm = x.shape
    n_out = heads * (2 * dk + dv) + npred
    if w.shape != (n_out, dm) or w.dtype != torch.bfloat16 or not w.is_contiguous():
        raise ShapeError(f"project_qkv: packed weights must be [{n_out}, {dm}] bf16")
    if out is None:
        q = torch.empty((batch * heads, L, dk), dtype=torch.bfloat16, device=x.device)
        k = torch.empty_like(q)
        v = torch.empty((batch * heads, L, dv), dtype=torch.bfloat16, device=x.device)
        r = torch.empty((batch, L, npred), dtype=torch.float32, device=x.device) if npred else None
    else:
        q, k, v, r = out
    _abi.check(_abi.lib().dsa_project_qkv(batch, L, dm, heads, dk, dv, npred, _ptr(x), _ptr(w), _ptr(q),
                                          _ptr(k), _ptr(v), _ptr(r), _stream(stream)))
    return q, k, v, r


def fused_pipeline(p: Preset, pairs: int | None = None) -> bool:
    """True when dsa_pipeline fuses selection + attention into one kernel."""
    c = config_of(p, pairs)
    r = _abi.lib().dsa_pipeline_fused(C.byref(c))
    if r < 0:
        _abi.check(_abi.lib().dsa_config_validate(C.byref(c)))
    return r == 1


def prediction_accuracy(p: Preset, pred: Mask, oracle: Mask, pairs: int, stream=None) -> float:
    """prediction_accuracy (P/src/maskgen.cpp:94-107) of two device masks of
    the preset's layout: |pred n oracle| / |pred| over every pair."""
    c = config_of(p, pairs)
    out = C.c_double()
    a, b = pred.as_c(), oracle.as_c()
    _abi.check(_abi.lib().dsa_prediction_accuracy(C.byref(c), C.byref(a), C.byref(b), C.byref(out),
                                                  _stream(stream)))
    return out.value


SCHEDULES = {"row_by_row": 0, "row_parallel": 1, "row_parallel_reordered": 2}


def dataflow_trace(p: Preset, mask: Mask, pairs: int, schedule: str, band: int, stream=None):
    """The reference's dataflow::simulate (P/src/dataflow.cpp:10-62) on a device
    mask: per (b,h) pair, (operand_fetches, pe_idle_steps) as two uint64 arrays."""
    c = config_of(p, pairs)
    cm = mask.as_c()
    f = np.zeros(pairs, dtype=np.uint64)
    i = np.zeros(pairs, dtype=np.uint64)
    _abi.check(_abi.lib().dsa_dataflow_trace(C.byref(c), C.byref(cm), SCHEDULES[schedule], band,
                                             f.ctypes.data, i.ctypes.data, _stream(stream)))
    return f, i


def row_topk(scores: torch.Tensor, keep: int, stream=None) -> torch.Tensor:
    """The reference's row_topk_indices (P/src/linalg.cpp:69-85) on a CUDA float64
    matrix: [rows, keep] int32 column indices, ascending per row."""
    if scores.dim() != 2 or scores.dtype != torch.float64 or not scores.is_cuda or not scores.is_contiguous():
        raise ParamError("dsa: row_topk takes a contiguous CUDA float64 matrix")
    out = torch.empty((scores.shape[0], max(keep, 0)), dtype=torch.int32, device=scores.device)
    _abi.check(_abi.lib().dsa_row_topk_f64(scores.shape[0], scores.shape[1], _ptr(scores), keep, _ptr(out),
                                           _stream(stream)))
    return out


def _check_csr(rowptr: torch.Tensor, cols: torch.Tensor, *vals: torch.Tensor) -> None:
    if rowptr.dtype != torch.int64 or cols.dtype != torch.int32 or not rowptr.is_cuda or not cols.is_cuda:
        raise ParamError("dsa: CSR needs CUDA int64 rowptr (u64 bits) and int32 cols (u32 bits)")
    for t in vals:
        if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
            raise ParamError("dsa: the unfused operators take contiguous CUDA float64 tensors")


def sddmm(q: torch.Tensor, k: torch.Tensor, rowptr: torch.Tensor, cols: torch.Tensor, scale: bool = True,
          stream=None) -> torch.Tensor:
    """The reference's sddmm (P/src/sparse.cpp:38-53) for one head: f64 Q, K
    [L, d], CSR (rowptr [L + 1], cols [nnz]); returns the nnz scores."""
    _check_csr(rowptr, cols, q, k)
    if q.shape != k.shape:
        raise ShapeError("sddmm: Q/K feature dims differ")
    vals = torch.empty(cols.numel(), dtype=torch.float64, device=q.device)
    _abi.check(_abi.lib().dsa_sddmm_f64(q.shape[0], q.shape[1], _ptr(q), _ptr(k), _ptr(rowptr), _ptr(cols),
                                        1 if scale else 0, _ptr(vals), _stream(stream)))
    return vals


def sparse_softmax(scores: torch.Tensor, rowptr: torch.Tensor, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
    """The reference's sparse_softmax (P/src/sparse.cpp:55-78): (weights, empty_row flags)."""
    _check_csr(rowptr, torch.empty(0, dtype=torch.int32, device=scores.device), scores)
    rows = rowptr.numel() - 1
    w = torch.zeros_like(scores)
    empty = torch.zeros(rows, dtype=torch.uint8, device=scores.device)
    _abi.check(_abi.lib().dsa_sparse_softmax_f64(rows, _ptr(rowptr), _ptr(scores), _ptr(w), _ptr(empty),
                                                 _stream(stream)))
    return w, empty


def spmm(weights: torch.Tensor, rowptr: torch.Tensor, cols: torch.Tensor, v: torch.Tensor, stream=None) -> torch.Tensor:
    """The reference's spmm (P/src/sparse.cpp:80-91): Z [L, d_v] in f64, empty rows zero."""
    _check_csr(rowptr, cols, weights, v)
    rows = rowptr.numel() - 1
    if v.shape[0] != rows:
        raise ShapeError("spmm: V rows != sequence length")
    z = torch.empty((rows, v.shape[1]), dtype=torch.float64, device=v.device)
    _abi.check(_abi.lib().dsa_spmm_f64(rows, v.shape[1], _ptr(rowptr), _ptr(cols), _ptr(weights), _ptr(v), _ptr(z),
                                       _stream(stream)))
    return z


def launch_counter() -> int:
    return int(_abi.lib().dsa_launch_counter())


def counters(p: Preset, mask: Mask, pairs: int, stream=None) -> dict:
    c = config_of(p, pairs)
    out = _abi.DsaCounts()
    cm = mask.as_c()
    _abi.check(_abi.lib().dsa_counters(C.byref(c), C.byref(cm), C.byref(out), _stream(stream)))
    return {f: getattr(out, f) for f, _ in out._fields_}


# --------------------------------------------------------- mask utilities
def mask_rows(p: Preset, mask: Mask, pairs: int) -> list[list[np.ndarray]]:
    """Per pair, per query row, the kept key columns (host, ascending)."""
    cols = mask.cols.cpu().numpy().astype(np.int64)
    out = []
    if p.mask_mode == "threshold":
        rp = mask.rowptr.cpu().numpy()
        for pr in range(pairs):
            out.append([cols[rp[pr * p.L + i]:rp[pr * p.L + i + 1]] for i in range(p.L)])
        return out
    if p.mask_mode == "row_topk":
        c3 = cols[: pairs * p.L * p.keep].reshape(pairs, p.L, p.keep)
        return [[c3[pr, i] for i in range(p.L)] for pr in range(pairs)]
    if p.mask_mode == "colvec":
        nb = -(-p.L // p.vec_v)
        c3 = cols[: pairs * nb * p.keep].reshape(pairs, nb, p.keep)
        return [[c3[pr, i // p.vec_v] for i in range(p.L)] for pr in range(pairs)]
    nb = -(-p.L // p.block)
    c3 = cols[: pairs * nb * p.keep].reshape(pairs, nb, p.keep)
    res = []
    for pr in range(pairs):
        rows = []
        for ib in range(nb):
            ks = np.concatenate([np.arange(b * p.block, min((b + 1) * p.block, p.L)) for b in c3[pr, ib]])
            rows.extend([ks] * (min((ib + 1) * p.block, p.L) - ib * p.block))
        res.append(rows)
    return res


def to_csr(rows: list[np.ndarray]) -> tuple[np.ndarray, np.ndarray]:
    rp = np.zeros(len(rows) + 1, dtype=np.uint64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    cols = np.concatenate(rows).astype(np.uint32) if rows and rp[-1] > 0 else np.zeros(0, np.uint32)
    return rp, cols
