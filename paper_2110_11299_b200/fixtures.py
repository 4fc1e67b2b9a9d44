"""Fixture / wire formats of the reference, read and written by the GPU
harness so masks, sparse scores and matrices round-trip with the reference
tools:

* DSAMASK 1   -- text mask (P/src/mask.cpp:75-114): header ``DSAMASK 1``,
  then ``<l> <balanced count or -1>``, then one line per query row with its
  ascending kept columns;
* DSASPARSE 1 -- text sparse scores (P/src/sparse.cpp:122-171): the same
  layout with ``col:value`` tokens, values at 17 significant digits;
* DSAC 1      -- binary matrix container (P/src/serialize.cpp:38-95):
  ``"DSAC" | u32 1 | u32 count | u32 meta_len | meta`` then per entry
  ``u32 name_len | name | u64 rows | u64 cols | u8 precision (0 f32, 1 f64) |
  payload``, little-endian.

Errors raise the reference's types (IoError for format problems, ParamError
for invalid masks, P/src/mask.cpp:60-72).  Masks are (rowptr, cols) CSR
arrays (uint64 / uint32), the layout of the C-ABI threshold masks and of
``ops.to_csr``.
"""
from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np

from .errors import IoError, ParamError

__all__ = ["write_mask", "read_mask", "write_sparse_scores", "read_sparse_scores",
           "write_container", "read_container", "export_pair", "validate_mask"]


def _rows(rowptr: np.ndarray, cols: np.ndarray) -> list[np.ndarray]:
    rp = np.asarray(rowptr, dtype=np.int64)
    c = np.asarray(cols)
    return [c[rp[i]:rp[i + 1]] for i in range(len(rp) - 1)]


def validate_mask(l: int, rowptr: np.ndarray, cols: np.ndarray) -> None:
    """SparseMask::validate (P/src/mask.cpp:60-72): columns < l, strictly
    ascending (hence duplicate-free) per row."""
    for i, r in enumerate(_rows(rowptr, cols)):
        if r.size == 0:
            continue
        if int(r.max()) >= l:
            raise ParamError("SparseMask: column index out of range")
        if r.size > 1 and np.any(np.diff(r.astype(np.int64)) <= 0):
            raise ParamError("SparseMask: row not strictly ascending")


def _balanced(rowptr: np.ndarray) -> int:
    n = np.diff(np.asarray(rowptr, dtype=np.int64))
    if n.size == 0 or np.any(n != n[0]):
        return -1
    return int(n[0])


def write_mask(path, rowptr: np.ndarray, cols: np.ndarray) -> None:
    l = len(rowptr) - 1
    lines = ["DSAMASK 1", f"{l} {_balanced(rowptr)}"]
    lines += [" ".join(str(int(c)) for c in r) for r in _rows(rowptr, cols)]
    try:
        Path(path).write_text("\n".join(lines) + "\n")
    except OSError as e:
        raise IoError(f"write_mask: cannot open {path}") from e


def _read_header(path, magic: str):
    try:
        text = Path(path).read_text()
    except OSError as e:
        raise IoError(f"read: cannot open {path}") from e
    lines = text.split("\n")
    if lines and lines[-1] == "":  # std::getline: a final newline ends the last line
        lines.pop()
    head = lines[0].split() if lines else []
    if len(head) != 2 or head[0] != magic or head[1] != "1":
        raise IoError(f"read: bad header in {path}")
    if len(lines) < 2 or len(lines[1].split()) < 2:
        raise IoError(f"read: truncated file {path}")
    l, balanced = (int(x) for x in lines[1].split()[:2])
    body = lines[2:]
    if len(body) < l:
        raise IoError(f"read: truncated file {path}")
    return l, balanced, body[:l]


def read_mask(path) -> tuple[np.ndarray, np.ndarray]:
    l, balanced, body = _read_header(path, "DSAMASK")
    rows = [np.array([int(t) for t in line.split()], dtype=np.uint32) for line in body]
    rp = np.zeros(l + 1, dtype=np.uint64)
    rp[1:] = np.cumsum([r.size for r in rows]) if rows else []
    cols = np.concatenate(rows).astype(np.uint32) if rows and rp[-1] > 0 else np.zeros(0, np.uint32)
    validate_mask(l, rp, cols)
    if balanced >= 0 and _balanced(rp) != balanced:
        raise IoError(f"read_mask: balanced-count header mismatch in {path}")
    return rp, cols


def write_sparse_scores(path, rowptr: np.ndarray, cols: np.ndarray, values: np.ndarray) -> None:
    l = len(rowptr) - 1
    rp = np.asarray(rowptr, dtype=np.int64)
    vals = np.asarray(values, dtype=np.float64)
    lines = ["DSASPARSE 1", f"{l} {_balanced(rowptr)}"]
    for i in range(l):
        lines.append(" ".join(f"{int(cols[p])}:{format(float(vals[p]), '.17g')}" for p in range(rp[i], rp[i + 1])))
    try:
        Path(path).write_text("\n".join(lines) + "\n")
    except OSError as e:
        raise IoError(f"write_sparse_scores: cannot open {path}") from e


def read_sparse_scores(path) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    l, _, body = _read_header(path, "DSASPARSE")
    cols, vals, rp = [], [], np.zeros(l + 1, dtype=np.uint64)
    for i, line in enumerate(body):
        for tok in line.split():
            if ":" not in tok:
                raise IoError(f"read_sparse_scores: bad token in {path}")
            c, v = tok.split(":", 1)
            cols.append(int(c))
            vals.append(float(v))
        rp[i + 1] = len(cols)
    cols_a = np.array(cols, dtype=np.uint32)
    validate_mask(l, rp, cols_a)
    return rp, cols_a, np.array(vals, dtype=np.float64)


def write_container(path, entries: list[tuple[str, np.ndarray, bool]], meta: str | dict = "") -> None:
    """entries: (name, 2-D array, f32).  f32 entries are stored as 4-byte floats."""
    meta_s = json.dumps(meta) if isinstance(meta, dict) else meta
    mb = meta_s.encode()
    out = [b"DSAC", struct.pack("<III", 1, len(entries), len(mb)), mb]
    for name, arr, f32 in entries:
        a = np.asarray(arr)
        if a.ndim != 2:
            raise ParamError("write_container: entries must be 2-D")
        nb = name.encode()
        out.append(struct.pack("<I", len(nb)) + nb + struct.pack("<QQB", a.shape[0], a.shape[1], 0 if f32 else 1))
        out.append(np.ascontiguousarray(a, dtype="<f4" if f32 else "<f8").tobytes())
    try:
        Path(path).write_bytes(b"".join(out))
    except OSError as e:
        raise IoError(f"write_container: cannot open {path}") from e


def read_container(path) -> tuple[str, dict[str, tuple[np.ndarray, bool]]]:
    """Returns (meta, {name: (array as float64, f32)})."""
    try:
        b = Path(path).read_bytes()
    except OSError as e:
        raise IoError(f"read_container: cannot open {path}") from e
    if b[:4] != b"DSAC":
        raise IoError(f"read_container: bad magic in {path}")
    try:
        ver, count, mlen = struct.unpack_from("<III", b, 4)
        if ver != 1:
            raise IoError(f"read_container: unsupported version in {path}")
        off = 16
        meta = b[off:off + mlen].decode()
        off += mlen
        out = {}
        for _ in range(count):
            (nlen,) = struct.unpack_from("<I", b, off)
            off += 4
            name = b[off:off + nlen].decode()
            off += nlen
            rows, cols, prec = struct.unpack_from("<QQB", b, off)
            off += 17
            dt, sz = ("<f4", 4) if prec == 0 else ("<f8", 8)
            n = rows * cols
            if off + n * sz > len(b):
                raise IoError(f"read_container: truncated file {path}")
            arr = np.frombuffer(b, dtype=dt, count=n, offset=off).astype(np.float64).reshape(rows, cols)
            off += n * sz
            out[name] = (arr, prec == 0)
    except struct.error as e:
        raise IoError(f"read_container: truncated file {path}") from e
    return meta, out


def export_pair(p, mask, z, pair: int, directory) -> dict:
    """Writes one (b,h) pair of a GPU run as reference fixtures: the mask
    (DSAMASK) and Z (DSAC, entry "z", f32 when the config computes in f32)."""
    from . import ops

    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    rows = ops.mask_rows(p, mask, pair + 1)[pair]
    rp, cols = ops.to_csr(rows)
    mpath, zpath = d / f"{p.name}_pair{pair}.mask", d / f"{p.name}_pair{pair}.dsac"
    write_mask(mpath, rp, cols)
    zp = z[pair].double().cpu().numpy()
    write_container(zpath, [("z", zp, p.dtype == "f32")], {"config": p.name, "pair": pair})
    return {"mask": str(mpath), "z": str(zpath)}
