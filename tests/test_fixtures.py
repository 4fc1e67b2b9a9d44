"""Fixture / wire formats: the harness's DSAMASK,
DSASPARSE and DSAC writers produce byte-identical files to the reference's
own writers (P/src/mask.cpp:75-89, P/src/sparse.cpp:122-139,
P/src/serialize.cpp:38-63, compiled into oracle/_ref), and each side reads
the other's files back exactly.  Error behaviour follows the reference
(IoError for format problems, ParamError for invalid masks)."""
import numpy as np
import pytest

from paper_2110_11299_b200 import fixtures as fx
from paper_2110_11299_b200.errors import IoError, ParamError

from oracle.oracle import REF_SO, REF_SRC


def _ref():
    from oracle.oracle import Reference

    if not REF_SO.exists() and not REF_SRC.exists():
        pytest.skip("reference library not built and sources absent")
    return Reference()


def _mask(rng, l, counts):
    rows = [np.sort(rng.choice(l, size=c, replace=False)).astype(np.uint32) for c in counts]
    rp = np.zeros(l + 1, np.uint64)
    rp[1:] = np.cumsum(counts)
    cols = np.concatenate(rows) if sum(counts) else np.zeros(0, np.uint32)
    return rp, cols.astype(np.uint32)


CASES = [("ragged", [3, 0, 7, 1, 5, 0, 2, 9]), ("balanced", [4] * 8), ("empty", [0] * 5)]


@pytest.mark.parametrize("name,counts", CASES)
def test_mask_bytes_and_roundtrip(tmp_path, name, counts):
    ref = _ref()
    rng = np.random.default_rng(7)
    l = len(counts) if name != "ragged" else 16
    counts = counts[:l] + [0] * (l - len(counts))
    rp, cols = _mask(rng, l, counts)
    ours, theirs = tmp_path / "ours.mask", tmp_path / "theirs.mask"
    fx.write_mask(ours, rp, cols)
    ref.write_mask(theirs, rp, cols)
    assert ours.read_bytes() == theirs.read_bytes()
    for path in (ours, theirs):
        a_rp, a_cols = fx.read_mask(path)
        b_rp, b_cols = ref.read_mask(path)
        assert np.array_equal(a_rp, rp) and np.array_equal(b_rp, rp)
        assert np.array_equal(a_cols, cols) and np.array_equal(b_cols, cols)


def test_sparse_scores_bytes_and_roundtrip(tmp_path):
    ref = _ref()
    rng = np.random.default_rng(11)
    rp, cols = _mask(rng, 12, [2, 0, 5, 3, 1, 0, 4, 6, 2, 2, 0, 1])
    vals = rng.normal(size=int(rp[-1])) * np.array([1e-7, 1.0, 3e5, 0.1] * 10)[: int(rp[-1])]
    vals[0] = 2.0  # integer-valued prints without a fraction
    ours, theirs = tmp_path / "ours.sparse", tmp_path / "theirs.sparse"
    fx.write_sparse_scores(ours, rp, cols, vals)
    ref.write_sparse_scores(theirs, rp, cols, vals)
    assert ours.read_bytes() == theirs.read_bytes()
    for path in (ours, theirs):
        a = fx.read_sparse_scores(path)
        b = ref.read_sparse_scores(path)
        for x, y, want in zip(a, b, (rp, cols, vals)):
            assert np.array_equal(x, want) and np.array_equal(y, want)


@pytest.mark.parametrize("f32", [False, True])
def test_container_bytes_and_roundtrip(tmp_path, f32):
    ref = _ref()
    rng = np.random.default_rng(3)
    a = rng.normal(size=(5, 7))
    if f32:
        a = a.astype(np.float32).astype(np.float64)
    meta = '{"config": "c0_smoke", "pair": 0}'
    ours, theirs = tmp_path / "ours.dsac", tmp_path / "theirs.dsac"
    fx.write_container(ours, [("z", a, f32)], meta)
    ref.write_container1(theirs, "z", a, f32=f32, meta=meta)
    assert ours.read_bytes() == theirs.read_bytes()
    m, entries = fx.read_container(theirs)
    assert m == meta and entries["z"][1] == f32 and np.array_equal(entries["z"][0], a)
    b, bf32, bmeta = ref.read_container1(ours, "z")
    assert bmeta == meta and bf32 == f32 and np.array_equal(b, a)


def test_errors(tmp_path):
    p = tmp_path / "bad.mask"
    p.write_text("DSAMASK 2\n1 -1\n\n")
    with pytest.raises(IoError):
        fx.read_mask(p)
    p.write_text("DSAMASK 1\n2 -1\n3 1\n")  # truncated + unsorted
    with pytest.raises(IoError):
        fx.read_mask(p)
    p.write_text("DSAMASK 1\n2 -1\n3 1\n0\n")
    with pytest.raises(ParamError):
        fx.read_mask(p)
    p.write_text("DSAMASK 1\n2 5\n0\n1\n")  # balanced header mismatch
    with pytest.raises(IoError):
        fx.read_mask(p)
    q = tmp_path / "bad.dsac"
    q.write_bytes(b"DSAX")
    with pytest.raises(IoError):
        fx.read_container(q)
    with pytest.raises(IoError):
        fx.read_mask(tmp_path / "missing.mask")


@pytest.mark.gpu
def test_gpu_run_exports_reference_readable_fixtures(tmp_path, oracle):
    """A GPU run's mask and Z written as fixtures are read back by the
    reference's own readers and match the oracle's mask / the GPU output."""
    from paper_2110_11299_b200 import load_preset, ops

    from test_gpu_parity import oracle_levels, oracle_mask_rows, run_gpu

    ref = _ref()
    p = load_preset("c2_vector").replace(L=512, keep=26)
    sub, (q, k, v, P), lv, mask, z = run_gpu(p, 2)
    files = fx.export_pair(sub, mask, z, 1, tmp_path)
    rp, cols = ref.read_mask(files["mask"])
    lq, sq = oracle_levels(oracle, sub, q[1], P)
    lk, sk = oracle_levels(oracle, sub, k[1], P)
    want_rp, want_cols = ops.to_csr(oracle_mask_rows(oracle, sub, lq, lk, sq, sk))
    assert np.array_equal(rp, want_rp) and np.array_equal(cols, want_cols)
    zr, f32, meta = ref.read_container1(files["z"], "z")
    assert not f32 and '"pair": 1' in meta
    assert np.array_equal(zr, z[1].double().cpu().numpy())
