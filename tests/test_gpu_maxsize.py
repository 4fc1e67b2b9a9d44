"""The largest sequence lengths the C ABI accepts (dsa_config_validate:
L <= 51200 for row top-k / colvec / threshold, 25600 for per-row scales) --
far beyond the tuned kernels' tiles, so the large-L paths (the generic
CTA-per-row / per-band selection, the streaming projection, u64 CSR offsets)
run.  One (b,h) pair each; the oracle checks a SUBSET of query rows / bands
(rows and bands are independent of each other in every rule but the causal
threshold, which is checked in full at a smaller L): levels bit-exact on every
row, masks bit-exact and Z within tolerance on the subset."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops
from test_gpu_parity import TOL, oracle_levels

pytestmark = pytest.mark.gpu


def _run(p):
    q, k, v, P = ops.generate(p, pair0=1, npairs=1)
    dev = torch.device("cuda:0")
    qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, P))
    lv = ops.predict(p, qd, kd, Pd)
    mask = ops.select(p, lv)
    z = ops.sparse_attention(p, qd, kd, vd, mask)
    torch.cuda.synchronize()
    return q, k, v, P, lv, mask, z


def _levels_equal(oracle, p, lv, q, k, P):
    lq, sq = oracle_levels(oracle, p, q[0], P)
    lk, sk = oracle_levels(oracle, p, k[0], P)
    assert np.array_equal(ops.levels_rows(lv.lq)[0].float().cpu().numpy().astype(np.int32), lq)
    assert np.array_equal(ops.levels_rows(lv.lk)[0].float().cpu().numpy().astype(np.int32), lk)
    return lq, lk, sq, sk


def _check_z(oracle, p, q, k, v, z, rows, lists):
    rp = np.zeros(len(rows) + 1, np.uint64)
    rp[1:] = np.cumsum([len(c) for c in lists])
    zr, _ = oracle.sparse_attention(q[0][rows].double().numpy(), k[0].double().numpy(), v[0].double().numpy(),
                                    rp, np.concatenate(lists), True, False)
    zg = z[0][rows].double().cpu().numpy()
    assert np.abs(zg - zr).max() / np.abs(zr).max() <= TOL[p.dtype]


@pytest.mark.parametrize("scope,L,keep", [("tensor", 51200, 64), ("row", 25600, 33)])
def test_row_topk_at_max_L(scope, L, keep, oracle):
    p = load_preset("c1_bert_base").replace(batch=1, heads=1, L=L, keep=keep, quant_scope=scope)
    q, k, v, P, lv, mask, z = _run(p)
    lq, lk, sq, sk = _levels_equal(oracle, p, lv, q, k, P)
    rows = np.unique(np.concatenate([np.arange(0, L, 997), [0, 1, L - 2, L - 1]]))
    # the oracle's row rule (value desc, lowest column first) on the exact integer scores of the
    # subset rows; per-row scope ranks (double) S_int * s_k[j]
    S = (lq[rows].astype(np.int64) @ lk.T.astype(np.int64)).astype(np.float64)
    if scope == "row":
        S = S * np.asarray(sk, np.float64)[None, :]
    want = np.stack([oracle.row_topk(S[i], keep) for i in range(len(rows))])
    got = mask.cols[: L * keep].view(L, keep)[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, want)
    _check_z(oracle, p, q, k, v, z, rows, [want[i] for i in range(len(rows))])


def test_colvec_at_max_L(oracle):
    L, keep = 51200, 100
    p = load_preset("c2_vector").replace(batch=1, heads=1, L=L, keep=keep)
    q, k, v, P, lv, mask, z = _run(p)
    lq, lk, _, _ = _levels_equal(oracle, p, lv, q, k, P)
    nb = L // 8
    bands = np.unique(np.concatenate([np.arange(0, nb, 331), [0, nb - 1]]))
    rows = (bands[:, None] * 8 + np.arange(8)[None, :]).ravel()
    # band score = max over the band's 8 rows of the exact integer scores, then the row rule
    S = (lq[rows].astype(np.int64) @ lk.T.astype(np.int64)).reshape(len(bands), 8, L).max(axis=1).astype(np.float64)
    want = np.stack([oracle.row_topk(S[i], keep) for i in range(len(bands))])
    got = mask.cols[: nb * keep].view(nb, keep)[torch.from_numpy(bands).cuda()].cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, want)
    _check_z(oracle, p, q, k, v, z, rows, [want[i // 8] for i in range(len(rows))])


def test_causal_threshold_large_L(oracle):
    """L = 40000 (2.4x C4's length), causal, cap 60: the whole mask against the oracle."""
    L = 40000
    p = load_preset("c4_threshold").replace(batch=1, heads=1, L=L, cap=60)
    q, k, v, P, lv, mask, z = _run(p)
    lq, lk, sq, sk = _levels_equal(oracle, p, lv, q, k, P)
    c = float(np.atleast_1d(sq)[0]) * float(np.atleast_1d(sk)[0]) / np.sqrt(float(p.d))
    rp, cols, _ = oracle.mask_threshold(lq, lk, c, p.frac_num, p.frac_den, p.cap, True)
    grp = mask.rowptr[: L + 1].cpu().numpy().astype(np.uint64)
    assert np.array_equal(grp, rp)
    assert np.array_equal(mask.cols[: int(rp[-1])].cpu().numpy().astype(np.uint32), cols)
    rows = np.arange(0, L, 1999)
    _check_z(oracle, p, q, k, v, z, rows, [cols[int(rp[i]):int(rp[i + 1])] for i in rows])


@pytest.mark.parametrize("mode,base,over", [
    ("row_topk", "c1_bert_base", {"keep": 5, "quant_scope": "tensor"}),
    ("colvec", "c2_vector", {"keep": 5}),
    ("threshold", "c4_threshold", {"cap": 4}),
])
def test_max_pair_count(mode, base, over, oracle):
    """batch * heads = 32767, the most one call accepts (grid.y / grid.z carry the
    pair index): first, middle and last pairs against the oracle; 32768 is a ShapeError."""
    from paper_2110_11299_b200.errors import ShapeError
    from test_gpu_parity import oracle_mask_rows

    pairs, L = 32767, 24
    p = load_preset(base).replace(batch=pairs, heads=1, L=L, d=16, k=16, **over)
    q, k, v, P = ops.generate(p, pair0=0, npairs=pairs, threads=8)
    dev = torch.device("cuda:0")
    qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, P))
    lv = ops.predict(p, qd, kd, Pd)
    mask = ops.select(p, lv)
    z = ops.sparse_attention(p, qd, kd, vd, mask)
    torch.cuda.synchronize()
    rows_g = ops.mask_rows(p, mask, pairs)
    for pr in (0, 1, 16383, 32765, 32766):
        lq, sq = oracle_levels(oracle, p, q[pr], P)
        lk, sk = oracle_levels(oracle, p, k[pr], P)
        assert np.array_equal(ops.levels_rows(lv.lq)[pr].float().cpu().numpy().astype(np.int32), lq)
        rows = oracle_mask_rows(oracle, p, lq, lk, sq, sk)
        for i in range(L):
            assert np.array_equal(rows_g[pr][i], rows[i]), (pr, i)
        rp, cols = ops.to_csr(rows)
        zr, _ = oracle.sparse_attention(q[pr].double().numpy(), k[pr].double().numpy(), v[pr].double().numpy(),
                                        rp, cols, True, False)
        assert np.abs(z[pr].double().cpu().numpy() - zr).max() / max(np.abs(zr).max(), 1e-30) <= TOL[p.dtype]
    with pytest.raises(ShapeError):
        ops.validate(p.replace(batch=32768))
