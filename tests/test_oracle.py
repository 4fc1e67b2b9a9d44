"""The CPU oracle (oracle/dsa_oracle.c) pinned against the reference's own
known-answer tests and against the reference implementation itself
(oracle/_ref, compiled from /root/reference/proj/src), plus the committed
golden fixtures generated from that reference (oracle/gen_golden.py)."""
from pathlib import Path

import numpy as np
import pytest
import torch

GOLDEN = Path(__file__).resolve().parent / "golden"


# ------------------------------------------------ reference known answers
def test_round_half_away_known_answer(oracle):
    # P/tests/test_kernels.cpp:113-123 (s = 1, qmax = 7)
    xs = [0.5, -0.5, 1.49, -1.49, 100.0, -100.0]
    want = [1, -1, 1, -1, 7, -7]
    got = [max(-7, min(7, oracle.round_half_away(x))) for x in xs]
    assert got == want


def test_quantize_levels_known_answer(oracle):
    x = np.array([[0.5, -0.5, 1.49, -1.49, 7.0, -7.0]])
    lv, s = oracle.quantize_levels(x, 4)  # amax 7 -> s = 1
    assert s == 1.0
    assert lv.tolist() == [[1, -1, 1, -1, 7, -7]]


def test_quantize_all_zero_guard(oracle):
    lv, s = oracle.quantize_levels(np.zeros((3, 4)), 4)  # P/src/predictor.cpp:39
    assert s == 0.0 and not lv.any()


def test_quantize_properties(oracle):
    # P/tests/test_predictor.cpp:90-120: error <= s/2, <= 2^b distinct, endpoints kept
    rng = np.random.default_rng(0)
    x = rng.normal(size=(64, 16))
    for bits in (2, 4, 8):
        lv, s = oracle.quantize_levels(x, bits)
        qmax = (1 << (bits - 1)) - 1
        assert np.abs(lv).max() == qmax
        assert np.abs(lv * s - x).max() <= s / 2 + 1e-12
        assert len(np.unique(lv)) <= 2 ** bits


def test_topk_tie_known_answer(oracle):
    # P/tests/test_linalg.cpp:97-101
    assert oracle.row_topk([0.1, 0.9, 0.5, 0.9], 2).tolist() == [1, 3]
    assert oracle.row_topk([3.0, 1.0, 2.0], 3).tolist() == [0, 1, 2]


def test_topk_sort_oracle(oracle):
    # P/tests/test_linalg.cpp:107-121: stable sort by value desc
    rng = np.random.default_rng(8)
    s = rng.integers(-3, 4, size=(8, 16)).astype(float)  # many ties
    for i in range(8):
        order = sorted(range(16), key=lambda j: (-s[i, j], j))
        assert oracle.row_topk(s[i], 4).tolist() == sorted(order[:4])


def test_topk_keep_out_of_range(oracle):
    with pytest.raises(ValueError):
        oracle.row_topk([1.0, 2.0], 3)


def test_colvec_constant_scores_keep_first_columns(oracle):
    # P/tests/test_maskgen.cpp:89-94: equal band scores -> lowest columns
    lq = np.ones((8, 16), np.int32)
    lk = np.ones((8, 16), np.int32)
    m = oracle.mask_colvec(lq, lk, 4, 4)
    assert m.tolist() == [[0, 1, 2, 3], [0, 1, 2, 3]]


def test_colvec_ragged_band(oracle):
    # P/tests/test_maskgen.cpp:111-116: last band of 10 rows with v = 4 has 2 rows
    rng = np.random.default_rng(4)
    lq = rng.integers(-7, 8, size=(10, 16)).astype(np.int32)
    lk = rng.integers(-7, 8, size=(10, 16)).astype(np.int32)
    m = oracle.mask_colvec(lq, lk, 4, 2)
    assert m.shape == (3, 2)
    S = lq.astype(np.int64) @ lk.T
    pooled = S[8:10].max(axis=0)
    assert m[2].tolist() == sorted(sorted(range(10), key=lambda j: (-pooled[j], j))[:2])


def test_block_forced_diagonal(oracle):
    rng = np.random.default_rng(3)
    lq = rng.integers(-7, 8, size=(64, 16)).astype(np.int32)
    lk = rng.integers(-7, 8, size=(64, 16)).astype(np.int32)
    m = oracle.mask_block(lq, lk, 8, 3, True)
    S = lq.astype(np.int64) @ lk.T
    B = S.reshape(8, 8, 8, 8).sum(axis=(1, 3))
    for ib in range(8):
        others = sorted((j for j in range(8) if j != ib), key=lambda j: (-B[ib, j], j))[:2]
        assert m[ib].tolist() == sorted([ib] + others)


def test_exp_deterministic_matches_libm(oracle):
    for x in np.linspace(-40, 0, 257):
        assert abs(oracle.exp(x) - np.exp(x)) <= 4e-16 * np.exp(x)


def test_threshold_empty_row_and_cap(oracle):
    # uniform scores: p = 1/L < theta = 20/L -> every row empty (cf. test_maskgen.cpp:65-69)
    lq = np.zeros((40, 16), np.int32)
    lk = np.zeros((40, 16), np.int32)
    rp, cols, empty = oracle.mask_threshold(lq, lk, 0.1, 1, 20, 40, False)
    assert empty == 40 and rp[-1] == 0
    # one dominant key per row: kept, cap respected
    lq = np.ones((40, 16), np.int32)
    lk = np.zeros((40, 16), np.int32)
    lk[5] = 7
    rp, cols, empty = oracle.mask_threshold(lq, lk, 0.5, 1, 20, 1, False)
    assert empty == 0 and all(cols == 5)


def test_sparse_attention_semantics(oracle):
    rng = np.random.default_rng(2)
    L, d = 12, 8
    q, k, v = rng.uniform(-1, 1, (3, L, d))
    # single kept entry -> weight one -> z = V row (P/tests/test_sparse.cpp:70-73)
    rp = np.arange(L + 1, dtype=np.uint64)
    cols = np.arange(L, dtype=np.uint32)
    z, er = oracle.sparse_attention(q, k, v, rp, cols)
    assert np.abs(z - v).max() <= 1e-12 and not er.any()
    # empty row -> zero output, flagged (P/tests/test_sparse.cpp:89-97)
    rp2 = rp.copy()
    rp2[4:] -= 1
    cols2 = np.delete(cols, 3)
    z, er = oracle.sparse_attention(q, k, v, rp2, cols2)
    assert er[3] == 1 and not z[3].any()
    # sparse == masked dense Eq. 4 (P/tests/test_sparse.cpp:130-153)
    keep = 5
    cols3 = np.concatenate([np.sort(rng.choice(L, keep, replace=False)) for _ in range(L)]).astype(np.uint32)
    rp3 = np.arange(0, L * keep + 1, keep, dtype=np.uint64)
    zs, _ = oracle.sparse_attention(q, k, v, rp3, cols3)
    zd = oracle.masked_dense_attention(q, k, v, rp3, cols3)
    assert np.abs(zs - zd).max() <= 1e-4


# ------------------------------------------------ oracle == the reference
def test_oracle_equals_reference_projection_and_levels(oracle, reference):
    rng = np.random.default_rng(11)
    for f32, bits in ((True, 4), (False, 4), (False, 8), (False, 2)):
        x = rng.normal(size=(96, 64))
        if f32:
            x = x.astype(np.float32).astype(np.float64)
        p = rng.normal(scale=0.25, size=(64, 16)).astype(np.float32).astype(np.float64)
        xo, xr = oracle.project(x, p, f32), reference.project(x, p, f32)
        assert np.array_equal(xo, xr)
        lo, so = oracle.quantize_levels(xo, bits)
        lr, sr = reference.quantize_levels(xr, bits, f32)
        assert so == sr and np.array_equal(lo, lr)


def test_oracle_equals_reference_masks(oracle, reference):
    rng = np.random.default_rng(12)
    for L, k in ((64, 16), (129, 32)):
        lq = rng.integers(-7, 8, size=(L, k)).astype(np.int32)
        lk = rng.integers(-7, 8, size=(L, k)).astype(np.int32)
        S = oracle.scores_int(lq, lk).astype(np.float64)
        for keep in (1, 7, L):
            assert np.array_equal(oracle.mask_topk(lq, lk, keep), reference.topk_mask(S, keep))
        for v in (1, 4, 8):
            assert np.array_equal(oracle.mask_colvec(lq, lk, v, 9), reference.colvec_maxpool_mask(S, v, 9))


def test_rowscaled_topk_matches_reference(oracle, reference):
    rng = np.random.default_rng(13)
    L, k = 80, 16
    lq = rng.integers(-7, 8, size=(L, k)).astype(np.int32)
    lk = rng.integers(-7, 8, size=(L, k)).astype(np.int32)
    sk = rng.uniform(0.1, 2.0, size=L)
    S = (lq.astype(np.int64) @ lk.T).astype(np.float64) * sk[None, :]
    assert np.array_equal(oracle.mask_topk(lq, lk, 9, sk=sk), reference.topk_mask(S, 9))


def test_threshold_rule_matches_reference_softmax_threshold(oracle, reference):
    # The fixed-point rule (O6) agrees with the reference's threshold_mask on
    # row_softmax(c * S) (P/src/maskgen.cpp:22-31) except within ~1e-12 of theta.
    rng = np.random.default_rng(14)
    L, k = 200, 16
    lq = rng.integers(-7, 8, size=(L, k)).astype(np.int32)
    lk = rng.integers(-7, 8, size=(L, k)).astype(np.int32)
    c = 0.05
    rp, cols, _ = oracle.mask_threshold(lq, lk, c, 1, 20, L, False)
    S = (lq.astype(np.int64) @ lk.T).astype(np.float64) * c
    rpr, colsr = reference.threshold_mask(S, 20.0 / L, True)
    assert np.array_equal(rp, rpr) and np.array_equal(cols, colsr)


def test_attention_matches_reference_bit_exact(oracle, reference):
    rng = np.random.default_rng(15)
    L, d, keep = 50, 16, 7
    q, k, v = rng.normal(size=(3, L, d))
    cols = np.concatenate([np.sort(rng.choice(L, keep, replace=False)) for _ in range(L)]).astype(np.uint32)
    rp = np.arange(0, L * keep + 1, keep, dtype=np.uint64)
    for f32 in (False, True):
        if f32:  # f32 Matrices hold float-rounded values (P/include/dsattn/matrix.hpp:71-74)
            q, k, v = (a.astype(np.float32).astype(np.float64) for a in (q, k, v))
        zo, eo = oracle.sparse_attention(q, k, v, rp, cols, True, f32)
        zr, er, cnt = reference.sparse_attention(q, k, v, rp, cols, True, f32)
        assert np.array_equal(zo, zr) and np.array_equal(eo, er)
        assert cnt.tolist() == [L * keep * d, L * keep * d, L * keep]  # OpCounters exact


# ------------------- O5 / O6 pinned to compositions of reference primitives
def _pair_levels(oracle, name, pair, **over):
    from paper_2110_11299_b200 import load_preset, ops
    p = load_preset(name).replace(**over)
    sub = p.replace(batch=1, heads=1)
    q, k, _, P = ops.generate(sub, pair0=pair, npairs=1)
    Pn = P.double().numpy()
    lq, sq = oracle.levels(q[0].double().numpy(), Pn, p.bits)
    lk, sk = oracle.levels(k[0].double().numpy(), Pn, p.bits)
    return p, lq, lk, sq, sk


def test_block_rule_matches_reference_composition(oracle, reference):
    # C3 shape (L 8192, d 128, k 32, INT8, 32x32 blocks, keep 16 incl. the
    # forced diagonal) at full L, plus ragged / unforced variants
    cases = [("c3_block", 5, {}), ("c3_block", 63, {"L": 1000, "keep": 5}),
             ("c3_block", 1, {"L": 512, "force_diag": False, "block": 16, "keep": 7})]
    for name, pair, over in cases:
        p, lq, lk, _, _ = _pair_levels(oracle, name, pair, **over)
        got = oracle.mask_block(lq, lk, p.block, p.keep, p.force_diag)
        want = reference.block_mask(lq, lk, p.block, p.keep, p.force_diag)
        assert np.array_equal(got, want), (name, over)


def _threshold_agrees(oracle, reference, p, lq, lk, sq, sk):
    """Oracle O6 (2^-40 fixed-point softmax, exact integer compare) against
    the reference composition row_softmax -> ">= theta" -> row_topk_indices
    cap.  Returns (#rows compared, #rows that differ); every differing key
    must sit at theta to within 1e-9 relative (the two evaluations of
    p~ differ only by rounding)."""
    c = sq * sk / np.sqrt(float(p.d))
    theta = p.frac_den / (p.frac_num * p.L)
    rp, cols, _ = oracle.mask_threshold(lq, lk, c, p.frac_num, p.frac_den, p.cap, p.causal)
    rpr, colsr = reference.causal_threshold_mask(lq, lk, c, theta, p.cap, p.causal)
    bad = 0
    for i in np.nonzero((np.diff(rp.astype(np.int64)) != np.diff(rpr.astype(np.int64))))[0].tolist() + [
            i for i in range(p.L) if rp[i + 1] - rp[i] == rpr[i + 1] - rpr[i]
            and not np.array_equal(cols[rp[i]:rp[i + 1]], colsr[rpr[i]:rpr[i + 1]])]:
        bad += 1
        a, b = set(cols[rp[i]:rp[i + 1]].tolist()), set(colsr[rpr[i]:rpr[i + 1]].tolist())
        probs = reference.threshold_row_probs(lq, lk, c, i, p.causal)
        for j in a ^ b:
            assert abs(probs[j] - theta) <= 1e-9 * theta, (i, j, probs[j], theta)
    return p.L, bad


def test_causal_threshold_matches_reference_composition(oracle, reference):
    # C4 shape at full L = 16384 (causal, theta = 1/(0.05 L), cap 1311) on
    # two seeded pairs, plus a binding cap and a non-causal row softmax
    from concurrent.futures import ThreadPoolExecutor
    cases = [("c4_threshold", 0, {}), ("c4_threshold", 511, {}),
             ("c4_threshold", 3, {"L": 2048, "cap": 7}),
             ("c4_threshold", 4, {"L": 1500, "causal": False, "cap": 1500})]

    def one(case):
        name, pair, over = case
        p, lq, lk, sq, sk = _pair_levels(oracle, name, pair, **over)
        return _threshold_agrees(oracle, reference, p, lq, lk, sq, sk)

    with ThreadPoolExecutor(4) as ex:
        res = list(ex.map(one, cases))
    for (rows, bad), case in zip(res, cases):
        assert bad <= rows // 1000, (case, bad)  # and every difference sits at theta


def test_generator_matches_reference_rng():
    # dsa_generate (the repo's host generator) == the same procedure drawn
    # with the reference Rng (P/include/dsattn/rng.hpp:14-78), bit for bit
    from oracle.oracle import REF_SO, REF_SRC, Reference
    if not REF_SO.exists() and not REF_SRC.exists():
        pytest.skip("reference library absent")
    from paper_2110_11299_b200 import load_preset, ops
    ref = Reference()
    for name in ("c0_smoke", "c1_bert_base", "c3_block", "c4_threshold"):
        p = load_preset(name).replace(L=192)
        q, k, v, P = ops.generate(p, pair0=5, npairs=2)
        rq, rk, rv, rP = ref.generate(p.L, p.d, p.k, p.dtype == "bf16", p.seed, p.planted_per_mille,
                                      p.band_width, 5, 2)
        for a, b in ((q, rq), (k, rk), (v, rv), (P, rP)):
            assert np.array_equal(a.double().numpy(), b), name


# ------------------------------------------------------- golden fixtures
def _golden_inputs(g):
    q, k, v = g["q"], g["k"], g["v"]
    if q.dtype == np.int16:  # bf16 bits
        def f(a):
            return torch.from_numpy(a.copy()).view(torch.bfloat16).double().numpy()
        return f(q), f(k), f(v)
    return q.astype(np.float64), k.astype(np.float64), v.astype(np.float64)


@pytest.mark.parametrize("name", sorted(p.stem for p in GOLDEN.glob("*.npz")))
def test_golden_fixture(name, oracle):
    g = np.load(GOLDEN / f"{name}.npz")
    L, d, kd, bits, keep, vec_v, f32 = (int(x) for x in g["meta"])
    q, k, v = _golden_inputs(g)
    P = g["P"].astype(np.float64)
    lq, sq = oracle.levels(q, P, bits, round_f32=bool(f32))
    lk, sk = oracle.levels(k, P, bits, round_f32=bool(f32))
    assert np.array_equal(lq, g["lq"]) and np.array_equal(lk, g["lk"])
    assert sq == float(g["sq"]) and sk == float(g["sk"])
    mode = str(g["mode"])
    if mode == "row_topk":
        m = oracle.mask_topk(lq, lk, keep)
        rows = [m[i] for i in range(L)]
    elif mode == "colvec":
        m = oracle.mask_colvec(lq, lk, vec_v, keep)
        rows = [m[i // vec_v] for i in range(L)]
    elif mode == "block":
        bs, fd = (int(x) for x in g["block"])
        m = oracle.mask_block(lq, lk, bs, keep, bool(fd))
        rows = [np.concatenate([np.arange(b * bs, min((b + 1) * bs, L)) for b in m[i // bs]]) for i in range(L)]
    else:
        num, den, cap, causal = (int(x) for x in g["threshold"])
        rp_, cols_, _ = oracle.mask_threshold(lq, lk, sq * sk / np.sqrt(float(d)), num, den, cap, bool(causal))
        m = np.concatenate([rp_.astype(np.int64), cols_.astype(np.int64)])
        rows = [cols_[rp_[i]:rp_[i + 1]] for i in range(L)]
    assert np.array_equal(m, g["mask"])
    rp = np.zeros(L + 1, np.uint64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    z, er = oracle.sparse_attention(q, k, v, rp, np.concatenate(rows), True, bool(f32))
    assert np.array_equal(z, g["z"])
    if "empty_rows" in g:
        assert np.array_equal(er, g["empty_rows"])
