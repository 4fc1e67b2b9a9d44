"""Adversarial inputs at the shapes that select the tuned kernels (the
tensor-core projection / colvec / threshold / block / per-row top-k kernels):
massive exact ties (duplicated keys, constant queries), an all-zero K, one
huge outlier (every other level quantises to 0), sign-flipped copies, inputs
that are exactly representable integers.  Levels, scales and masks bit-exact
against the oracle, Z within tolerance, empty-row flags equal -- the tie rule
(value desc, LOWEST column first) is what these stress."""
import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops
from test_gpu_parity import TOL, oracle_levels, oracle_mask_rows

pytestmark = pytest.mark.gpu

SHAPES = {
    # name: (base preset, overrides)  -- L a multiple of the kernels' tiles AND ragged
    "c1": ("c1_bert_base", {"L": 1024, "keep": 51}),
    "c1r": ("c1_bert_base", {"L": 2048, "keep": 102}),
    "c2": ("c2_vector", {"L": 1024, "keep": 51}),
    "c2r": ("c2_vector", {"L": 1160, "keep": 58}),
    "c3": ("c3_block", {"L": 1024, "keep": 4}),
    "c4": ("c4_threshold", {"L": 1024, "cap": 82}),
    "c4r": ("c4_threshold", {"L": 900, "cap": 72}),
}


def _bf16(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16)


def _mutate(kind, q, k, v):
    """q, k, v: [pairs, L, d] bf16 tensors from the seeded generator."""
    L = q.shape[1]
    if kind == "dup_keys":            # 7 distinct keys: every score ties L/7 ways
        k = k[:, torch.arange(L) % 7, :].contiguous()
    elif kind == "const_queries":     # every query equal: every band / row sees the same ranking
        q = q[:, :1, :].expand_as(q).contiguous()
    elif kind == "zero_k":            # all-zero K: scale guard, all scores 0, ties everywhere
        k = torch.zeros_like(k)
    elif kind == "outlier":           # one huge entry: all other levels quantise to 0
        k = k.clone()
        k[:, L // 3, 5] = 3.0e4
        q = q.clone()
        q[:, L // 2, 9] = -2.0e4
    elif kind == "neg_copy":          # k_j and -k_j pairs: symmetric scores around 0
        k = k.clone()
        k[:, 1::2, :] = -k[:, 0::2, :][:, : k[:, 1::2, :].shape[1], :]
    elif kind == "small_ints":        # integer-valued inputs in [-3, 3]
        q = _bf16(torch.round(q.float() * 1.5).clamp(-3, 3))
        k = _bf16(torch.round(k.float() * 1.5).clamp(-3, 3))
    else:
        raise ValueError(kind)
    return q, k, v


@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("kind", ["dup_keys", "const_queries", "zero_k", "outlier", "neg_copy", "small_ints"])
def test_adversarial(shape, kind, oracle):
    base, over = SHAPES[shape]
    p = load_preset(base).replace(batch=2, heads=1, **over)
    npairs = 2
    q, k, v, P = ops.generate(p, pair0=3, npairs=npairs)
    q, k, v = _mutate(kind, q, k, v)
    dev = torch.device("cuda:0")
    qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, P))
    lv = ops.predict(p, qd, kd, Pd)
    mask = ops.select(p, lv)
    z = ops.sparse_attention(p, qd, kd, vd, mask)
    torch.cuda.synchronize()
    rows_g = ops.mask_rows(p, mask, npairs)
    L = p.L
    worst = 0.0
    for pr in range(npairs):
        lq, sq = oracle_levels(oracle, p, q[pr], P)
        lk, sk = oracle_levels(oracle, p, k[pr], P)
        assert np.array_equal(ops.levels_rows(lv.lq)[pr].float().cpu().numpy().astype(np.int32), lq)
        assert np.array_equal(ops.levels_rows(lv.lk)[pr].float().cpu().numpy().astype(np.int32), lk)
        rows = oracle_mask_rows(oracle, p, lq, lk, sq, sk)
        bad = [i for i in range(L) if not np.array_equal(rows_g[pr][i], rows[i])]
        assert not bad, f"{len(bad)} rows differ, first {bad[:4]}"
        rp, cols = ops.to_csr(rows)
        zr, er = oracle.sparse_attention(q[pr].double().numpy(), k[pr].double().numpy(), v[pr].double().numpy(),
                                         rp, cols, True, False)
        if mask.empty_rows is not None:
            ge = mask.empty_rows[pr * L:(pr + 1) * L].cpu().numpy()
            assert np.array_equal(ge.astype(bool), er.astype(bool)), "empty-row flags differ"
        worst = max(worst, np.abs(z[pr].double().cpu().numpy() - zr).max() / max(np.abs(zr).max(), 1e-30))
    assert worst <= TOL[p.dtype], worst
