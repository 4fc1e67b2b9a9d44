"""GPU properties at the BASELINE configs' FULL sizes (all (b,h) pairs, full
L), where the oracle cannot check every pair: size-independent invariants of
the path, plus exact oracle spot checks of a few seeded pairs.

* levels within [-qmax, qmax], scales positive;
* masks: every row list strictly ascending and in range, the exact per-row
  counts of the mode (keep; keep blocks incl. the forced diagonal; threshold:
  <= min(cap, L*num/den), causal j <= i), empty-row flags == zero counts;
* Z finite, every row a convex combination of the kept V rows
  (|z| <= max |V| of the pair), empty rows exactly zero;
* idempotence: a second run gives bit-identical levels, masks and Z;
* spot checks: the masks of two seeded pairs equal the oracle's bit for bit.
"""
import math

import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import load_preset, ops

from test_gpu_parity import oracle_levels, oracle_mask_rows

pytestmark = pytest.mark.gpu

CONFIGS = ["c1_bert_base", "c2_vector", "c3_block", "c4_threshold"]


def _run(p):
    q, k, v, P = ops.generate(p, pinned=True)
    dev = torch.device("cuda:0")
    qd, kd, vd, Pd = (t.to(dev) for t in (q, k, v, P))
    lv = ops.predict(p, qd, kd, Pd)
    mask = ops.select(p, lv)
    z = ops.sparse_attention(p, qd, kd, vd, mask)
    torch.cuda.synchronize()
    return (q, k, v, P), (qd, kd, vd), lv, mask, z


def _row_counts_and_bounds(p, mask, pairs):
    """Per query row: (start, count) into mask.cols (int64 tensors on GPU)."""
    L = p.L
    dev = mask.cols.device
    rows = pairs * L
    if p.mask_mode == "threshold":
        rp = mask.rowptr[: rows + 1]
        return rp[:-1], rp[1:] - rp[:-1]
    if p.mask_mode == "row_topk":
        start = torch.arange(rows, device=dev, dtype=torch.int64) * p.keep
        return start, torch.full((rows,), p.keep, device=dev, dtype=torch.int64)
    group = p.vec_v if p.mask_mode == "colvec" else p.block
    ng = (L + group - 1) // group
    r = torch.arange(rows, device=dev, dtype=torch.int64)
    start = ((r // L) * ng + (r % L) // group) * p.keep
    return start, torch.full((rows,), p.keep, device=dev, dtype=torch.int64)


@pytest.mark.parametrize("name", CONFIGS)
def test_full_size_properties(name, oracle):
    p = load_preset(name)
    pairs, L = p.pairs, p.L
    (q, k, v, P), (qd, kd, vd), lv, mask, z = _run(p)
    qmax = (1 << (p.bits - 1)) - 1

    # levels and scales
    for t in (lv.lq, lv.lk):
        a = t.float().abs().max().item()
        assert a <= qmax and a == int(a)
    assert bool((lv.sq > 0).all()) and bool((lv.sk > 0).all())

    # masks: per-list structure over the whole mask (vectorised on the GPU)
    cols = mask.cols.to(torch.int64)
    start, cnt = _row_counts_and_bounds(p, mask, pairs)
    if p.mask_mode == "threshold":
        nnz = int(mask.rowptr[pairs * L].item())
        bound = min(p.cap, (L * p.frac_num) // p.frac_den)
        assert int(cnt.max().item()) <= bound
        c = cols[:nnz]
        # strictly ascending inside each row: a non-increase only at row starts
        is_start = torch.zeros(nnz + 1, dtype=torch.bool, device=c.device)
        is_start[start[cnt > 0]] = True
        bad = torch.nonzero(c[1:] <= c[:-1]).flatten() + 1
        assert bool(is_start[bad].all())
        # causal: j <= i (checked pair by pair to bound memory)
        for pr in range(pairs):
            rp = mask.rowptr[pr * L: (pr + 1) * L + 1]
            n = rp[1:] - rp[:-1]
            rid = torch.repeat_interleave(torch.arange(L, device=cols.device), n)
            cc = cols[rp[0]: rp[-1]]
            assert bool((cc < L).all())
            if p.causal:
                assert bool((cc <= rid).all())
        assert mask.empty_rows is not None
        assert torch.equal(mask.empty_rows[: pairs * L].bool(), cnt == 0)
    else:
        # structured lists: [groups][keep], ascending, in range
        width = L if p.mask_mode != "block" else (L + p.block - 1) // p.block
        lists = cols[: mask_list_count(p, pairs) * p.keep].view(-1, p.keep)
        assert bool((lists >= 0).all()) and bool((lists < width).all())
        if p.keep > 1:
            assert bool((lists[:, 1:] > lists[:, :-1]).all())
        if p.mask_mode == "block" and p.force_diag:
            nb = width
            diag = torch.arange(lists.shape[0], device=lists.device) % nb
            assert bool((lists == diag[:, None]).any(dim=1).all())

    # Z: finite, convex combination of V rows (|z| <= max |V| of the pair)
    assert bool(torch.isfinite(z.float()).all())
    vmax = vd.float().abs().amax(dim=(1, 2))
    zmax = z.float().abs().amax(dim=(1, 2))
    assert bool((zmax <= vmax * (1 + 1e-2) + 1e-6).all())
    if p.mask_mode == "threshold" and bool((cnt == 0).any()):
        zr = z.view(pairs * L, -1)
        assert bool((zr[cnt == 0] == 0).all())

    # idempotence: bit-identical second run
    lv2 = ops.predict(p, qd, kd, P.to(qd.device))
    mask2 = ops.select(p, lv2)
    z2 = ops.sparse_attention(p, qd, kd, vd, mask2)
    torch.cuda.synchronize()
    assert torch.equal(lv2.lq, lv.lq) and torch.equal(lv2.lk, lv.lk)
    n = int(mask.rowptr[pairs * L].item()) if p.mask_mode == "threshold" else mask_list_count(p, pairs) * p.keep
    assert torch.equal(mask2.cols[:n], mask.cols[:n])
    assert torch.equal(z2, z)

    # exact oracle spot checks on two seeded pairs (first and last)
    for pr in (0, pairs - 1):
        sub = p.replace(batch=1, heads=1)
        lq, sq = oracle_levels(oracle, sub, q[pr], P)
        lk_, sk = oracle_levels(oracle, sub, k[pr], P)
        assert np.array_equal(ops.levels_rows(lv.lq[pr:pr + 1])[0].float().cpu().numpy().astype(np.int32), lq)
        want = oracle_mask_rows(oracle, sub, lq, lk_, sq, sk)
        got = pair_rows(p, mask, pr)
        bad = [i for i in range(L) if not np.array_equal(got[i], want[i])]
        assert not bad, f"{name} pair {pr}: {len(bad)} rows differ"


def mask_list_count(p, pairs):
    if p.mask_mode == "row_topk":
        return pairs * p.L
    group = p.vec_v if p.mask_mode == "colvec" else p.block
    return pairs * math.ceil(p.L / group)


def pair_rows(p, mask, pr):
    """The kept columns of every query row of pair `pr` (host)."""
    L = p.L
    if p.mask_mode == "threshold":
        rp = mask.rowptr[pr * L: (pr + 1) * L + 1].cpu().numpy()
        cols = mask.cols[int(rp[0]): int(rp[-1])].cpu().numpy().astype(np.int64)
        return [cols[rp[i] - rp[0]: rp[i + 1] - rp[0]] for i in range(L)]
    if p.mask_mode == "row_topk":
        c = mask.cols[pr * L * p.keep: (pr + 1) * L * p.keep].cpu().numpy().astype(np.int64).reshape(L, p.keep)
        return [c[i] for i in range(L)]
    group = p.vec_v if p.mask_mode == "colvec" else p.block
    ng = math.ceil(L / group)
    c = mask.cols[pr * ng * p.keep: (pr + 1) * ng * p.keep].cpu().numpy().astype(np.int64).reshape(ng, p.keep)
    if p.mask_mode == "colvec":
        return [c[i // group] for i in range(L)]
    return [np.concatenate([np.arange(b * group, min((b + 1) * group, L)) for b in c[i // group]]) for i in range(L)]
