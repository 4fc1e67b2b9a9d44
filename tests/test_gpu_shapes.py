"""GPU parity on ragged / edge shapes (the reference tests odd lengths and
ragged bands: P/tests/test_maskgen.cpp:111-116, acceptance l in [8,64]).

Each case regenerates seeded inputs, runs predict -> select -> attention
through the C-ABI and compares levels and masks bit-exactly, Z within the
dtype tolerance, against the oracle."""
import numpy as np
import pytest

from paper_2110_11299_b200 import load_preset
from test_gpu_parity import TOL, oracle_levels, oracle_mask_rows, run_gpu
from paper_2110_11299_b200 import ops

pytestmark = pytest.mark.gpu

BASE = {"row_topk": "c0_smoke", "colvec": "c2_vector", "block": "c3_block",
        "threshold": "c4_threshold"}

CASES = [
    # mode, L, d, k, bits, dtype, scope, extra
    ("row_topk", 100, 64, 16, 4, "bf16", "tensor", {"keep": 7}),
    ("row_topk", 333, 128, 32, 8, "f32", "tensor", {"keep": 333}),
    ("row_topk", 257, 32, 16, 2, "bf16", "row", {"keep": 1}),
    ("colvec", 1004, 64, 16, 4, "bf16", "tensor", {"keep": 51, "vec_v": 8}),
    ("colvec", 130, 128, 32, 4, "bf16", "tensor", {"keep": 130, "vec_v": 8}),
    ("colvec", 515, 64, 16, 8, "bf16", "tensor", {"keep": 20, "vec_v": 8}),
    ("colvec", 1000, 64, 32, 4, "bf16", "tensor", {"keep": 999, "vec_v": 8}),
    ("colvec", 640, 64, 16, 2, "bf16", "tensor", {"keep": 300, "vec_v": 8}),
    ("colvec", 300, 64, 16, 4, "f32", "tensor", {"keep": 17, "vec_v": 5}),
    ("block", 1000, 64, 16, 4, "bf16", "tensor", {"keep": 5, "block": 32, "force_diag": True}),
    ("block", 1024, 64, 16, 4, "bf16", "tensor", {"keep": 5, "block": 32, "force_diag": True}),
    ("block", 96, 128, 32, 4, "bf16", "tensor", {"keep": 3, "block": 32, "force_diag": False}),
    ("block", 333, 128, 32, 8, "bf16", "tensor", {"keep": 3, "block": 16, "force_diag": False}),
    ("block", 1024, 128, 32, 8, "bf16", "tensor", {"keep": 7, "block": 32, "force_diag": False}),
    ("block", 512, 64, 16, 4, "bf16", "tensor", {"keep": 16, "block": 16, "force_diag": True}),
    # last block ONE key wide (cross-multiplied means = the plain sums: adjacent
    # integers must not share a rank key -- found by test_gpu_sweep)
    ("block", 513, 32, 16, 4, "f32", "tensor", {"keep": 13, "block": 16, "force_diag": True}),
    ("block", 1025, 64, 16, 4, "bf16", "tensor", {"keep": 9, "block": 32, "force_diag": True}),
    ("row_topk", 512, 64, 16, 8, "bf16", "row", {"keep": 40}),
    ("row_topk", 640, 128, 32, 4, "bf16", "row", {"keep": 3}),
    ("row_topk", 1024, 64, 16, 4, "bf16", "tensor", {"keep": 64}),
    # per-row scales on the warp-per-row window select (L = 32 * NPL): every
    # group count G, k = 32, 2-bit levels (tied keys -> candidate sets /
    # overflow rows), keep 1 and keep = 32 G exactly
    ("row_topk", 2048, 64, 16, 2, "bf16", "row", {"keep": 102}),
    ("row_topk", 1024, 128, 32, 4, "bf16", "row", {"keep": 256}),
    ("row_topk", 2048, 64, 32, 8, "bf16", "row", {"keep": 1}),
    ("row_topk", 512, 64, 16, 4, "f32", "row", {"keep": 33}),
    ("row_topk", 1024, 64, 16, 4, "bf16", "row", {"keep": 64}),
    # per-row scales off the warp-per-row kernel's L grid: ragged L, k = 32,
    # 8-bit / 2-bit levels (tied keys), keep near L/2, L = 4096
    ("row_topk", 300, 64, 16, 4, "bf16", "row", {"keep": 30}),
    ("row_topk", 1000, 64, 32, 4, "bf16", "row", {"keep": 100}),
    ("row_topk", 513, 128, 16, 8, "bf16", "row", {"keep": 250}),
    ("row_topk", 2048, 64, 16, 4, "bf16", "row", {"keep": 200}),
    ("row_topk", 777, 64, 16, 2, "bf16", "row", {"keep": 97}),
    ("row_topk", 4096, 64, 16, 4, "bf16", "row", {"keep": 64}),
    ("row_topk", 65, 64, 16, 4, "bf16", "row", {"keep": 8}),
    ("threshold", 700, 64, 16, 4, "bf16", "tensor", {"cap": 5, "causal": True}),
    # theta = 400 / L: most rows keep one key or none (empty-row flags)
    ("threshold", 700, 64, 16, 4, "bf16", "tensor", {"cap": 50, "causal": True, "frac_num": 1, "frac_den": 400}),
    ("threshold", 640, 128, 32, 4, "bf16", "tensor", {"cap": 64, "causal": False}),
    ("threshold", 513, 64, 32, 4, "f32", "tensor", {"cap": 513, "causal": False}),
    # 8-bit levels: small exp scale c, so the cut lies beyond the 128-bin
    # histogram of the tensor-core threshold kernel (counting-pass path)
    ("threshold", 600, 64, 16, 8, "bf16", "tensor", {"cap": 600, "causal": False}),
    ("threshold", 1000, 64, 16, 8, "bf16", "tensor", {"cap": 9, "causal": True}),
    ("threshold", 384, 64, 16, 2, "bf16", "tensor", {"cap": 2, "causal": True}),
]


def check_shape(mode, L, d, k, bits, dtype, scope, extra, oracle):
    p = load_preset(BASE[mode]).replace(L=L, d=d, k=k, bits=bits, dtype=dtype, quant_scope=scope,
                                        round_proj_f32=(dtype == "f32"), seed=1234 + L, **extra)
    npairs = 2
    sub, (q, k_, v, P), lv, mask, z = run_gpu(p, npairs)
    rows_g = ops.mask_rows(sub, mask, npairs)
    worst = 0.0
    for pr in range(npairs):
        lq, sq = oracle_levels(oracle, sub, q[pr], P)
        lk, sk = oracle_levels(oracle, sub, k_[pr], P)
        assert np.array_equal(ops.levels_rows(lv.lq)[pr].float().cpu().numpy().astype(np.int32), lq)
        assert np.array_equal(ops.levels_rows(lv.lk)[pr].float().cpu().numpy().astype(np.int32), lk)
        rows = oracle_mask_rows(oracle, sub, lq, lk, sq, sk)
        bad = [i for i in range(L) if not np.array_equal(rows_g[pr][i], rows[i])]
        assert not bad, f"{len(bad)} rows differ, first {bad[:4]}"
        rp, cols = ops.to_csr(rows)
        zr, er = oracle.sparse_attention(q[pr].double().numpy(), k_[pr].double().numpy(),
                                         v[pr].double().numpy(), rp, cols, True, dtype == "f32")
        zg = z[pr].double().cpu().numpy()
        if mask.empty_rows is not None:
            ge = mask.empty_rows[pr * L:(pr + 1) * L].cpu().numpy()
            assert np.array_equal(ge.astype(bool), er.astype(bool)), "empty-row flags differ"
        worst = max(worst, np.abs(zg - zr).max() / max(np.abs(zr).max(), 1e-30))
    assert worst <= TOL[dtype], worst


@pytest.mark.parametrize("mode,L,d,k,bits,dtype,scope,extra", CASES)
def test_shape(mode, L, d, k, bits, dtype, scope, extra, oracle):
    check_shape(mode, L, d, k, bits, dtype, scope, extra, oracle)
