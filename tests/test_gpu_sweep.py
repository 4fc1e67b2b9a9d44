"""Seeded random sweep over the configuration space of the C ABI: mode x L x d
x k x bits x dtype x scope x keep / cap / block / vector height drawn from a
fixed generator (so failures reproduce), each case checked like
test_gpu_shapes (levels, scales and masks bit-exact, Z within tolerance,
empty-row flags) against the oracle.  Complements the hand-picked shapes: odd
L around every tile boundary, keep from 1 to L, every d / k / bits pairing."""
import os

import numpy as np
import pytest

from test_gpu_shapes import check_shape

pytestmark = pytest.mark.gpu


def _cases(n=72, seed=20211021):
    rng = np.random.default_rng(seed)
    edges = [1, 7, 8, 9, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 511, 512, 513, 1023, 1025]
    out = []
    for i in range(n):
        mode = ["row_topk", "colvec", "block", "threshold"][i % 4]
        d = int(rng.choice([16, 32, 64, 128]))
        k = 16 if d == 16 else int(rng.choice([16, 32]))
        bits = int(rng.choice([2, 4, 8]))
        dtype = "f32" if rng.random() < 0.25 else "bf16"
        L = int(rng.choice(edges[6:])) if rng.random() < 0.5 else int(rng.integers(40, 1400 if i % 3 else 4200))
        scope = "tensor"
        extra = {}
        if mode == "row_topk":
            scope = "row" if rng.random() < 0.5 else "tensor"
            extra["keep"] = int(rng.choice([1, L, max(1, L // 2), int(rng.integers(1, L + 1))]))
        elif mode == "colvec":
            extra["vec_v"] = 8 if rng.random() < 0.7 else int(rng.integers(1, 17))
            extra["keep"] = int(rng.choice([1, L, int(rng.integers(1, L + 1))]))
        elif mode == "block":
            blk = int(rng.choice([8, 16, 32, 64, int(rng.integers(3, 41))]))
            nb = -(-L // blk)
            extra["block"] = blk
            extra["keep"] = int(rng.integers(1, nb + 1))
            extra["force_diag"] = bool(rng.random() < 0.5)
        else:
            extra["causal"] = bool(rng.random() < 0.6)
            extra["cap"] = int(rng.choice([1, L, int(rng.integers(1, L + 1))]))
            extra["frac_num"] = int(rng.choice([1, 1, 2, 3]))
            extra["frac_den"] = int(rng.choice([20, 5, 100]))
        out.append((mode, L, d, k, bits, dtype, scope, extra))
    return out


# DSA_SWEEP_N / DSA_SWEEP_SEED: a longer one-off hunt (the committed default is what the suite runs)
@pytest.mark.parametrize("mode,L,d,k,bits,dtype,scope,extra",
                         _cases(int(os.environ.get("DSA_SWEEP_N", "72")), int(os.environ.get("DSA_SWEEP_SEED", "20211021"))),
                         ids=lambda v: str(v) if not isinstance(v, dict) else "-".join(f"{a}{b}" for a, b in v.items()))
def test_random_config(mode, L, d, k, bits, dtype, scope, extra, oracle):
    check_shape(mode, L, d, k, bits, dtype, scope, extra, oracle)
