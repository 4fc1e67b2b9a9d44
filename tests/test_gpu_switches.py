"""The library's kernel-selection switches (read once at load, kernels.h
`Options`) each force a simpler kernel: the result must not change.  Every
switch runs in a fresh process against a default-path run of the same
seeded inputs:

* levels, scales and masks: bit-identical;
* Z: within the dtype tolerance (bit-identical for the
  chunked pipeline, which run the same attention kernels).

DSA_PIPELINE_CHUNKS=3 on 7 pairs starts chunks at odd pairs 2 and 4 (the
x^-scratch alignment case of ADVICE round 1)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent
TOL = {"bf16": 1e-2, "f32": 1e-5}

C2S = {"preset": "c2_vector", "pairs": 3, "over": {"L": 1024, "keep": 51}}
C4S = {"preset": "c4_threshold", "pairs": 2, "over": {"L": 1500, "cap": 60}}
C3S = {"preset": "c3_block", "pairs": 2, "over": {"L": 1024, "keep": 5}}
C1S = {"preset": "c1_bert_base", "pairs": 2, "over": {"L": 1024, "keep": 51}}
C0T = {"preset": "c0_smoke", "pairs": 2, "over": {"dtype": "bf16", "round_proj_f32": False}}

CASES = [
    ("DSA_ATTN_GENERIC", "1", C2S, False),
    ("DSA_ATTN_GENERIC", "1", C4S, False),
    ("DSA_ATTN_GENERIC", "1", C3S, False),
    ("DSA_THRESHOLD_GENERIC", "1", C4S, True),
    ("DSA_BLOCK_GENERIC", "1", C3S, True),
    ("DSA_TOPK_GENERIC", "1", C1S, True),
    ("DSA_PREDICT_DFMA", "1", C2S, True),
    ("DSA_PREDICT_DFMA", "1", C0T, True),
    ("DSA_PREDICT_TILES", "1", C2S, True),
    ("DSA_PREDICT_TILES", "1", {"preset": "c2_vector", "pairs": 3, "over": {"L": 1000, "keep": 50}}, True),
    ("DSA_PREDICT_TILES", "1", {"preset": "c2_vector", "pairs": 2, "over": {"L": 4096, "keep": 205}}, True),
    ("DSA_PREDICT_TILES", "1", {"preset": "c2_vector", "pairs": 2, "over": {"L": 3000, "keep": 150, "bits": 8}}, True),
    ("DSA_PREDICT_TILES", "1", {"preset": "c3_block", "pairs": 3, "over": {"L": 1500, "keep": 8}}, True),
    ("DSA_PREDICT_TILES", "1", {"preset": "c4_threshold", "pairs": 2, "over": {"L": 5000, "cap": 300}}, True),
    ("DSA_PREDICT_TILES", "1", {"preset": "c2_vector", "pairs": 2, "over": {"L": 4500, "keep": 200, "bits": 8}}, True),
    ("DSA_FUSE", "1", C2S, False),
    ("DSA_BLOCK_CPASYNC", "1", {"preset": "c3_block", "pairs": 2, "over": {"L": 1024, "keep": 5}}, True),
    ("DSA_BLOCK_CPASYNC", "1", {"preset": "c3_block", "pairs": 3, "over": {"L": 2048, "keep": 16}}, True),
    ("DSA_BLOCK_TC", "1", {"preset": "c3_block", "pairs": 2, "over": {"L": 1024, "keep": 5}}, False),
    ("DSA_BLOCK_TC", "1", {"preset": "c3_block", "pairs": 3, "over": {"L": 2048, "keep": 16}}, False),
    ("DSA_PIPELINE_CHUNKS", "3", {"preset": "c2_vector", "pairs": 7, "over": {"L": 512, "keep": 26}}, True),
    ("DSA_PIPELINE_CHUNKS", "2", {"preset": "c3_block", "pairs": 3, "over": {"L": 512, "keep": 4}}, True),
]


def _run(tmp, tag, spec, env_extra):
    out = tmp / f"{tag}.npz"
    env = {k: v for k, v in os.environ.items() if not k.startswith("DSA_")}
    env.update(env_extra)
    r = subprocess.run([sys.executable, str(HERE / "_switch_run.py"), str(out), json.dumps(spec)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("var,val,spec,exact", CASES, ids=[f"{c[0]}={c[1]}-{c[2]['preset']}" for c in CASES])
def test_switch_preserves_results(var, val, spec, exact, tmp_path):
    base = _run(tmp_path, "base", spec, {})
    alt = _run(tmp_path, "alt", spec, {var: val})
    for key in ("lq", "lk", "sq", "sk", "rp", "cols", "prp", "pcols"):
        assert np.array_equal(base[key], alt[key]), f"{var}: {key} differs"
    assert np.array_equal(base["rp"], base["prp"]) and np.array_equal(base["cols"], base["pcols"])
    from paper_2110_11299_b200 import load_preset
    dt = load_preset(spec["preset"]).replace(**spec["over"]).dtype
    for key in ("z", "zp"):
        a, b = base[key], alt[key]
        if exact:
            assert np.array_equal(a, b), f"{var}: {key} differs"
        else:
            rel = np.abs(a - b).max() / max(np.abs(a).max(), 1e-30)
            assert rel <= TOL[dt], f"{var}: {key} rel {rel}"
