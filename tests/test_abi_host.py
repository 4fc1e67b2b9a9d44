"""CPU-side checks of the drop-in boundary and the host logic: the C-ABI
library loads and exports every symbol include/dsa_b200.h declares,
validation maps onto the reference exception types, workspace / capacity
planning, the preset format, and the seeded generator.  No kernel runs."""
import ctypes as C
import json

import numpy as np
import pytest
import torch

from paper_2110_11299_b200 import (CONFIG_NAMES, ConfigError, CudaError, ParamError, ShapeError,
                                   UnsupportedError, load_preset, ops, parse_preset)
from paper_2110_11299_b200 import _abi


def test_library_exports_every_header_symbol():
    lib = _abi.lib()
    syms = _abi.header_symbols()
    assert len(syms) >= 12
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.dsa_abi_version() == 1
    assert b"sm_100a" in lib.dsa_build_info()


def test_kernels_are_sm100a_cubins():
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "LDTM", "DMMA", "HMMA"):
        assert mnemonic in sass, mnemonic  # tcgen05 / TMEM / fp64 tensor / mma.sync paths


@pytest.mark.parametrize("name", CONFIG_NAMES)
def test_baseline_presets_validate(name):
    p = load_preset(name)
    ops.validate(p)
    assert ops.workspace_bytes(p) > 0
    assert ops.mask_capacity(p) > 0


def test_preset_values_match_baseline_configs():
    c = {n: load_preset(n) for n in CONFIG_NAMES}
    assert (c["c0_smoke"].pairs, c["c0_smoke"].L, c["c0_smoke"].keep, c["c0_smoke"].dtype) == (1, 512, 51, "f32")
    assert (c["c1_bert_base"].pairs, c["c1_bert_base"].L, c["c1_bert_base"].keep) == (96, 2048, 102)
    assert c["c1_bert_base"].quant_scope == "row" and c["c1_bert_base"].band_width == 32
    assert (c["c2_vector"].pairs, c["c2_vector"].L, c["c2_vector"].vec_v, c["c2_vector"].keep) == (128, 4096, 8, 205)
    assert (c["c3_block"].pairs, c["c3_block"].L, c["c3_block"].d, c["c3_block"].k, c["c3_block"].bits) == (64, 8192, 128, 32, 8)
    assert c["c3_block"].force_diag and c["c3_block"].keep == 16 and c["c3_block"].planted_per_mille == 10
    c4 = c["c4_threshold"]
    assert (c4.pairs, c4.L, c4.causal, c4.cap, c4.frac_num, c4.frac_den) == (512, 16384, True, 1311, 1, 20)
    assert c["c2_vector"].tokens == 65536


def test_preset_format_is_strict():
    doc = json.loads((load_preset.__globals__["PRESET_DIR"] / "c2_vector.json").read_text())
    parse_preset(doc)
    bad = json.loads(json.dumps(doc))
    bad["shape"]["unknown"] = 1
    with pytest.raises(ConfigError, match="unknown key 'unknown'"):
        parse_preset(bad)
    bad = json.loads(json.dumps(doc))
    del bad["shape"]["ffn"]
    with pytest.raises(ConfigError, match="missing required key 'ffn'"):
        parse_preset(bad)
    bad = json.loads(json.dumps(doc))
    bad["shape"]["pred_bits"] = 5
    with pytest.raises(ConfigError):
        parse_preset(bad)
    bad = json.loads(json.dumps(doc))
    del bad["dsa"]["keep"]
    with pytest.raises(ConfigError, match="keep"):
        parse_preset(bad)
    with pytest.raises(ConfigError):
        load_preset("no_such_preset")


def test_validation_errors_map_to_reference_types():
    p = load_preset("c0_smoke")
    with pytest.raises(ParamError, match="k_keep out of range"):
        ops.validate(p.replace(keep=0))
    with pytest.raises(ParamError, match="k_keep out of range"):
        ops.validate(p.replace(keep=513))
    with pytest.raises(ShapeError):
        ops.validate(p.replace(L=0))
    with pytest.raises(UnsupportedError):
        ops.validate(p.replace(d=48))
    with pytest.raises(UnsupportedError):
        ops.validate(p.replace(bits=16))
    with pytest.raises(ParamError):
        ops.validate(p.replace(bits=3))
    with pytest.raises(ParamError, match="vector height"):
        ops.validate(load_preset("c2_vector").replace(vec_v=0))
    with pytest.raises(UnsupportedError):
        ops.validate(load_preset("c4_threshold").replace(quant_scope="row"))


def test_threshold_capacity_bound():
    p = load_preset("c4_threshold")
    b = min(p.cap, p.L * p.frac_num // p.frac_den)  # <= L/20 keys can reach p >= 20/L
    per_pair = b * (b + 1) // 2 + (p.L - b) * b
    assert ops.mask_capacity(p) == p.pairs * per_pair
    assert ops.mask_capacity(p.replace(causal=False)) == p.pairs * p.L * b


def test_hot_path_fails_loudly_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = ops.config_of(load_preset("c0_smoke"))
    st = _abi.lib().dsa_predict(C.byref(c), None, None, None, None, None, None, None, None, 0, None)
    assert st == CudaError.code
    assert b"no CUDA device" in _abi.lib().dsa_last_error()


def test_generator_is_seeded_and_pairwise_independent():
    p = load_preset("c2_vector").replace(L=256, batch=4, heads=1)
    q1, k1, v1, P1 = ops.generate(p)
    q2, k2, v2, P2 = ops.generate(p)
    assert torch.equal(q1, q2) and torch.equal(v1, v2) and torch.equal(P1, P2)
    # pair 2 regenerated alone equals pair 2 of the batch (substream per pair)
    q3, k3, v3, _ = ops.generate(p, pair0=2, npairs=1)
    assert torch.equal(q3[0], q1[2]) and torch.equal(k3[0], k1[2])
    assert not torch.equal(q1[0], q1[1])
    assert q1.dtype == torch.bfloat16 and P1.dtype == torch.float32
    # P ~ N(0, 1/k)
    assert abs(float(P1.std()) - (1 / p.k) ** 0.5) < 0.05
    # 2% planted keys: exactly round(0.02 L) K rows differ from the unplanted draw
    pp = p.replace(L=4096, batch=1)
    _, k, _, _ = ops.generate(pp, npairs=1)
    _, k0, _, _ = ops.generate(pp.replace(planted_per_mille=0), npairs=1)
    changed = (k[0] != k0[0]).any(dim=1)
    assert int(changed.sum()) == 82


def test_generator_f32_and_band():
    p = load_preset("c1_bert_base").replace(L=128, batch=1, heads=1)
    q, k, _, _ = ops.generate(p)
    # band bias: same-window q.k raised by ~1 relative to other windows
    s = (q[0].double() @ k[0].double().T).numpy()
    same = np.mean([s[i, j] for i in range(128) for j in range(128) if i // 32 == j // 32 and i != j])
    diff = np.mean([s[i, j] for i in range(128) for j in range(128) if i // 32 != j // 32])
    assert 0.5 < same - diff < 1.5
    q0, _, _, _ = ops.generate(load_preset("c0_smoke"))
    assert q0.dtype == torch.float32
