"""Preset format: the reference's cost-preset ``shape`` schema plus a sibling
``dsa`` block (SURVEY.md 8(b) "Preset format to keep").

``shape`` keeps the reference keys and meaning exactly: required
``l, d, d_k, d_v, heads, ffn``; optional ``proj_k, pred_bits, beta_override``
(P/src/cli_commands.cpp:167-182); unknown keys are rejected like
``check_keys`` (P/src/cli_commands.cpp:26-34) with ConfigError.  Here
``proj_k`` is the projection width k, ``pred_bits`` the prediction precision
("full" | 2 | 4 | 8 | 16, P/src/cli_commands.cpp:36-49) and d_k = d_v = d_head.

The ``dsa`` block carries everything the reference has no key for, with
explicit integer keep counts.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field, asdict
from pathlib import Path

from .errors import ConfigError

PRESET_DIR = Path(__file__).resolve().parent / "presets"

_SHAPE_REQUIRED = {"l", "d", "d_k", "d_v", "heads", "ffn"}
_SHAPE_OPTIONAL = {"proj_k", "pred_bits", "beta_override"}
_TOP_KEYS = {"shape", "dsa", "out_prefix", "preset", "sparsities", "energy_table"}
_DSA_KEYS = {"batch", "dtype", "quant_scope", "mask_mode", "keep", "vec_v", "block",
             "force_diag", "theta_frac", "cap", "causal", "scale", "seed",
             "planted_per_mille", "band_width", "round_proj_f32"}

MASK_MODES = {"row_topk": 0, "colvec": 1, "block": 2, "threshold": 3}
DTYPES = {"f32": 0, "bf16": 1}
QUANT_SCOPES = {"tensor": 0, "row": 1}


def check_keys(obj, ctx: str, required: set, optional: set) -> None:
    """Strict key check, as P/src/cli_commands.cpp:26-34."""
    if not isinstance(obj, dict):
        raise ConfigError(f"{ctx}: expected an object")
    for k in sorted(required):
        if k not in obj:
            raise ConfigError(f"{ctx}: missing required key '{k}'")
    for k in obj:
        if k not in required and k not in optional:
            raise ConfigError(f"{ctx}: unknown key '{k}'")


def parse_bits(v, ctx: str) -> int:
    """P/src/cli_commands.cpp:36-49: a number or "full" (0)."""
    if isinstance(v, str):
        if v != "full":
            raise ConfigError(f'{ctx}: bits must be a number or "full"')
        return 0
    if isinstance(v, bool) or not isinstance(v, int):
        raise ConfigError(f'{ctx}: bits must be a number or "full"')
    if v not in (0, 2, 4, 8, 16):
        raise ConfigError(f"{ctx}: QuantSpec: bits must be one of {{2,4,8,16,full}}")
    return v


@dataclass
class Preset:
    name: str
    batch: int
    heads: int
    L: int
    d: int           # per-head width (d_k = d_v)
    k: int           # projection width (proj_k)
    bits: int
    dtype: str = "bf16"
    quant_scope: str = "tensor"
    mask_mode: str = "row_topk"
    keep: int = 0
    vec_v: int = 8
    block: int = 32
    force_diag: bool = False
    frac_num: int = 1
    frac_den: int = 20
    cap: int = 1
    causal: bool = False
    scale: bool = True
    round_proj_f32: bool = False
    seed: int = 0
    planted_per_mille: int = 20
    band_width: int = 0
    shape: dict = field(default_factory=dict)

    @property
    def pairs(self) -> int:
        return self.batch * self.heads

    @property
    def tokens(self) -> int:
        return self.batch * self.L

    def replace(self, **kw) -> "Preset":
        d = asdict(self)
        d.update(kw)
        return Preset(**d)

    def summary(self) -> dict:
        out = {"workload": self.name, "batch": self.batch, "heads": self.heads, "L": self.L,
               "d_head": self.d, "proj_k": self.k, "pred_bits": self.bits,
               "quant": self.quant_scope, "mask": self.mask_mode, "dtype": self.dtype}
        if self.mask_mode in ("row_topk", "colvec", "block"):
            out["keep"] = self.keep
        if self.mask_mode == "colvec":
            out["vec_v"] = self.vec_v
        if self.mask_mode == "block":
            out["block"] = self.block
            out["force_diag"] = self.force_diag
        if self.mask_mode == "threshold":
            out["theta"] = f"{self.frac_den}/({self.frac_num}*L)"
            out["cap"] = self.cap
            out["causal"] = self.causal
        return out


def parse_preset(doc: dict, name: str = "custom") -> Preset:
    check_keys(doc, "config", set(), _TOP_KEYS)
    if "shape" not in doc:
        raise ConfigError("dsa: need 'shape'")
    sh = doc["shape"]
    check_keys(sh, "shape", _SHAPE_REQUIRED, _SHAPE_OPTIONAL)
    for key in ("l", "d", "d_k", "d_v", "heads", "ffn"):
        if isinstance(sh[key], bool) or not isinstance(sh[key], int) or sh[key] < 1:
            raise ConfigError(f"shape.{key}: must be a positive integer")
    if sh["d_k"] != sh["d_v"]:
        raise ConfigError("shape: the DSA hot path needs d_k == d_v")
    bits = parse_bits(sh.get("pred_bits", 4), "shape.pred_bits")
    dsa = doc.get("dsa", {})
    check_keys(dsa, "dsa", set(), _DSA_KEYS)
    mode = dsa.get("mask_mode", "row_topk")
    if mode not in MASK_MODES:
        raise ConfigError(f"dsa.mask_mode: unknown mode '{mode}'")
    dtype = dsa.get("dtype", "bf16")
    if dtype not in DTYPES:
        raise ConfigError(f"dsa.dtype: unknown dtype '{dtype}'")
    scope = dsa.get("quant_scope", "tensor")
    if scope not in QUANT_SCOPES:
        raise ConfigError(f"dsa.quant_scope: unknown scope '{scope}'")
    tf = dsa.get("theta_frac", [1, 20])
    if (not isinstance(tf, list) or len(tf) != 2 or not all(isinstance(x, int) for x in tf)):
        raise ConfigError("dsa.theta_frac: expected [num, den] integers")
    p = Preset(
        name=doc.get("out_prefix", name), batch=int(dsa.get("batch", 1)), heads=sh["heads"],
        L=sh["l"], d=sh["d_k"], k=int(sh.get("proj_k", 0) or 16), bits=bits, dtype=dtype,
        quant_scope=scope, mask_mode=mode, keep=int(dsa.get("keep", 0)),
        vec_v=int(dsa.get("vec_v", 8)), block=int(dsa.get("block", 32)),
        force_diag=bool(dsa.get("force_diag", False)), frac_num=tf[0], frac_den=tf[1],
        cap=int(dsa.get("cap", sh["l"])), causal=bool(dsa.get("causal", False)),
        scale=bool(dsa.get("scale", True)),
        round_proj_f32=bool(dsa.get("round_proj_f32", dtype == "f32")),
        seed=int(dsa.get("seed", 0)), planted_per_mille=int(dsa.get("planted_per_mille", 20)),
        band_width=int(dsa.get("band_width", 0)), shape=dict(sh))
    if mode in ("row_topk", "colvec", "block") and p.keep < 1:
        raise ConfigError("dsa.keep: explicit integer keep count required")
    return p


def load_preset(name_or_path: str) -> Preset:
    path = Path(name_or_path)
    if not path.exists():
        path = PRESET_DIR / f"{name_or_path}.json"
    if not path.exists():
        raise ConfigError(f"unknown preset: {name_or_path}")
    try:
        doc = json.loads(path.read_text())
    except json.JSONDecodeError as e:
        raise ConfigError(f"{path}: {e}") from None
    return parse_preset(doc, path.stem)


# BASELINE.json configs[0..4]
CONFIG_NAMES = ["c0_smoke", "c1_bert_base", "c2_vector", "c3_block", "c4_threshold"]


def baseline_configs() -> list[Preset]:
    return [load_preset(n) for n in CONFIG_NAMES]
