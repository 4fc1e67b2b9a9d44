"""Runs the C++ drop-in test (tests/cpp/test_shim.cpp -> oracle/_ref/test_shim):
include/dsattn_gpu.hpp called with the reference's own types and compared with
the reference implementation linked into the same binary."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "test_shim"


def test_cpp_shim_against_reference():
    if not BIN.exists():
        pytest.skip("oracle/_ref/test_shim not built (needs /root/reference at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


EVAL_BIN = BIN.parent / "test_eval"


def test_cpp_evaluate_through_gpu_path():
    """the reference's evaluate / forward_batch against
    include/dsattn_gpu_eval.hpp (identical masks, identical predictions,
    unchanged accuracy), reference trainer objects linked in the same binary."""
    if not EVAL_BIN.exists():
        pytest.skip("oracle/_ref/test_eval not built (needs /root/reference at build time)")
    r = subprocess.run([str(EVAL_BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
