"""Builds libdsa_b200.so in-tree with nvcc for sm_100a (no JIT cache).

Every CUDA translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``; host code with the
same nvcc driver.  The .so lands next to this file so it travels to the GPU
box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build" / "obj"
LIB = PKG / "libdsa_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          f"-I{ROOT / 'include'}", f"-I{CSRC}", "--expt-relaxed-constexpr", "-Xptxas", "-v"]
SOURCES = ["project.cu", "project_fast.cu", "project_tc.cu", "project_tensor.cu", "select.cu", "attention.cu", "attention_band.cu", "attention_block_tc.cu", "select_colvec.cu", "select_thr.cu", "select_rowsel.cu", "predict_wtilde.cu", "mask_ops.cu", "sparse_ops.cu", "qkv_gemm.cu", "abi.cu", "gen.cpp"]


def _needs(obj: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, jobs: int = 8) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "dsa_b200.h"]
    procs = []
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        objs.append(o)
        if not _needs(o, [s] + headers):
            continue
        cmd = [NVCC, *ARCH, *COMMON, "-c", str(s), "-o", str(o)]
        if s.suffix == ".cpp":
            cmd = [NVCC, *COMMON, "-x", "c++", "-c", str(s), "-o", str(o)]
        log = OBJ / (s.stem + ".log")
        procs.append((s, log, subprocess.Popen(cmd, stdout=open(log, "w"), stderr=subprocess.STDOUT)))
        while len([p for p in procs if p[2].poll() is None]) >= jobs:
            procs[0][2].wait()
    failed = []
    for s, log, p in procs:
        if p.wait() != 0:
            failed.append((s, log))
        elif verbose:
            sys.stdout.write(log.read_text())
    if failed:
        msg = "\n".join(f"--- {s.name}\n{log.read_text()}" for s, log in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    if _needs(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart", "-lpthread"]
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
