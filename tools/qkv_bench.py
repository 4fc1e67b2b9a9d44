"""Times dsa_project_qkv (the fused Q/K/V + predictor-input GEMM, SURVEY
8(f) item 3) on the BASELINE layer shapes with CUDA events and reports
TFLOP/s against the measured bf16 peak (MEASURED_PEAKS.json).
usage: python tools/qkv_bench.py [--reps N]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2110_11299_b200 import load_preset, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--configs", default="c1_bert_base,c2_vector,c3_block,c4_threshold")
a = ap.parse_args()
peak = None
try:
    mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    peak = mp.get("bf16_tflops")
except Exception:
    pass
for name in a.configs.split(","):
    p = load_preset(name)
    sh = p.shape
    dm, heads, dk, dv = sh["d"], p.heads, sh["d_k"], sh["d_v"]
    batch = p.batch
    if name == "c4_threshold":
        batch = 4  # 4 x 16384 rows (the full 32-batch layer is 8x the same work)
    npred = p.k
    x = torch.randn(batch, p.L, dm, device="cuda").to(torch.bfloat16)
    w = (torch.randn(heads * (2 * dk + dv) + npred, dm, device="cuda") / dm ** 0.5).to(torch.bfloat16)
    out = (torch.empty(batch * heads, p.L, dk, dtype=torch.bfloat16, device="cuda"),
           torch.empty(batch * heads, p.L, dk, dtype=torch.bfloat16, device="cuda"),
           torch.empty(batch * heads, p.L, dv, dtype=torch.bfloat16, device="cuda"),
           torch.empty(batch, p.L, npred, dtype=torch.float32, device="cuda"))
    for _ in range(3):
        ops.project_qkv(x, w, heads, dk, dv, npred, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        ops.project_qkv(x, w, heads, dk, dv, npred, out=out)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    M, N = batch * p.L, heads * (2 * dk + dv) + npred
    flops = 2.0 * M * N * dm
    byts = M * dm * 2 + N * dm * 2 + M * heads * (2 * dk + dv) * 2 + M * npred * 4
    tf = flops / ms / 1e9
    # cuBLAS (torch.matmul) on the same GEMM, for reference (no head split)
    y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    xm = x.reshape(M, dm)
    for _ in range(3):
        torch.matmul(xm, w.t(), out=y)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        torch.matmul(xm, w.t(), out=y)
    e1.record()
    e1.synchronize()
    ms_cublas = e0.elapsed_time(e1) / a.reps
    print(json.dumps({"config": name, "M": M, "N": N, "K": dm, "ms": round(ms, 4), "tflops": round(tf, 1),
                      "frac_of_peak": round(tf / peak, 3) if peak else None, "peak_tflops": peak,
                      "GBps": round(byts / ms / 1e6, 1), "cublas_ms": round(ms_cublas, 4),
                      "cublas_tflops": round(flops / ms_cublas / 1e9, 1)}))
