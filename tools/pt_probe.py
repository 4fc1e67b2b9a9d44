"""Phase timeline of project_tensor_kernel (profiling-only build with
-DDSA_PT_PROBE; usage: python tools/pt_probe.py build | run [config])."""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
OUT = ROOT / "ablate" / "ptprobe"

if sys.argv[1] == "build":
    from paper_2110_11299_b200 import build as b
    OUT.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in b.SOURCES:
        s = b.CSRC / src
        o = b.OBJ / (s.stem + ".o")
        if s.name == "project_tensor.cu":
            o = OUT / "project_tensor.o"
            subprocess.run([b.NVCC, *b.ARCH, *b.COMMON, "-DDSA_PT_PROBE", "-c", str(s), "-o", str(o)], check=True)
        objs.append(str(o))
    subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", str(OUT / "libdsa_b200.so"), *objs, "-lcudart", "-lpthread"],
                   check=True)
    print(OUT / "libdsa_b200.so")
    sys.exit(0)

os.environ["DSA_LIB"] = str(OUT / "libdsa_b200.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2110_11299_b200 import load_preset, ops  # noqa: E402
from paper_2110_11299_b200 import _abi  # noqa: E402

cfg = sys.argv[2] if len(sys.argv) > 2 else "c2_vector"
p = load_preset(cfg)
npairs = p.pairs
q, k, v, P = (t.cuda() for t in ops.generate(p, npairs=npairs))
ph = ops.Phases(p, npairs)
for _ in range(4):
    ph.predict(q, k, P)
torch.cuda.synchronize()
n = 2 * npairs
buf = (ctypes.c_ulonglong * (8 * 4096))()
lib = _abi.lib()
assert lib.dsa_pt_probe_read(buf, ctypes.c_int(min(n, 4096))) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8)[:n].astype(np.float64)
t0 = a[:, 0].min()
names = ["prologue", "stream", "cand", "chains", "quant", "chains2"]
d = np.diff(a[:, :7], axis=1) / 1000.0
print(f"CTAs {n}, kernel span {(a[:, 6].max() - t0) / 1000:.2f} us")
for i, nm in enumerate(names):
    print(f"{nm:9s} mean {d[:, i].mean():7.2f} us  max {d[:, i].max():7.2f}")
st = (a[:, 0] - t0) / 1000
print("start times: first wave <", np.sort(st)[147], "us; last start", st.max())
print("per-CTA total mean", ((a[:, 6] - a[:, 0]) / 1000).mean())
cb = (ctypes.c_uint * (2 * 4096))()
if lib.dsa_pt_count_read(cb, ctypes.c_int(min(n, 4096))) == 0:
    c = np.frombuffer(cb, dtype=np.uint32).reshape(4096, 2)[:n] / 4.0  # 3 warm-up calls + 1
    print(f"per CTA per call: streaming chains mean {c[:, 0].mean():.1f} max {c[:, 0].max():.0f}; "
          f"listed levels mean {c[:, 1].mean():.1f} max {c[:, 1].max():.0f}")
