"""Profiling-only builds of libdsa_b200.so with -DDSA_ABLATE=<bits> (parts of
the colvec kernel switched off) into ablate/<bits>/; load one with
DSA_LIB=ablate/<bits>/libdsa_b200.so.  Never the product library."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2110_11299_b200 import build as b  # noqa: E402

for spec in sys.argv[1:]:
    # "<bits>" or "<bits>,<MACRO>=<value>,.." (extra -D for the profiled sources)
    bits, *defs = spec.split(",")
    out = b.ROOT / "ablate" / spec
    out.mkdir(parents=True, exist_ok=True)
    objs = []
    for src in b.SOURCES:
        s = b.CSRC / src
        o = b.OBJ / (s.stem + ".o")
        if s.name in ("select_colvec.cu", "project_tc.cu", "select_thr.cu", "attention_band.cu"):
            o = out / (s.stem + ".o")
            subprocess.run([b.NVCC, *b.ARCH, *b.COMMON, f"-DDSA_ABLATE={bits}", *[f"-D{d}" for d in defs], "-c", str(s), "-o", str(o)],
                           check=True, capture_output=True)
        objs.append(str(o))
    subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", str(out / "libdsa_b200.so"), *objs, "-lcudart", "-lpthread"],
                   check=True)
    print(out / "libdsa_b200.so")
