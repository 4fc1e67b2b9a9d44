"""One-line summary of a bench.py JSON line: value, ms/step, e2e, phase ms."""
import json
import sys

try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:  # noqa: BLE001
    print("bench failed:", e)
    sys.exit(0)
print("value %.4e tok/s  ms %.4f  e2e %.4e  roofline %s %.3f" % (
    d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["kernel"], d["roofline"]["frac"]))
print({k: round(v["ms"], 4) for k, v in d["phases"].items()})
