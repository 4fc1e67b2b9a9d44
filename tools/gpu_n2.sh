timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-adjacent > gpurun_out/n1.json 2> gpurun_out/n1.err
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-adjacent > gpurun_out/n2.json 2> gpurun_out/n2.err
python - <<'P'
import json
for f in ("gpurun_out/n1.json", "gpurun_out/n2.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "n_gpus", d["n_gpus"], "checksum", d["checksum"], "pairs_per_gpu", d["config"]["pairs_per_gpu"], d["config"].get("oversubscribed_gpus"))
    except Exception as e:
        print(f, "failed", e)
P
tail -5 gpurun_out/n2.err
