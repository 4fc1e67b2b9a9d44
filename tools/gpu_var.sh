for e in "X=1" "DSA_NO_FUSE=1" "DSA_PIPELINE_CHUNKS=2" "DSA_PIPELINE_CHUNKS=4"; do
  env $e timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-adjacent > gpurun_out/var.json 2>/dev/null
  echo "$e"; python tools/bench_summary.py gpurun_out/var.json
done
