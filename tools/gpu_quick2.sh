# parity (all attention tests) + bench C2, C4, C1 (usage: bash tools/gpu_quick2.sh tag)
tag=${1:-q2}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_switches.py tests/test_gpu_counters.py -x -q 2>&1 | tail -15 > gpurun_out/${tag}_pytest.log
cat gpurun_out/${tag}_pytest.log
for c in c2_vector c4_threshold c1_bert_base; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-adjacent > gpurun_out/${tag}_$c.json 2> gpurun_out/${tag}_$c.err
  echo "== $c"; python tools/bench_summary.py gpurun_out/${tag}_$c.json; tail -2 gpurun_out/${tag}_$c.err
done
