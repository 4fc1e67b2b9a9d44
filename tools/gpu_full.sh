# full GPU check: every GPU test, smoke, bench of every config (usage: bash tools/gpu_full.sh tag)
tag=${1:-full}
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
for c in c2_vector c3_block c4_threshold c1_bert_base c0_smoke; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-adjacent > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  echo "== $c"; python tools/bench_summary.py gpurun_out/${tag}_bench_$c.json
done
tail -3 gpurun_out/${tag}_pytest.log; cat gpurun_out/${tag}_smoke.log | tail -2
