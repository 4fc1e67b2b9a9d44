# colvec ablation builds vs the product library (usage: ABL="1 3" bash tools/gpu_abl.sh)
for v in base ${ABL:-1 3}; do
  unset DSA_LIB
  if [ $v != base ]; then export DSA_LIB=ablate/$v/libdsa_b200.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-adjacent > gpurun_out/abl.json 2>gpurun_out/abl.err
  echo "== $v"; python tools/bench_summary.py gpurun_out/abl.json; tail -2 gpurun_out/abl.err
done
