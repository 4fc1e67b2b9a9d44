for v in base ${ABL:-1 3 5}; do
  if [ $v = base ]; then unset DSA_LIB; else export DSA_LIB=ablate/$v/libdsa_b200.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-adjacent > gpurun_out/abl.json 2>gpurun_out/abl.err
  echo "== $v"; python tools/bench_summary.py gpurun_out/abl.json; tail -2 gpurun_out/abl.err
done
