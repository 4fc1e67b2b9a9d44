timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_switches.py tests/test_gpu_properties.py -x -q -m gpu -k "threshold or c4" 2>&1 | tail -15 > gpurun_out/g1_pytest.log
timeout 600 python bench.py --config c4_threshold --steps 5 --warmup 3 --no-cpu-baseline --no-adjacent > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
cat gpurun_out/g1_pytest.log; python tools/bench_summary.py gpurun_out/g1_bench.json; tail -3 gpurun_out/g1_bench.err
