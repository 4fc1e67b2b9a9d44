timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_bounds.py -x -q -k "c3 or block" 2>&1 | tail -12
timeout 300 python bench.py --config c3_block --steps 10 --warmup 3 --no-cpu-baseline --no-adjacent > gpurun_out/c3.json 2> gpurun_out/c3.err
python tools/bench_summary.py gpurun_out/c3.json; tail -3 gpurun_out/c3.err
