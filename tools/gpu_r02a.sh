set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r02a_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_c2.json 2> gpurun_out/r02a_bench_c2.err
tail -3 gpurun_out/r02a_pytest_gpu.log; cat gpurun_out/r02a_smoke.log; cat gpurun_out/r02a_bench_c2.json | head -c 1500
