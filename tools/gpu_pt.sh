# one-pass tensor predict: parity + switch + C2 bench + launch list
tag=${1:-pt}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_switches.py tests/test_gpu_predict_edges.py -x -q -k "c2 or PREDICT or predict or xhat or vector" 2>&1 | tail -15 > gpurun_out/${tag}_pytest.log
cat gpurun_out/${tag}_pytest.log
timeout 300 python bench.py --config c2_vector --steps 20 --warmup 5 --no-cpu-baseline --no-adjacent > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python tools/bench_summary.py gpurun_out/${tag}_bench.json; tail -3 gpurun_out/${tag}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/${tag}_launch.csv python bench.py --config c2_vector --steps 2 --warmup 3 --no-cpu-baseline --no-adjacent > /dev/null 2>&1
python tools/launch_means.py gpurun_out/${tag}_launch.csv
