bash tools/gpu_quick.sh pq1 "c2 or c4 or predict or xhat" c2_vector
timeout 300 python bench.py --config c4_threshold --steps 10 --warmup 3 --no-cpu-baseline --no-adjacent > gpurun_out/pq1_c4.json 2>/dev/null; python tools/bench_summary.py gpurun_out/pq1_c4.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/pq1_launch.csv python bench.py --config c2_vector --steps 2 --warmup 3 --no-cpu-baseline --no-adjacent > /dev/null 2>&1
python tools/ncu_lines.py gpurun_out/pq1_launch.csv 2>&1 | tail -12
