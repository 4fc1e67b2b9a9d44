# quick GPU check: colvec parity + C2 bench (usage: bash tools/gpu_quick.sh tag [pytest -k expr] [config])
tag=${1:-q}
kexpr=${2:-"colvec or c2 or fused"}
cfg=${3:-c2_vector}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_switches.py -x -q -k "$kexpr" 2>&1 | tail -15 > gpurun_out/${tag}_pytest.log
timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-adjacent > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
cat gpurun_out/${tag}_pytest.log
python tools/bench_summary.py gpurun_out/${tag}_bench.json
tail -5 gpurun_out/${tag}_bench.err
