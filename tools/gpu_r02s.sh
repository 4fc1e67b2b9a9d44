# r02s: full GPU suite + C2 bench (session re-entry check)
tag=${1:-r02s}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -3 gpurun_out/${tag}_pytest.log
python tools/bench_summary.py gpurun_out/${tag}_bench.json
