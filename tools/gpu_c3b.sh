timeout 900 python -m pytest tests/test_gpu_switches.py -x -q -k "BLOCK_TC" 2>&1 | tail -3
DSA_BLOCK_TC=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_bounds.py -x -q -k "c3 or block" 2>&1 | tail -3
