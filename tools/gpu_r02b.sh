python -m pytest tests/test_gpu_wtilde.py tests/test_gpu_counters.py tests/test_gpu_cpp_shim.py -x -q -s 2>&1 | tail -30 > gpurun_out/r02b_pytest.log
cat gpurun_out/r02b_pytest.log
