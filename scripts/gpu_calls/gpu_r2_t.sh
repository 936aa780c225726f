mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_dist.py tests/test_gpu_config3_reduced.py tests/test_gpu_config3_128.py -q > gpurun_out/gpu_tests_r2t.log 2>&1; echo rc_tests=$?; tail -30 gpurun_out/gpu_tests_r2t.log
