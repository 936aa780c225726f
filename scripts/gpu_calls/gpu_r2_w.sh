mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r2w.log 2>&1; echo rc_tests=$?; tail -25 gpurun_out/gpu_tests_r2w.log
