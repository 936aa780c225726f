mkdir -p gpurun_out
timeout 600 python scripts/dist_virtual_passes.py 512 1,8 5 2>&1 | grep fused | cut -c1-200
timeout 600 python scripts/dist_virtual_passes.py 256 1,8 10 2>&1 | grep fused | cut -c1-200
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/gpu_tests_r2ab.log 2>&1; echo rc_tests=$?; tail -3 gpurun_out/gpu_tests_r2ab.log
