mkdir -p gpurun_out
timeout 600 python scripts/x_ab.py 512 1,2,3 > gpurun_out/x_ab_512_r2c.jsonl 2>&1; echo rc_xab=$?; cat gpurun_out/x_ab_512_r2c.jsonl
timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_dist.py tests/test_gpu_config4_known_answer.py -q -x > gpurun_out/gpu_tests_r2c.log 2>&1; echo rc_tests=$?; tail -5 gpurun_out/gpu_tests_r2c.log
