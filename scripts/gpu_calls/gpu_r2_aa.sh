mkdir -p gpurun_out
timeout 600 python scripts/dist_virtual_passes.py 512 1,2,4,8 5 > gpurun_out/dist_virtual_512_r2aa.jsonl 2>&1; cut -c1-260 gpurun_out/dist_virtual_512_r2aa.jsonl
timeout 600 python scripts/dist_virtual_passes.py 256 1,2,4,8 10 > gpurun_out/dist_virtual_256_r2aa.jsonl 2>&1; cut -c1-260 gpurun_out/dist_virtual_256_r2aa.jsonl
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_projection.py -q -x > gpurun_out/gpu_tests_r2aa.log 2>&1; echo rc_tests=$?; tail -3 gpurun_out/gpu_tests_r2aa.log
