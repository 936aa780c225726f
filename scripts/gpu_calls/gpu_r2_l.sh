mkdir -p gpurun_out
python scripts/x_stride.py 128x128x128,256x256x256,512x512x512 10 > gpurun_out/x_r2l.jsonl 2>&1; cat gpurun_out/x_r2l.jsonl
for d in 1 2 3; do FM_X_DBG=$d python scripts/x_stride.py 512x512x512 5; done > gpurun_out/x_dbg_r2l.jsonl 2>&1; cat gpurun_out/x_dbg_r2l.jsonl
timeout 1500 python -m pytest tests/test_gpu_projection.py tests/test_gpu_dist.py tests/test_gpu_config4_known_answer.py -q -x > gpurun_out/gpu_tests_r2l.log 2>&1; echo rc_tests=$?; tail -3 gpurun_out/gpu_tests_r2l.log
