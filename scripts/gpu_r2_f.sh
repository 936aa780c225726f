mkdir -p gpurun_out
timeout 900 python scripts/x_ab.py 512 2,3,4,6 > gpurun_out/x_ab_512_r2f.jsonl 2>&1; cat gpurun_out/x_ab_512_r2f.jsonl
FM_TMA_PROMO=0 timeout 900 python scripts/x_ab.py 512 2,3,4,6 > gpurun_out/x_ab_512_r2f_p0.jsonl 2>&1; cat gpurun_out/x_ab_512_r2f_p0.jsonl
FM_TMA_PROMO=3 timeout 900 python scripts/x_ab.py 512 2,4 > gpurun_out/x_ab_512_r2f_p3.jsonl 2>&1; cat gpurun_out/x_ab_512_r2f_p3.jsonl
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r2f.log 2>&1; echo rc_tests=$?; tail -8 gpurun_out/gpu_tests_r2f.log
