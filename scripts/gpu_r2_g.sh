mkdir -p gpurun_out
for mb in 4 6 22 23; do FM_HYPER_MINB=$mb python scripts/prof_constitutive.py 256 5 hyper; done > gpurun_out/hyper_ab_r2g.jsonl 2>&1; cat gpurun_out/hyper_ab_r2g.jsonl
for mb in 4 23; do FM_HYPER_MINB=$mb timeout 600 python -m pytest tests/test_gpu_constitutive.py tests/test_gpu_svk_oracle.py -q -k "hyper or k4" 2>&1 | tail -2; done
