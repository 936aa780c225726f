# round 2, call B: long-line x pass A/B (k_x_stream), its parity tests, and
# the k_hyper / k_simo register-budget A/B
mkdir -p gpurun_out
timeout 600 python scripts/x_ab.py 512 0,1,2,3 > gpurun_out/x_ab_512_r2b.jsonl 2>&1; echo rc_xab=$?; cat gpurun_out/x_ab_512_r2b.jsonl
timeout 1200 python -m pytest tests/test_gpu_projection.py tests/test_gpu_dist.py tests/test_gpu_svk_oracle.py tests/test_gpu_config4_known_answer.py -q > gpurun_out/gpu_tests_r2b.log 2>&1; echo rc_tests=$?; tail -5 gpurun_out/gpu_tests_r2b.log
for mb in 1 4 6 8; do FM_HYPER_MINB=$mb python scripts/prof_constitutive.py 256 5 hyper; done > gpurun_out/hyper_ab_r2b.jsonl 2>&1; cat gpurun_out/hyper_ab_r2b.jsonl
for mb in 1 2 3; do FM_SIMO_MINB=$mb python scripts/prof_constitutive.py 256 3 simo; done > gpurun_out/simo_ab_r2b.jsonl 2>&1; cat gpurun_out/simo_ab_r2b.jsonl
