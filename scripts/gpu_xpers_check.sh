# A/B of a persistent k_x_fast4 with next-tile prefetch (FM_XPERS, measured and dropped in v13: DESIGN §3)
for i in 1 2; do
  for v in 0 1; do FM_XPERS=$v timeout 120 python scripts/svk_check.py 256 svk; done
done 2>&1 | tee gpurun_out/xpers_check.log
for v in 0 1; do FM_XPERS=$v timeout 120 python scripts/svk_check.py 128 svk; done 2>&1 | tee -a gpurun_out/xpers_check.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_x0.log 2>&1; echo "TESTS0 EXIT $?" >> gpurun_out/gpu_tests_x0.log; tail -2 gpurun_out/gpu_tests_x0.log
FM_XPERS=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_x1.log 2>&1; echo "TESTS1 EXIT $?" >> gpurun_out/gpu_tests_x1.log; tail -2 gpurun_out/gpu_tests_x1.log
