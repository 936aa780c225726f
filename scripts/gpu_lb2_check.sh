# A/B of the two-line-buffer pipelined pass 1 (FM_ZPIPE_LB2=1, default) against one line buffer:
# matvec pass times (bitwise checksums must agree), the config-2 fused-CG Newton solve, then the GPU suite and bench
for i in 1 2; do
  for v in 0 1; do FM_ZPIPE_LB2=$v timeout 120 python scripts/svk_check.py 256 svk; done
done 2>&1 | tee gpurun_out/lb2_check.log
for v in 0 1; do FM_ZPIPE_LB2=$v timeout 120 python scripts/svk_check.py 128 svk; done 2>&1 | tee -a gpurun_out/lb2_check.log
for v in 0 1 0 1; do echo "FM_ZPIPE_LB2=$v"; FM_ZPIPE_LB2=$v timeout 200 python scripts/solve_cfg2.py 256 mf; done 2>&1 | tee -a gpurun_out/lb2_check.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_lb2.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/gpu_tests_lb2.log
tail -2 gpurun_out/gpu_tests_lb2.log
timeout 600 python bench.py > gpurun_out/bench_lb2.json 2> gpurun_out/bench_lb2.err; echo "BENCH EXIT $?"
