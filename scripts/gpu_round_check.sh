set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_v12.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/gpu_tests_v12.log
tail -3 gpurun_out/gpu_tests_v12.log
timeout 600 python bench.py > gpurun_out/bench_v12.json 2> gpurun_out/bench_v12.err; echo "BENCH EXIT $?"
tail -c 600 gpurun_out/bench_v12.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_v12.json 2> gpurun_out/bench_ref_v12.err; echo "REF EXIT $?"
tail -c 400 gpurun_out/bench_ref_v12.json
