mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r2s.log 2>&1; echo rc_tests=$?; tail -5 gpurun_out/gpu_tests_r2s.log
python bench.py > gpurun_out/bench_r2s.json 2> gpurun_out/bench_r2s.err; echo rc_bench=$?; tail -2 gpurun_out/bench_r2s.err
