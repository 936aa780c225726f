# round 2, call X: smoke, full GPU suite, bench + reference arm, ncu launch list of the bench command
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2x.log 2>&1; echo rc_smoke=$?; tail -2 gpurun_out/smoke_r2x.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r2x.log 2>&1; echo rc_tests=$?; tail -4 gpurun_out/gpu_tests_r2x.log
( time python bench.py > gpurun_out/bench_r2x.json 2> gpurun_out/bench_r2x.err ) 2> gpurun_out/bench_r2x.time; echo rc_bench=$?; tail -3 gpurun_out/bench_r2x.err; cat gpurun_out/bench_r2x.time
( time python bench.py --impl reference > gpurun_out/bench_ref_r2x.json 2> gpurun_out/bench_ref_r2x.err ) 2> gpurun_out/bench_ref_r2x.time; echo rc_ref=$?; cat gpurun_out/bench_ref_r2x.time
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-config3 > gpurun_out/bench_short_r2x.json 2>/dev/null && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/bench_launches_r2x.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-config3 > gpurun_out/ncu_bench_r2x.log 2>&1; echo rc_ncu=$?
