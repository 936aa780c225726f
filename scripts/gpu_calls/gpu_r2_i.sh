# round 2, call I (re-entry baseline): smoke, full GPU suite, bench, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2i.log 2>&1; echo rc_smoke=$?; tail -2 gpurun_out/smoke_r2i.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r2i.log 2>&1; echo rc_tests=$?; tail -8 gpurun_out/gpu_tests_r2i.log
( time python bench.py > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err ) 2> gpurun_out/bench_r2i.time; echo rc_bench=$?; tail -3 gpurun_out/bench_r2i.err; cat gpurun_out/bench_r2i.time
( time python bench.py --impl reference > gpurun_out/bench_ref_r2i.json 2> gpurun_out/bench_ref_r2i.err ) 2> gpurun_out/bench_ref_r2i.time; echo rc_ref=$?; cat gpurun_out/bench_ref_r2i.time
