# round 2, final call on HEAD: smoke, full GPU suite, bench, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2final.log 2>&1; echo rc_smoke=$?; tail -2 gpurun_out/smoke_r2final.log | cut -c1-200
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r2final.log 2>&1; echo rc_tests=$?; tail -4 gpurun_out/gpu_tests_r2final.log
( time python bench.py > gpurun_out/bench_r2final.json 2> gpurun_out/bench_r2final.err ) 2> gpurun_out/bench_r2final.time; echo rc_bench=$?; tail -2 gpurun_out/bench_r2final.err; cat gpurun_out/bench_r2final.time
( time python bench.py --impl reference > gpurun_out/bench_ref_r2final.json 2> gpurun_out/bench_ref_r2final.err ) 2> gpurun_out/bench_ref_r2final.time; echo rc_ref=$?; cat gpurun_out/bench_ref_r2final.time
