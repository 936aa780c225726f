# round-1 final check on HEAD: smoke, bench (both arms)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke13.log 2>&1; echo rc_smoke=$?; tail -1 gpurun_out/smoke13.log
timeout 600 python bench.py > gpurun_out/bench13.json 2> gpurun_out/bench13.err; echo rc_bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench13_ref.json 2> gpurun_out/bench13_ref.err; echo rc_ref=$?
tail -c 300 gpurun_out/bench13_ref.json
