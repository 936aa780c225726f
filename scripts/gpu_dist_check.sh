timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python scripts/dist_virtual_timing.py 256 10 > gpurun_out/dist_virtual_256.log 2>&1; tail -1 gpurun_out/dist_virtual_256.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_quick.json'));print(d['ms_per_step'], d['roofline']['passes_ms'])"
