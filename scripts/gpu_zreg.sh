timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python scripts/pass_times.py 128 256 512 2>&1 | tail -4
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_quick.json'));print(d['ms_per_step'], d['roofline']['passes_ms'], d['value_k4']['ms_per_step'], d['e2e']['value'], d['newton_solve']['device_solve_s'], d['newton_solve']['cg_iterations'], d['newton_solve_31'])"
