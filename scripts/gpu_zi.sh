timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for v in 0 1 6; do
FM_ZIPIPE=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_zi$v.json 2> gpurun_out/bench_zi$v.err
python -c "import json;d=json.load(open('gpurun_out/bench_zi$v.json'));print('ZIPIPE=$v', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['roofline']['passes_ms'].items()}, round(d['value_k4']['ms_per_step'],4), {k:round(v,4) for k,v in d['value_k4']['roofline']['passes_ms'].items()}, d['newton_solve']['device_solve_s'], d['newton_solve']['cg_iterations'])"
done
