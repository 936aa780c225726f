timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bq.json 2>gpurun_out/bq.err
python -c "
import json; d=json.load(open('gpurun_out/bq.json')); print('mf', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['passes_ms'].items()}); print('k4', round(d['value_k4']['ms_per_step'],3), {k: round(v,3) for k,v in d['value_k4']['roofline']['passes_ms'].items()})"
