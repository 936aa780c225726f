for v in 2 4 5; do
FM_XPASS=$v timeout 900 python -m pytest tests/test_gpu_projection.py -q -x -k "matches_oracle" 2>&1 | tail -1
FM_XPASS=$v timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bx$v.json 2>gpurun_out/bx$v.err
python -c "
import json; d=json.load(open('gpurun_out/bx$v.json')); print('x$v mf', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['passes_ms'].items()})"
done
