timeout 900 python -m pytest tests/test_gpu_projection.py tests/test_gpu_solver.py -q -x 2>&1 | tail -2
for v in 1 2 3; do
FM_XPASS=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bx$v.json 2>gpurun_out/bx$v.err
python -c "
import json; d=json.load(open('gpurun_out/bx$v.json')); print('x$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['passes_ms'].items()})"
done
python scripts/bench_configs.py 2 | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items(): print(k, round(v['wall_s'],3), 'matvecs', v['matvecs'], 'per-mv ms', round(1e3*v['wall_s']/v['matvecs'],3))"
