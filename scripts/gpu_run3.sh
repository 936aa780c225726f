timeout 900 python -m pytest tests/test_gpu_projection.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo rc=$?
tail -3 gpurun_out/bench3.err; python -c "
import json; d=json.load(open('gpurun_out/bench3.json')); print(d['ms_per_step'], d['roofline']['passes_ms'], d['roofline']['matvec'])"
