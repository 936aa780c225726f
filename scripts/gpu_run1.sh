set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_projection.py -x -q 2>&1 | tail -30
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$?
tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
