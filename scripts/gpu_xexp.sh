# 512-point x pass: direct lane-pair kernel (default) against the staged k_x_fast4
mkdir -p gpurun_out
for m in 0 1; do FM_XDIRECT=$m timeout 300 python scripts/xdirect_check.py > gpurun_out/xd$m.json 2>&1; echo "xdirect=$m rc=$?"; cat gpurun_out/xd$m.json; done
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo rc_tests=$?; tail -3 gpurun_out/pytest_gpu.log
python scripts/pass_times.py 256 512 > gpurun_out/pt.json; cat gpurun_out/pt.json
