timeout 600 python -m pytest tests/test_gpu_solver.py -x -q -k "simo" > gpurun_out/simo_fail.log 2>&1
python scripts/solve_cfg2.py 256 > gpurun_out/solve_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/launches_solve.csv python scripts/solve_cfg2.py 256 > gpurun_out/ncu_solve.log 2>&1
cat gpurun_out/solve_plain.log
