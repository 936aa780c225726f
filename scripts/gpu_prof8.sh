# round-1 v8 evidence: GPU tests, bench (both arms), ncu launch list and --set full captures of the matvec passes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo rc_tests=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rcref=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc_smoke=$?
python scripts/prof_matvec.py 256 2 mf > /dev/null 2>&1 && python scripts/prof_matvec.py 256 2 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1v8.csv python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu8c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zf|k_y_fast|k_x_fast|k_zi_reg" -s 5 -c 5 -o gpurun_out/prof_r1v8_mf python scripts/prof_matvec.py 256 2 mf > gpurun_out/ncu8a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zf_fast" -s 1 -c 1 -o gpurun_out/prof_r1v8_k4 python scripts/prof_matvec.py 256 2 > gpurun_out/ncu8b.log 2>&1
echo done
