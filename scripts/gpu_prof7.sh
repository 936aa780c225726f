# round-1 v7 evidence: bench (both arms), ncu launch list and --set full captures of the matvec passes
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo rcref=$?
python scripts/prof_matvec.py 256 2 mf > /dev/null 2>&1 && python scripts/prof_matvec.py 256 2 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1v7.csv python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu7c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zf|k_y_fast|k_x_fast|k_zi_reg" -s 5 -c 5 -o gpurun_out/prof_r1v7_mf python scripts/prof_matvec.py 256 2 mf > gpurun_out/ncu7a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zf_fast" -s 1 -c 1 -o gpurun_out/prof_r1v7_k4 python scripts/prof_matvec.py 256 2 > gpurun_out/ncu7b.log 2>&1
echo done
