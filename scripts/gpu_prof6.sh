python scripts/prof_matvec.py 256 2 mf > /dev/null 2>&1 && python scripts/prof_matvec.py 256 2 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_zf|k_y_fast|k_x_fast|k_zi_fast" -s 5 -c 5 -o gpurun_out/prof_r1h_mf python scripts/prof_matvec.py 256 2 mf > gpurun_out/ncu6a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zf_fast" -s 1 -c 1 -o gpurun_out/prof_r1h_k4 python scripts/prof_matvec.py 256 2 > gpurun_out/ncu6b.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1h.csv python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu6c.log 2>&1
echo done
