python scripts/prof_matvec.py 256 3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python scripts/prof_matvec.py 256 3 > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_x_fast|k_zi_fast|k_zf_fast|k_y_fast" -s 5 -c 5 -o gpurun_out/prof_r1 python scripts/prof_matvec.py 256 3 > gpurun_out/ncu2.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu2.log
