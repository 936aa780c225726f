timeout 900 python bench.py > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; echo rc=$?
python scripts/prof_matvec.py 256 3 mf > gpurun_out/prof3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu3a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_zf_fast|k_x_fast3|k_zi_fast|k_y_fast" -s 5 -c 5 -o gpurun_out/prof_r1c python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu3b.log 2>&1
echo rc2=$?
