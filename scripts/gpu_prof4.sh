timeout 900 python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err; echo rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r1d_ref.json 2>&1
python scripts/prof_matvec.py 256 3 mf > gpurun_out/prof4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu4a.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_zf_pipe|k_x_fast4|k_zi_fast|k_y_fast" -s 5 -c 5 -o gpurun_out/prof_r1d python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu4b.log 2>&1
echo rc2=$?
