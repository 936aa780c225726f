python scripts/prof_matvec.py 256 3 mf > gpurun_out/prof2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_zf_fast|k_x_fast2|k_zi_fast" -s 4 -c 3 -o gpurun_out/prof_r1_mf python scripts/prof_matvec.py 256 3 mf > gpurun_out/ncu_mf.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_mf.log
