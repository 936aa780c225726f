python scripts/prof_matvec.py 256 2 mf > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_zi_fast|k_zf_pipe" -s 2 -c 2 -o gpurun_out/prof_zi python scripts/prof_matvec.py 256 2 mf > gpurun_out/ncu5a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zi_fast" -s 30 -c 1 -o gpurun_out/prof_zi_fused python scripts/solve_cfg2.py 256 mf > gpurun_out/ncu5b.log 2>&1
echo done
